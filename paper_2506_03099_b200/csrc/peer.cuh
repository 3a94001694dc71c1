// peer.cuh -- device side of the peer-memory Ulysses transport (rows a2, a6;
// PAPER.md P:171 sequence parallelism): stores into other ranks' windows over
// NVLink (addresses mapped with CUDA IPC), monotone counters bumped with
// release semantics at system scope, acquire-polled by the owner.
//
// Ordering argument (PTX memory model):
//   sender thread:  st [window] ... ; fence.acq_rel.sys ; bar.sync
//   sender CTA t0:  atom.add ticket (gpu scope) -- the LAST CTA of the grid then
//                   fence.acq_rel.sys ; red.release.sys.add [owner counter]
//   owner:          ld.acquire.sys [own counter] >= epoch ; fence.proxy.async ; TMA / ld
// The fences make every CTA's window stores precede its ticket increment; the
// last CTA's release to the owner is ordered after all of them (causality is
// transitive), and the owner's acquire makes them visible to its later reads,
// including async-proxy (TMA) reads after the proxy fence.
#pragma once
#include <cstdint>

#include "internal.h"
#include "peer_map.h"

namespace tmk {

// A device-side wait gives up after this many ns (sets PeerCounters::err) so a
// missing peer becomes an error, never a hung GPU.
constexpr unsigned long long kPeerTimeoutNs = 10ull * 1000 * 1000 * 1000;

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_sys_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Wait until *ctr >= target (wrap-safe, counters are monotone mod 2^32).
// Returns false (and flags `err`) on timeout.
__device__ __forceinline__ bool peer_wait_ge(const uint32_t* ctr, uint32_t target, uint32_t* err) {
    if (int32_t(ld_acquire_sys(ctr) - target) >= 0) return true;
    const unsigned long long t0 = globaltimer();
    while (int32_t(ld_acquire_sys(ctr) - target) < 0) {
        if (*reinterpret_cast<volatile uint32_t*>(err)) return false;   // an earlier wait timed out
        __nanosleep(128);
        if (globaltimer() - t0 > kPeerTimeoutNs) {
            atomicExch(err, 1u);
            return false;
        }
    }
    return true;
}

// Last-CTA signal: every thread of the CTA calls this after its stores; when
// the grid's last CTA arrives, it bumps slot `slot` of counter array `which`
// (0..2: arr[T], 3: done) at every peer.
// `wait_epoch` (done signals only, 0 = none): the grid's last CTA then also
// waits until every source's done counter reaches it, so the kernel completes
// only when all ranks' rows have landed here (replaces a receive kernel).
__device__ __forceinline__ void peer_signal(PeerCounters* const* ctr, PeerCounters* own, int P,
                                            int rank, int which, uint32_t wait_epoch = 0) {
    fence_acq_rel_sys();
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t prev = atomicAdd(&own->ticket[which], 1u);
        if (prev == gridDim.x - 1) {
            own->ticket[which] = 0;          // next launch starts from zero (kernel boundary)
            fence_acq_rel_sys();
            for (int p = 0; p < P; ++p) {
                uint32_t* c = which < 3 ? &ctr[p]->arr[which][rank] : &ctr[p]->done[rank];
                red_release_sys_add(c, 1u);
            }
            if (wait_epoch != 0)
                for (int p = 0; p < P; ++p)
                    if (!peer_wait_ge(&own->done[p], wait_epoch, &own->err)) break;
        }
    }
}

// Single-thread release for the whole CTA: the caller's CTA-wide barrier
// (bar.sync) already orders every thread's window stores before this thread,
// so its system-scope fence covers them (cumulativity); then the grid's last
// CTA bumps arr[T][rank] at every owner (`which` = 1 releases K and V).
__device__ __forceinline__ void peer_release(PeerCounters* const* ctr, PeerCounters* own, int P,
                                             int rank, int which) {
    fence_acq_rel_sys();
    const uint32_t prev = atomicAdd(&own->ticket[which], 1u);
    if (prev == gridDim.x - 1) {
        own->ticket[which] = 0;
        fence_acq_rel_sys();
        for (int p = 0; p < P; ++p) {
            if (which == 0) {
                red_release_sys_add(&ctr[p]->arr[0][rank], 1u);
            } else {
                red_release_sys_add(&ctr[p]->arr[1][rank], 1u);
                red_release_sys_add(&ctr[p]->arr[2][rank], 1u);
            }
        }
    }
}

// This CTA's share of pushing tensor T of `pp`: the local shard [B][Ls][H][d]
// is read linearly as 16-B words; the words of head block p of token t go to
// rank p's window row rank*Ls + t (tokens >= L are shard padding, dropped).
// `tid` / `nthr`: this thread's index among the CTA threads taking part.
__device__ __forceinline__ void peer_push_share(const PeerPush& pp, int T, int tid, int nthr) {
    const uint4* src = static_cast<const uint4*>(pp.src[T]);
    const uint32_t n = uint32_t(pp.B) * uint32_t(pp.Ls) * uint32_t(pp.P) * pp.W;   // shard words (< 2^31)
    const uint32_t per = (n + gridDim.x - 1) / gridDim.x;
    const uint32_t lo = blockIdx.x * per;
    const uint32_t hi = min(n, lo + per);
    constexpr int U = 4;
    for (uint32_t base = lo + tid; base < hi; base += U * nthr) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t i = base + u * nthr;
            if (i < hi) v[u] = __ldg(src + i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t i = base + u * nthr;
            if (i >= hi) continue;
            uint32_t p;
            int64_t off;
            if (!peer_push_route(i, pp.W, pp.P, uint32_t(pp.Ls), pp.L, pp.Lw, pp.rank, p, off)) continue;
            static_cast<uint4*>(pp.dst[T][p])[off] = v[u];
        }
    }
}

}  // namespace tmk
