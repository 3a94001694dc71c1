// peer.cu -- standalone kernels of the peer-memory Ulysses transport
// (rows a1/a2/a6 at P > 1).  The chunk-attention path fuses
// the push into the attention kernel and scatters O from its epilogue
// (fmha_sm100.cu); these kernels are the separate phases:
//   peer_push_kernel      sequence shard -> owners' windows (phase SEND alone,
//                         and the reference K/V of tm_kvcache_put_reference)
//   peer_recv_o_kernel    wait for every rank's O rows, copy the O window to o
//   peer_ref_store_kernel wait for the reference K/V, copy window -> cache, signal
//   peer_wait_kernel      barrier on the done counters
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"
#include "peer.cuh"

namespace tmk {
namespace {

constexpr int kThreads = 512;

int sm_count_peer() { return current_sm_count(); }

__global__ void __launch_bounds__(kThreads) peer_push_kernel(const __grid_constant__ PeerPush pp) {
    for (int T = 0; T < 3; ++T) {
        if (!pp.src[T]) continue;
        peer_push_share(pp, T, threadIdx.x, blockDim.x);
        peer_signal(pp.ctr, pp.own, pp.P, pp.rank, T);
    }
}

// Warp 0 waits on counters[which] >= epoch for every source -- lane s polls
// source s, so the P system-scope acquire round trips overlap -- then the CTA
// proceeds.
__device__ __forceinline__ void cta_wait_all(PeerCounters* own, int which, uint32_t epoch, int P) {
    if (threadIdx.x < 32) {
        const int s = threadIdx.x;
        if (s < P) {
            const uint32_t* c = which < 3 ? &own->arr[which][s] : &own->done[s];
            peer_wait_ge(c, epoch, &own->err);
        }
        __syncwarp();
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kThreads) peer_recv_o_kernel(PeerCounters* own, uint32_t epoch,
                                                               int P, const uint4* owin, uint4* o,
                                                               int B, int64_t Ls, int64_t L,
                                                               int rank, int W) {
    asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: after the attention grid
    cta_wait_all(own, 3, epoch, P);
    // 16-B words, 4 loads in flight per thread; rows of global token >= L are
    // shard padding (zero).  32-bit index math (the window is < 2^31 words).
    const uint32_t n = uint32_t(int64_t(B) * Ls * W);
    // per batch element; a shard lying wholly in padding (e.g. L = 5, P = 4,
    // rank 3) has none: clamp before the cast
    const int64_t vr = L - int64_t(rank) * Ls;
    const uint32_t valid_rows = uint32_t(vr < 0 ? 0 : (vr > Ls ? Ls : vr));
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < n; base += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t i = base + u * stride;
            v[u] = make_uint4(0, 0, 0, 0);
            if (i < n && (i / uint32_t(W)) % uint32_t(Ls) < valid_rows) v[u] = __ldcg(owin + i);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t i = base + u * stride;
            if (i < n) o[i] = v[u];
        }
    }
}

struct RefStoreArgs {
    PeerCounters* ctr[kMaxPeers];
    PeerCounters* own;
    uint32_t epoch;
    int P, rank, B, W;
    int64_t Lw, Lr;
    const uint4* kwin;
    const uint4* vwin;
    uint4* kref;
    uint4* vref;
};

__global__ void __launch_bounds__(kThreads) peer_ref_store_kernel(const __grid_constant__ RefStoreArgs a) {
    cta_wait_all(a.own, 1, a.epoch, a.P);
    cta_wait_all(a.own, 2, a.epoch, a.P);
    const int64_t per_b = a.Lr * a.W, n = int64_t(a.B) * per_b;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = i / per_b, r = i - b * per_b;
        a.kref[i] = __ldcg(a.kwin + b * a.Lw * a.W + r);
        a.vref[i] = __ldcg(a.vwin + b * a.Lw * a.W + r);
    }
    peer_signal(a.ctr, a.own, a.P, a.rank, 3);     // our windows may be reused
}

__global__ void peer_wait_kernel(PeerCounters* own, uint32_t epoch, int P) {
    cta_wait_all(own, 3, epoch, P);
}

}  // namespace

cudaError_t launch_peer_push(const PeerPush& pp, cudaStream_t s, int* launches, int ctas) {
    if (pp.P < 1 || pp.P > kMaxPeers || pp.W <= 0) return cudaErrorInvalidValue;
    if (int64_t(pp.B) * pp.Ls * pp.P * pp.W >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
    peer_push_kernel<<<ctas > 0 ? ctas : sm_count_peer(), kThreads, 0, s>>>(pp);
    if (launches) ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_peer_recv_o(PeerCounters* own, uint32_t epoch, int P, const void* owin, void* o,
                               int B, int64_t Ls, int64_t L, int rank, int row_bytes,
                               cudaStream_t s, int* launches) {
    if (row_bytes % 16) return cudaErrorInvalidValue;
    if (int64_t(B) * Ls * (row_bytes / 16) >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
    const cudaError_t e = launch_pdl(peer_recv_o_kernel, dim3(4 * sm_count_peer()), dim3(kThreads), 0, s,
                                     own, epoch, P, static_cast<const uint4*>(owin),
                                     static_cast<uint4*>(o), B, Ls, L, rank, row_bytes / 16);
    if (e == cudaSuccess && launches) ++*launches;
    return e;
}

cudaError_t launch_peer_ref_store(PeerCounters* const* ctr, PeerCounters* own, uint32_t epoch,
                                  int P, int rank, const void* kwin, const void* vwin, void* kref,
                                  void* vref, int B, int64_t Lw, int64_t Lr, int row_bytes,
                                  cudaStream_t s, int* launches) {
    if (row_bytes % 16 || P < 1 || P > kMaxPeers) return cudaErrorInvalidValue;
    RefStoreArgs a{};
    for (int p = 0; p < P; ++p) a.ctr[p] = ctr[p];
    a.own = own;
    a.epoch = epoch;
    a.P = P;
    a.rank = rank;
    a.B = B;
    a.W = row_bytes / 16;
    a.Lw = Lw;
    a.Lr = Lr;
    a.kwin = static_cast<const uint4*>(kwin);
    a.vwin = static_cast<const uint4*>(vwin);
    a.kref = static_cast<uint4*>(kref);
    a.vref = static_cast<uint4*>(vref);
    peer_ref_store_kernel<<<sm_count_peer(), kThreads, 0, s>>>(a);
    if (launches) ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_peer_wait_done(PeerCounters* own, uint32_t epoch, int P, cudaStream_t s,
                                  int* launches) {
    peer_wait_kernel<<<1, 32, 0, s>>>(own, epoch, P);
    if (launches) ++*launches;
    return cudaGetLastError();
}

}  // namespace tmk
