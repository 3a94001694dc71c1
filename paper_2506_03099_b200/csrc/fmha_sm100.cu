// fmha_sm100.cu -- sparse-causal chunk attention core (row a5) for sm_100a.
//
// Computes, per head and query token of chunk c_t,
//     O = softmax(Q K^T / sqrt(d)) V                    (Eq 7)
// where "K and V include tokens from {c_0, c_{t-1}, c_t} only".  The
// mask is realised as a SEGMENT SCHEDULE (row a4): the kernel walks the KV
// tiles of up to three segments (reference c_0, previous c_{t-1}, current
// c_t); every other chunk is never touched.  Ragged segment tails are
// masked to -inf by key index.
//
// Blackwell design.  Work unit = (batch, head, pair of 128-row Q tiles).
// PERSISTENT grid of min(#SMs, 160) CTAs, one per SM: CTA c runs units c,
// c+C, ... (whole); the KV tiles of the T = U mod C tail units are then cut
// into contiguous ranges over the CTAs (stream-K, host-balanced with a
// per-item cost).  A unit cut by range ends becomes pieces; piece 0 is its
// CTA's last item, so it keeps O in TMEM, pulls the other pieces' partials
// (O, m, l) into shared memory by bulk copy and merges them in piece order
// (deterministic, no floating-point atomics).
// Warp roles (384 threads; setmaxnreg gives the softmax warpgroups 216 regs):
//   all         (peer transport, P > 1) push this rank's Q, then K/V shards
//               into the head owners' windows before taking roles.
//   warp 8      TMA producer: per item Q_0, K_lo, Q_1, then K/V through a
//               4-slot smem ring in the order K_lo+1, V_lo, K_lo+2, V_lo+1, ...
//               (K one tile ahead of V; cp.async.bulk.tensor, 128B swizzle).
//   warp 9      S issuer + TMEM owner: S_i(j) = Q_i K_j^T (SS, M=128 N=128
//               K=d, fp32) into ONE S buffer shared by both Q tiles, refilled
//               as soon as the previous S is in registers (s_free).
//   warp 11     PV issuer: O_i += P_i(j) V_j (TS: P_i bf16 from TMEM, V
//               MN-major).  Independent of warp 9 (a blocked PV issue never
//               delays the next S); each commits only its own MMAs.
//   warp 10     a3 append: TMA-stores the current chunk's K/V tiles from the
//               ring to the cache slot.
//   warps 0-7   softmax, one warpgroup per Q tile, one thread per query row
//               (tcgen05.ld 32x32b puts a whole S row in one thread's
//               registers): exact tile max (3-input max tree), running max
//               moved only when it grows by > 8 in log2 units (O and l
//               rescaled then; exact after the final 1/l), exp2 with
//               scale*log2(e) folded into one packed FFMA2, exponentials on the
//               MUFU pipe with a share on an FMA-pipe polynomial (kPolyMask),
//               packed FADD2 row sums, P rounded to bf16 (RNE) and held in
//               registers until the previous PV_i has consumed P_i; epilogue
//               O/l -> bf16 through a per-warp swizzled smem staging buffer
//               (coalesced rows; or the unnormalised partial of a piece).
// Launched with programmatic dependent launch: the prologue overlaps the
// previous kernel's tail (griddepcontrol.wait before any global access).
// TMEM: S [0,128) (shared), P0 [128,192) P1 [192,256), O0 [256,256+d) O1 [256+d,256+2d).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "internal.h"
#include "peer.cuh"
#include "ptx.cuh"

namespace tmk {
namespace {

constexpr int kBM = 128;          // query rows per Q tile
constexpr int kBN = 128;          // keys per KV tile
// K/V smem ring slots: Q 64 KB + 4 x 32 KB + 32 KB of epilogue staging fit in
// 227 KB (the 5th slot measured within noise at 512^2, +3 % at 720^2 when the
// epilogue wrote rows straight from registers; the staging makes every output
// store instruction write 4 rows x 128 B instead of 32 rows x 16 B).
#ifndef TM_KV_STAGES
#define TM_KV_STAGES 4
#endif
constexpr int kStages = TM_KV_STAGES;
constexpr int kEpiBytes = 8 * 4096;   // per softmax warp: 32 rows x 128 B (bf16 half row)
constexpr int kThreads = 384;     // 2 softmax warpgroups + {TMA, MMA, 2 spare} warpgroup
constexpr int kRegsSoftmax = 216; // setmaxnreg budgets (see the static_assert)
constexpr int kRegsOther = 72;
// The CTA launches with 168 regs/thread (64K / 384 rounded down to 8); setmaxnreg
// only redistributes that pool, so the budgets must fit in 384 x 168.
static_assert(256 * kRegsSoftmax + 128 * kRegsOther <= kThreads * 168, "register pool");
constexpr int kHalfBytes = 128 * 128;   // one 64-column (128 B) half of a 128-row tile
// TMEM columns: one S buffer shared by both Q tiles, P0/P1 (bf16 pairs), O0/O1.
constexpr uint32_t kColS = 0, kColP = 128, kColO = 256;
// Lazy running-max threshold (log2 units): weights stay <= 2^8 between rescales.
constexpr float kLazyLog2 = 8.f;
// Fused peer push: the producer releases K/V after this many tile loads at the
// latest (about 3 tiles of compute after Q arrived; the pushes have drained).
constexpr int kKvReleaseLoads = 6;

// One attention problem of a launch: a range of query rows and its KV
// segments (row a4).  A launch holds one problem (a chunk call: segments
// c_0, c_{t-1}, c_t, each its own tensor map) or several sharing one Q, one
// K/V and one O tensor (the f1 full window: query chunk c over key chunks
// {0, c-1, c} as row ranges of the window; f4 audio: a frame's face rows
// over its clamped window of audio frames).
struct Prob {
    int q_row0;                       // first query row in the Q map
    int Lq;                           // query rows
    int o_row0;                       // first output row in O (before o_row_map)
    int o_clip;                       // 1: row o_row0 + Lq is O's end (a TMA store may clip there)
    int n_qpairs;                     // Q-tile pairs per (b, h)
    int n_tiles;                      // KV tiles of a unit
    int nseg;
    int seg_tile_start[kMaxSegments + 1];
    int seg_len[kMaxSegments];
    int seg_row0[kMaxSegments];       // first key row of the segment in its map
    int seg_map[kMaxSegments];        // tensor map (tk / tv index) of the segment
    // PACKED keys (f4 audio windows): the segments are concatenated without
    // padding -- tile j holds keys [128 j, 128 j + 128) of the concatenation,
    // loaded as 128 / packed_R boxes of packed_R rows (tk_sub / tv_sub), each
    // from the segment its first key falls in.  0: every segment tile-padded.
    int packed_R;
    int Lk;                           // packed: total keys
    int seg_key0[kMaxSegments];       // packed: first key of each segment in the concatenation
};

// SCHEDULE BLOCKS.  A launch runs a sequence of blocks; block = (problem,
// head range), scheduled exactly as if it were launched alone: its units
// (b, h, pair of Q tiles) over the C persistent CTAs, R whole rounds (unit
// c + k*C) then the T = U - R*C tail units' KV tiles in contiguous ranges
// (stream-K, bounds of its class).  CTA c runs its items of block 0, then of
// block 1, ...  So a block's arithmetic -- which units are split where and
// merged in which order -- depends only on the block's own shape, never on
// the other blocks of the launch: the f1 window's chunk c equals a streaming
// call over the same segments bit for bit, and with schedule blocks
// of a fixed head count (tm_config.sched_heads) a head's output is bitwise
// the same for every world size.
struct Block {
    int pr;                           // problem
    int h0, nh;                       // heads [h0, h0 + nh)
    int rounds;                       // R: whole rounds
    int cls;                          // stream-K class of the tail
    int tail0;                        // first tail unit (R * C)
    int off;                          // the block's CTA c runs on CTA (c + off) mod C: consecutive
                                      // blocks' tails start where the previous tail ended
};
struct SkClass {
    int ctas;                         // G': CTAs with a tail range
    int bound[kMaxPersistentCtas + 1];   // CTA c takes tail tiles [bound[c], bound[c+1])
};

struct __align__(64) FmhaParams {
    CUtensorMap tq;                   // Q [B][L][H][d]
    CUtensorMap tk[kMaxSegments];     // K maps [B][len][H][d]
    CUtensorMap tv[kMaxSegments];     // V maps
    CUtensorMap tk_store, tv_store;   // a3: cache slot that the current segment is copied to
    CUtensorMap tk_sub, tv_sub;       // packed problems: the tk[0] / tv[0] tensors with packed_R-row boxes
    int store_seg;                    // segment whose tiles are appended to the slot (-1: none; one problem only)
    int nmaps;                        // tk / tv maps in use
    int nprob;
    Prob prob[kMaxProblems];
    int nblk, ncls;
    Block blk[kMaxBlocks];
    SkClass cls[kMaxSkClasses];
    int cls_key[kMaxSkClasses][2];    // host bookkeeping: (T, n) of each class
    const int* o_row_map;             // nullable: output row of problem-local query q is o_row0 + map[q]
    int H, B;
    float scale_log2;                 // softmax scale * log2(e)
    // Output rows (a6 scatter): query row q is stored to o_dst[q / o_rows], row
    // q % o_rows, heads [o_h0, o_h0 + H) of o_H; P = 1: o_dst[0] = o, o_rows = Lq.
    uint16_t* o_dst[kMaxPeers];       // bf16 bits [B][o_rows][o_H][d] each
    CUtensorMap to;                   // o as a TMA store map (box 32 rows x 64), one owner only
    int tma_epi;                      // 1: epilogue rows leave through TMA stores of the staging
    int exit_wait_full;               // A/B: wait for the epilogue TMA stores' global writes at exit
    int dbg_nomerge;                  // timing experiments only (TM_DBG_NOMERGE=1): pieces store unmerged
    int dbg_nolatestore;              // timing bound only (TM_DBG_NOLATESTORE=1): no append stores in a CTA's last item
    int64_t o_bstride;                // rows between batch elements of an o_dst
    int o_rows, o_H, o_h0;
    // f4 zero fill (spare warp, concurrent with the attention): rows r in
    // [zf_row0, zf_row0 + zf_rows) of each batch element of o_dst[0] whose token
    // r % zf_T has zf_inv[token] < 0 are zeroed (no audio update).
    const int* zf_inv;
    int zf_T;
    int64_t zf_row0, zf_rows;
    // Peer transport: waits on the own counters before Q tiles (T=0)
    // and before tiles of segment wait_seg (K: T=1, V: T=2); fused push of
    // this rank's shard at kernel start; done signal at kernel end.
    int peer, push, signal_done, wait_seg, src_rows, P, rank;
    uint32_t wait_done;               // nonzero: the last CTA waits for every rank's done (zero-copy O)
    uint32_t epoch[3];
    PeerCounters* own;
    PeerCounters* done_ctr[kMaxPeers];
    PeerPush pp;
    // persistent schedule
    int ctas;                         // C: persistent CTAs the blocks are scheduled over
    int l2_prefetch;                  // K/V tiles of the first item prefetched into L2 (with its Q) before the PDL wait
    float* part;                      // piece partials: per (block, CTA) slot [d/8][256] fp16x8 + m, l, m-s [256]
    unsigned long long* counters;     // per (block, first CTA of a split unit, Q tile): bit n = contributor n in; zero between launches
    unsigned long long* trace;        // debug timeline (TM_TRACE=1), CTA 0 only; may be null
};

// Debug timeline: role r in [0,13) owns trace[r*kTraceCap ..]; entry =
// clock64() << 8 | event code.  Only CTA 0 records; off when p.trace == 0.
[[maybe_unused]] constexpr int kTraceCap = 4096;
// Compiled in only with -DTM_TRACE_ENABLED (TM_TRACE_BUILD=1 python -m
// paper_2506_03099_b200.build); the production build has no trace code.
__device__ __forceinline__ void trace_ev(const FmhaParams& p, int role, int& n, int code) {
#ifdef TM_TRACE_ENABLED
    if (p.trace != nullptr && blockIdx.x == 0 && n < kTraceCap)
        p.trace[role * kTraceCap + n++] = (static_cast<unsigned long long>(clock64()) << 8) | code;
#else
    (void)p; (void)role; (void)n; (void)code;
#endif
}

// Per-CTA span stamps (globaltimer ns) after the role timelines; debug build only.
__device__ __forceinline__ void trace_span(const FmhaParams& p, int j, long long val = -1) {
#if defined(TM_TRACE_ENABLED) || defined(TM_SPANS_ENABLED)
    if (p.trace != nullptr) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[13 * kTraceCap + blockIdx.x * 8 + j] = val >= 0 ? (unsigned long long)val : t;
    }
#else
    (void)p; (void)j; (void)val;
#endif
}

struct Item {
    int pr, blk, b, h, qp, lo, hi, piece;
    int cfirst, npieces, pidx;        // split units: first CTA, piece count, this piece's index
    int cl;                           // this CTA's index within the block (blockIdx.x - off mod C)
};

// Tail (stream-K) CTA holding tile x of the flattened tail space: the c with
// sk_bound[c] <= x < sk_bound[c+1] (ranges are non-empty; binary search).
__device__ __forceinline__ int sk_cta_of(const SkClass& k, int x) {
    int lo = 0, hi = k.ctas - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (k.bound[mid] <= x) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}
// Piece k of a split unit whose first CTA is cf is held by CTA cf + k.  Piece
// 0 is CTA cf's LAST item and merges; piece k >= 1 is CTA cf+k's FIRST item and
// leaves its partial in slot cf + k (one partial slot per CTA suffices).

// Item k of this CTA within block bi: first its R whole units c, c+C, ...;
// then its range of the block's tail tiles (stream-K: each of the first G'
// CTAs takes a contiguous range of the T tail units' KV tiles, sized on the
// host so that tiles plus a per-item cost are equal (tail_bounds); a unit cut
// by range ends becomes pieces, merged by piece 0).
__device__ __forceinline__ bool get_item(const FmhaParams& p, int bi, int k, Item& it) {
    const Block& B = p.blk[bi];
    const Prob& P = p.prob[B.pr];
    const int c = B.off ? (int(blockIdx.x) + p.ctas - B.off) % p.ctas : int(blockIdx.x);
    const int n = P.n_tiles;
    int unit;
    it.pr = B.pr;
    it.blk = bi;
    it.cl = c;
    it.cfirst = 0;
    it.npieces = 1;
    it.pidx = 0;
    if (k < B.rounds) {
        unit = c + k * p.ctas;
        it.lo = 0;
        it.hi = n;
        it.piece = 0;
    } else {
        if (B.cls < 0) return false;
        const SkClass& K = p.cls[B.cls];
        if (c >= K.ctas) return false;
        const int start = K.bound[c], end = K.bound[c + 1];
        const int u = start / n + (k - B.rounds);
        const int ub = u * n;
        if (start >= end || ub >= end) return false;
        it.lo = (start > ub ? start : ub) - ub;
        it.hi = (end < ub + n ? end : ub + n) - ub;
        it.piece = it.lo > 0 || it.hi < n;
        if (it.piece) {
            it.cfirst = sk_cta_of(K, ub);
            it.npieces = sk_cta_of(K, ub + n - 1) - it.cfirst + 1;
            it.pidx = c - it.cfirst;
        }
        unit = B.tail0 + u;
    }
    it.qp = unit % P.n_qpairs;
    const int bh = unit / P.n_qpairs;
    it.h = B.h0 + bh % B.nh;
    it.b = bh / B.nh;
    return true;
}

// Every role walks the same item sequence: block by block, each block's items.
struct Cursor {
    int bi = 0, k = 0;
};
__device__ __forceinline__ bool next_item(const FmhaParams& p, Cursor& cu, Item& it) {
    while (cu.bi < p.nblk) {
        if (get_item(p, cu.bi, cu.k, it)) {
            ++cu.k;
            return true;
        }
        ++cu.bi;
        cu.k = 0;
    }
    return false;
}

// KV tile j of a unit of problem `pr`: its segment, first key row within the
// segment, valid keys (ragged tail masked), and the row in the segment's map.
__device__ __forceinline__ int packed_seg(const Prob& P, int key) {   // segment holding `key`
    int seg = 0;
#pragma unroll
    for (int s = 1; s < kMaxSegments; ++s)
        if (s < P.nseg && key >= P.seg_key0[s]) seg = s;
    return seg;
}
template <bool kMulti>
__device__ __forceinline__ void tile_info(const FmhaParams& p, int pr, int j, int& seg, int& row,
                                          int& valid) {
    const Prob& P = p.prob[pr];
    if (kMulti && P.packed_R) {
        const int k0 = j * kBN;
        seg = packed_seg(P, k0);
        row = k0 - P.seg_key0[seg];            // key offset within its segment
        valid = min(kBN, P.Lk - k0);
        return;
    }
    seg = 0;
#pragma unroll
    for (int s = 1; s < kMaxSegments; ++s)
        if (s < P.nseg && j >= P.seg_tile_start[s]) seg = s;
    row = (j - P.seg_tile_start[seg]) * kBN;
    valid = min(kBN, P.seg_len[seg] - row);
}

// Position q (0..2n-1) of an item's K/V load sequence K0, K1, V0, K2, V1, ...,
// V_{n-1} (K one tile ahead of V) -> (tile offset jj, is_v).
__device__ __forceinline__ void load_order(int q, int nkv, int& jj, int& kv) {
    if (q == 0) { jj = 0; kv = 0; }
    else if (q == 2 * nkv - 1) { jj = nkv - 1; kv = 1; }
    else if (q & 1) { jj = (q + 1) / 2; kv = 0; }
    else { jj = q / 2 - 1; kv = 1; }
}
// a3 fused append: tile `row / kBN` of the current segment is written to the
// cache slot by exactly one item of its (b, h): the unit with qp == tile % n_qpairs
// (or the piece of that unit whose KV range holds it).
__device__ __forceinline__ bool stores_tile(const FmhaParams& p, const Item& it, int seg, int row) {
    return seg == p.store_seg && (row / kBN) % p.prob[it.pr].n_qpairs == it.qp;
}

// Destination of output row q of head h (row a6: the owner's O window when the
// path is Ulysses-sharded over peer memory, else o itself); null for pad rows.
template <int D, int kKind>
__device__ __forceinline__ uint16_t* out_row(const FmhaParams& p, const Prob& P, int b, int q, int h) {
    if (q >= P.Lq) return nullptr;
    if (kKind != 2 || p.o_rows >= P.Lq) {   // one owner (P = 1): no division
        const int row = P.o_row0 + (p.o_row_map ? p.o_row_map[q] : q);
        return p.o_dst[0] + ((int64_t(b) * p.o_bstride + row) * p.o_H + p.o_h0 + h) * D;
    }
    int own;
    const int64_t row = peer_out_route(b, q, h, p.o_rows, p.o_bstride, p.o_H, p.o_h0, own);
    return p.o_dst[own] + row * D;
}

// Epilogue: the warp's 32 threads each hold one output row (lane l = row
// q0 + l) as D fp32 values in TMEM columns [tsrc, tsrc + D); scale, round to
// bf16 and store.  Through a 4 KB per-warp staging buffer (32 rows x 64
// columns, 16-B chunks XOR-swizzled by row: conflict-free both ways) each
// store instruction writes 4 rows x 128 B instead of 32 rows x 16 B.
template <int D, int kKind>
__device__ __forceinline__ void store_rows_bf16(const FmhaParams& p, const Prob& P, uint32_t tsrc,
                                                float scale, uint8_t* stg, int b, int q0, int h,
                                                int lane) {
    // TMA store of the warp's 32 rows when they are contiguous in O and either
    // all inside the problem or clipped by O's end (a window's inner problems
    // must not spill into the next problem's rows).
    if (p.tma_epi && (q0 + 32 <= P.Lq || P.o_clip)) {
        // One owner: the swizzled staging tile is exactly a 128B-swizzled TMA box
        // (32 rows x 64 columns), so lane 0 stores it asynchronously (rows past
        // Lq clipped) and the warp moves on; the buffer is reused only after the
        // previous store has read it.
#pragma unroll 1
        for (int half = 0; half < D / 64; ++half) {
            uint32_t o[64];
            tmem_ld32(tsrc + half * 64, o);
            tmem_ld32(tsrc + half * 64 + 32, o + 32);
            tmem_wait_ld();
            if (lane == 0) tma_store_wait_read();
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                uint4 v;
                v.x = pack_bf16x2(__uint_as_float(o[8 * j]) * scale, __uint_as_float(o[8 * j + 1]) * scale);
                v.y = pack_bf16x2(__uint_as_float(o[8 * j + 2]) * scale, __uint_as_float(o[8 * j + 3]) * scale);
                v.z = pack_bf16x2(__uint_as_float(o[8 * j + 4]) * scale, __uint_as_float(o[8 * j + 5]) * scale);
                v.w = pack_bf16x2(__uint_as_float(o[8 * j + 6]) * scale, __uint_as_float(o[8 * j + 7]) * scale);
                *reinterpret_cast<uint4*>(stg + lane * 128 + ((j ^ (lane & 7)) << 4)) = v;
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                tma_store_4d(&p.to, stg, half * 64, h, P.o_row0 + q0, b);
                tma_store_commit();
            }
        }
        return;
    }
    // This lane stores rows t*4 + lane/8 (t < 8), 16 B at column chunk lane%8:
    // destinations computed once for both halves (32-bit index math).
    uint16_t* dsts[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const int q = q0 + t * 4 + (lane >> 3);
        dsts[t] = out_row<D, kKind>(p, P, b, q, h);
    }
#pragma unroll 1
    for (int half = 0; half < D / 64; ++half) {
        uint32_t o[64];
        tmem_ld32(tsrc + half * 64, o);
        tmem_ld32(tsrc + half * 64 + 32, o + 32);
        tmem_wait_ld();
#ifdef TM_SPANS_MERGE
        if (threadIdx.x == 0 && half == 0) trace_span(p, 1);
#endif
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            uint4 v;
            v.x = pack_bf16x2(__uint_as_float(o[8 * j]) * scale, __uint_as_float(o[8 * j + 1]) * scale);
            v.y = pack_bf16x2(__uint_as_float(o[8 * j + 2]) * scale, __uint_as_float(o[8 * j + 3]) * scale);
            v.z = pack_bf16x2(__uint_as_float(o[8 * j + 4]) * scale, __uint_as_float(o[8 * j + 5]) * scale);
            v.w = pack_bf16x2(__uint_as_float(o[8 * j + 6]) * scale, __uint_as_float(o[8 * j + 7]) * scale);
            *reinterpret_cast<uint4*>(stg + lane * 128 + ((j ^ (lane & 7)) << 4)) = v;
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const int r = t * 4 + (lane >> 3), j = lane & 7;
            const uint4 v = *reinterpret_cast<const uint4*>(stg + r * 128 + ((j ^ (r & 7)) << 4));
            if (dsts[t]) *reinterpret_cast<uint4*>(dsts[t] + half * 64 + j * 8) = v;
        }
        __syncwarp();
    }
}

// Peer transport: before the producer's first TMA read of window rows
// [r0, r0 + n) of tensor T, wait until every source rank owning them has
// landed its push (once per source per launch; `ok` caches satisfied ones).
__device__ __forceinline__ void peer_ready(const FmhaParams& p, uint32_t& ok, int T, int r0, int n) {
    if (n <= 0) return;
    const int s0 = r0 / p.src_rows, s1 = (r0 + n - 1) / p.src_rows;
    bool waited = false;
    for (int s = s0; s <= s1; ++s) {
        const uint32_t bit = 1u << (T * kMaxPeers + s);
        if (ok & bit) continue;
        peer_wait_ge(&p.own->arr[T][s], p.epoch[T], &p.own->err);
        ok |= bit;
        waited = true;
    }
    if (waited) fence_proxy_async_global();   // generic-proxy acquire -> TMA (async proxy) reads
}

// One merge step of an output element (stream-K pieces):
// o <- o * wo + wk * x with explicit roundings (the product o * wo rounded,
// then one FMA), so every code path gives the same bits.
__device__ __forceinline__ uint32_t merge_elem(uint32_t o, float wo, float wk, float x) {
    return __float_as_uint(__fmaf_rn(wk, x, __fmul_rn(__uint_as_float(o), wo)));
}

__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {   // RN, lo in the low half
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ float2 unpack_f16x2(uint32_t v) {
    const __half2 h = *reinterpret_cast<const __half2*>(&v);
    return __half22float2(h);
}

__device__ __forceinline__ float max3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ uint64_t f2u(float2 a) { return *reinterpret_cast<uint64_t*>(&a); }
__device__ __forceinline__ float2 u2f(uint64_t a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}

// 2^x for a pair, on the FMA pipe: x = n + f, n = rint(x), f in [-0.5, 0.5];
// 2^f by a degree-3 minimax polynomial (max rel. error 8.0e-5, far below
// the bf16 rounding of P); 2^n inserted into the exponent field.  x is
// clamped at -125 (result stays a normal float; 2^-125 is ~0 for softmax).
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
    constexpr float kMagic = 12582912.f;    // 1.5 * 2^23: round-to-nearest trick
    x.x = fmaxf(x.x, -125.f);
    x.y = fmaxf(x.y, -125.f);
    const float2 j = fadd2(x, make_float2(kMagic, kMagic));
    const float2 n = fadd2(j, make_float2(-kMagic, -kMagic));
    const float2 f = ffma2(n, make_float2(-1.f, -1.f), x);
    float2 p = ffma2(make_float2(0.055171094834804535f, 0.055171094834804535f), f,
                     make_float2(0.24260999262332916f, 0.24260999262332916f));
    p = ffma2(p, f, make_float2(0.6932609677314758f, 0.6932609677314758f));
    p = ffma2(p, f, make_float2(0.9999281167984009f, 0.9999281167984009f));
    // exponent insertion on the ALU pipe (SHL + IADD), not IMAD on the busy FMA pipe
    uint32_t ex, ey;
    asm("{\n\t.reg .b32 t;\n\tshl.b32 t, %1, 23;\n\tadd.u32 %0, %2, t;\n\t}"
        : "=r"(ex) : "r"(__float_as_uint(j.x)), "r"(__float_as_uint(p.x)));
    asm("{\n\t.reg .b32 t;\n\tshl.b32 t, %1, 23;\n\tadd.u32 %0, %2, t;\n\t}"
        : "=r"(ey) : "r"(__float_as_uint(j.y)), "r"(__float_as_uint(p.y)));
    return make_float2(__uint_as_float(ex), __uint_as_float(ey));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
        : "memory");
}

// Stream-K piece publication: release by the publishing thread after a
// barrier over its warpgroup (cumulative), acquire by the merger's poller.
__device__ __forceinline__ void red_release_or(unsigned long long* a, unsigned long long v) {
    asm volatile("red.release.gpu.global.or.b64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ void wg_bar(int i) {   // the 128 threads of softmax warpgroup i
    asm volatile("bar.sync %0, 128;" ::"r"(2 + i) : "memory");
}

// Stream-K partials (scratch, zeroed at context creation).  Per (block, CTA)
// slot of 256 d + 512 floats: three TILE PARTIALS of 64 d + 384 floats, each
// 128 fp16 O rows as [d/8][128] uint4 (row-fastest: a warp's 16-B accesses are
// contiguous) followed by m[128], l[128], (m - s)[128]:  kind 0 / 1 = the
// CTA's first item (a piece k >= 1) for Q tile 0 / 1; kind 2 = its last item
// (piece 0 of a co-merged unit) for Q tile 1.  Counters: two per (block,
// first CTA of a split unit), one per Q tile, after the slots.
template <int D>
__device__ __forceinline__ float* part_tile(const FmhaParams& p, int blk, int cta, int kind) {
    constexpr int kTileFloats = 64 * D + 3 * 128;
    static_assert(3 * kTileFloats <= 256 * D + 512, "tile partials fit the slot");
    return p.part + (size_t(blk) * kMaxPersistentCtas + cta) * (256 * D + 512) + kind * kTileFloats;
}

// kKind: 0 one-GPU chunk attention; 1 launches of several problems (f1 window,
// f4 audio) -- the only ones with packed keys or the f4 zero fill; 2 the peer
// transport (fused push, window waits, routed O rows, done signal).  Each kind
// compiles only its own paths: code the chunk-attention kernel never runs
// measured 1-3 % slower when compiled in (layout).
template <int D, uint32_t kPolyMask, int kKind>
__global__ void __launch_bounds__(kThreads, 1) fmha_sm100_kernel(const __grid_constant__ FmhaParams p) {
    constexpr bool kMulti = kKind == 1, kPeerKind = kKind == 2;
    constexpr int kTileBytes = kBN * D * 2;
    constexpr int kTileO = 64 * D;   // floats of a tile partial's fp16 O rows (then m, l, m - s)
    constexpr uint32_t kIdescS = make_idesc_bf16(kBM, kBN, 0, 0);   // Q, K both K-major
    constexpr uint32_t kIdescO = make_idesc_bf16(kBM, D, 0, 1);     // P (TMEM), V MN-major

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* sQ = smem;                                  // 2 tiles
    uint8_t* sKV = smem + 2 * kTileBytes;                // kStages slots
    uint8_t* sEpi = sKV + kStages * kTileBytes;          // epilogue staging, 4 KB per softmax warp
    uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + kEpiBytes);
    uint64_t* q_full = bars;                 // [2]
    uint64_t* q_empty = q_full + 2;          // [2]
    uint64_t* kv_full = q_empty + 2;         // [kStages]
    uint64_t* kv_empty = kv_full + kStages;  // [kStages]
    uint64_t* s_full = kv_empty + kStages;   // [2]  S_i computed into the S buffer
    uint64_t* p_full = s_full + 2;           // [2]  P_i stored into TMEM
    uint64_t* o_final = p_full + 2;          // [2]  last PV_i of an item complete
    uint64_t* o_empty = o_final + 2;         // [2]  epilogue done reading O_i
    uint64_t* o_done = o_empty + 2;          // [2]  each PV_i complete (P_i reusable)
    uint64_t* s_free = o_done + 2;           // [1]  S buffer loaded into registers
    uint64_t* store_idle = s_free + 1;       // [1] append warp done (one phase per launch)
    uint64_t* merge_bar = store_idle + 1;    // [6] merge buffer j of warpgroup i: 3 i + j
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(merge_bar + 6);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) trace_span(p, 0);

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 128);
            mbar_init(&o_final[i], 1);
            mbar_init(&o_empty[i], 128);
            mbar_init(&o_done[i], 1);
        }
        mbar_init(s_free, 128);
        mbar_init(store_idle, 1);
        for (int j = 0; j < 6; ++j) mbar_init(&merge_bar[j], 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&kv_full[s], 1);
            // with the a3 append active, a fill is released by the MMA commit AND
            // by the append warp (which has then passed it, stored or not)
            mbar_init(&kv_empty[s], p.store_seg >= 0 ? 2 : 1);
        }
        fence_mbar_init();
    }
    if (warp == 8 && lane == 0) {
        tma_prefetch(&p.tq);
        for (int s = 0; s < p.nmaps; ++s) {
            tma_prefetch(&p.tk[s]);
            tma_prefetch(&p.tv[s]);
        }
        if (kMulti && p.prob[0].packed_R) {
            tma_prefetch(&p.tk_sub);
            tma_prefetch(&p.tv_sub);
        }
        // The first item's Q tiles and first K/V tiles into L2 while the
        // previous grid drains (one-GPU problems; peer windows are filled by
        // other ranks during the launch).  TM_L2_PREFETCH=n: n K/V tiles (0: off).
        Item it0;
        Cursor cu0;
        if (p.l2_prefetch && next_item(p, cu0, it0)) {
            for (int i = 0; i < 2; ++i)
                for (int hf = 0; hf < D / 64; ++hf)
                    tma_prefetch_l2_4d(&p.tq, hf * 64, it0.h,
                                       p.prob[it0.pr].q_row0 + it0.qp * 2 * kBM + i * kBM, it0.b);
            for (int j = it0.lo; j < it0.hi && j < it0.lo + p.l2_prefetch; ++j) {
                int seg, row, valid;
                tile_info<kMulti>(p, it0.pr, j, seg, row, valid);
                const Prob& P0 = p.prob[it0.pr];
                const int m = P0.seg_map[seg], r = P0.seg_row0[seg] + row;
                for (int hf = 0; hf < D / 64; ++hf) {
                    tma_prefetch_l2_4d(&p.tk[m], hf * 64, it0.h, r, it0.b);
                    tma_prefetch_l2_4d(&p.tv[m], hf * 64, it0.h, r, it0.b);
                }
            }
        }
    }
    if (warp == 9) tmem_alloc(tmem_holder, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;
#ifdef TM_SPANS_PROLOGUE
    if (threadIdx.x == 0) trace_span(p, 4);   // (spans A/B) prologue done
#endif
    // Programmatic dependent launch: everything above (barriers, TMEM, tensor-map
    // prefetch) overlaps the previous kernel's tail; no global data is touched
    // before the previous grid has completed.  (No-op without the attribute.)
    asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef TM_SPANS_PROLOGUE
    if (threadIdx.x == 0) trace_span(p, 5);   // (spans A/B) previous grid complete
#endif
    if (kPeerKind && p.push) {
        // a2 fused.  All 384 threads store this rank's shard of Q into the owners'
        // windows (NVLink stores).  Then warp 10 alone releases Q (a system-scope
        // fence waits until the CTA's stores have landed; the grid's last CTA
        // bumps arr[0][rank] at every owner) while the other 11 warps store K
        // and V.  K/V are released later by the producer (peer_release), once
        // their stores have long drained, so no role waits for NVLink: owners
        // start on Q and the cached c_0 / c_{t-1} segments while c_t is in flight.
        peer_push_share(p.pp, 0, threadIdx.x, kThreads);
        __syncthreads();
        if (warp == 10) {
            if (lane == 0) peer_release(p.pp.ctr, p.pp.own, p.pp.P, p.pp.rank, 0);
            __syncwarp();
        } else {
            const int t = threadIdx.x < 320 ? threadIdx.x : threadIdx.x - 32;
            peer_push_share(p.pp, 1, t, kThreads - 32);
            peer_push_share(p.pp, 2, t, kThreads - 32);
        }
        __syncthreads();
    }

    if (warp >= 8) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsOther));
      if (warp == 8) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            int tn = 0;
            uint32_t kv_it = 0, n_item = 0;
            uint32_t ok = 0;                               // peer (tensor, source) pairs already landed
            bool kv_released = !kPeerKind || !p.push;      // fused push: K/V not yet released
#ifdef TM_SPANS_PROD
            long long cyc_empty = 0, cyc_store = 0;
#endif
            int n_loads = 0;
            Item it;
            Cursor cu;
            for (; next_item(p, cu, it); ++n_item) {
                // Load order Q_0, K_lo, Q_1, K_lo+1, V_lo, K_lo+2, V_lo+1, ..., V_hi-1:
                // S_0(lo) needs only Q_0 and K_lo, and K runs one tile ahead of V,
                // matching the MMA's use (S(j+1) before PV(j)).
                const int nkv = it.hi - it.lo;
                for (int step = 0; step < 2 * nkv + 2; ++step) {
                    if (step == 0 || step == 2) {
                        const int i = step >> 1;
                        if (kPeerKind && p.peer) {
                            const int r0 = it.qp * 2 * kBM + i * kBM;
                            peer_ready(p, ok, 0, r0, min(kBM, p.prob[0].Lq - r0));
                        }
                        mbar_wait(&q_empty[i], (n_item & 1) ^ 1);
                        mbar_arrive_expect_tx(&q_full[i], kTileBytes);
                        for (int hf = 0; hf < D / 64; ++hf)
                            tma_load_4d(sQ + i * kTileBytes + hf * kHalfBytes, &p.tq, &q_full[i],
                                        hf * 64, it.h,
                                        p.prob[it.pr].q_row0 + it.qp * 2 * kBM + i * kBM, it.b);
                        continue;
                    }
                    const int q = step == 1 ? 0 : step - 2;
                    int jj, kv;
                    load_order(q, nkv, jj, kv);
                    int seg, row, valid;
                    tile_info<kMulti>(p, it.pr, it.lo + jj, seg, row, valid);
                    const int s = kv_it % kStages;
                    trace_ev(p, 0, tn, 3 + kv);
#ifdef TM_SPANS_PROD
                    long long tw0 = clock64();
#endif
                    mbar_wait(&kv_empty[s], ((kv_it / kStages) & 1) ^ 1);
#ifdef TM_SPANS_PROD
                    long long tw1 = clock64();
                    cyc_empty += tw1 - tw0;
#endif
                    // (With the a3 append active, kv_empty also counts the append
                    // warp's release of the slot's previous fill, stored or not:
                    // the append warp waits on EVERY fill's kv_full phase in order,
                    // and were a slot refillable without it, two fills of a slot
                    // whose store is not pending could complete while the append
                    // warp is still blocked on an earlier store -- a parity ABA
                    // that desynchronised it: a hang, seen at 10 and 20 heads under
                    // some timings.)
                    // Release this CTA's K/V pushes before the first wait on K/V
                    // (own rank included) or after a few loads, whichever first:
                    // by then the stores have drained and the fence is cheap.
                    if (!kv_released && (seg == p.wait_seg || ++n_loads > kKvReleaseLoads)) {
                        peer_release(p.pp.ctr, p.pp.own, p.pp.P, p.pp.rank, 1);
                        kv_released = true;
                    }
                    if (kPeerKind && p.peer && seg == p.wait_seg) peer_ready(p, ok, 1 + kv, row, valid);
                    trace_ev(p, 0, tn, 1 + kv);
                    const Prob& P = p.prob[it.pr];
                    mbar_arrive_expect_tx(&kv_full[s], kTileBytes);
                    const int k0t = (it.lo + jj) * kBN;
                    if (kMulti && P.packed_R &&
                        !(k0t + kBN <= P.Lk && packed_seg(P, k0t) == packed_seg(P, k0t + kBN - 1))) {
                        // packed keys across segments: 128 / R boxes of R rows,
                        // each from its own segment (box offsets are multiples of
                        // 1024 B, so the 128-B swizzle matches a whole-tile load);
                        // boxes past the last key reload key 0 (finite data,
                        // masked to -inf).  A tile inside one segment is one
                        // 128-row box per half, as below.
                        const int R = P.packed_R;
                        const CUtensorMap* m = kv ? &p.tv_sub : &p.tk_sub;
                        for (int r = 0; r < kBN / R; ++r) {
                            int kk = (it.lo + jj) * kBN + r * R;
                            if (kk >= P.Lk) kk = 0;
                            const int sg = packed_seg(P, kk);
                            const int rr = P.seg_row0[sg] + kk - P.seg_key0[sg];
                            for (int hf = 0; hf < D / 64; ++hf)
                                tma_load_4d(sKV + s * kTileBytes + hf * kHalfBytes + r * R * 128, m,
                                            &kv_full[s], hf * 64, it.h, rr, it.b);
                        }
                    } else {
                        const int mi = P.seg_map[seg];
                        const CUtensorMap* m = kv ? &p.tv[mi] : &p.tk[mi];
                        for (int hf = 0; hf < D / 64; ++hf)
                            tma_load_4d(sKV + s * kTileBytes + hf * kHalfBytes, m, &kv_full[s],
                                        hf * 64, it.h, P.seg_row0[seg] + row, it.b);
                    }
                    (void)k0t;
                    ++kv_it;
                }
            }
            if (!kv_released) peer_release(p.pp.ctr, p.pp.own, p.pp.P, p.pp.rank, 1);
#ifdef TM_SPANS_PROD
            trace_span(p, 1, cyc_store);
            trace_span(p, 5, cyc_empty);
#endif
        }
      } else if (warp == 10) {
#ifdef TM_TRACE_ENABLED
        if (lane == 1) {
        // ------------------------------------------------ trace observer (debug build)
        // Records when each S MMA group lands (30+i = S_i(j) complete).  The
        // observer gates nothing, so it can lag two phases behind s_full and
        // alias; it then stops observing after a bounded wait instead of
        // trapping (debug instrumentation only).
        if (p.trace != nullptr && blockIdx.x == 0) {
            int tn = 0;
            uint32_t g = 0;
            Item it;
            Cursor cu;
            bool live = true;
            while (live && next_item(p, cu, it))
                for (int j = it.lo; live && j < it.hi; ++j, ++g)
                    for (int i = 0; live && i < 2; ++i) {
                        const uint32_t a = smem_u32(&s_full[i]);
                        const long long t0 = clock64();
                        while (!mbar_try_wait(a, g & 1))
                            if (clock64() - t0 > (1ll << 24)) { live = false; break; }
                        if (live) trace_ev(p, 4, tn, 30 + i);
                    }
        }
        }
#endif
        // ------------------------------------------------ a3 append: TMA store of c_t tiles
        if (lane == 0 && p.store_seg >= 0) {
            uint32_t kv_it = 0;
            int tn = 0;
            int pend = -1;                 // slot of the last stored fill, its read maybe in flight
            Item it;
            Cursor cu;
            while (next_item(p, cu, it)) {
                const int nkv = it.hi - it.lo;
                bool skip_store = false;
                if (p.dbg_nolatestore) {
                    Cursor pk = cu;
                    Item nx;
                    skip_store = !next_item(p, pk, nx);
                }
                for (int q = 0; q < 2 * nkv; ++q, ++kv_it) {
                    int jj, kv;
                    load_order(q, nkv, jj, kv);
                    int seg, row, valid;
                    tile_info<kMulti>(p, it.pr, it.lo + jj, seg, row, valid);
                    // Observe EVERY position's kv_full phase in order, and release
                    // every fill (stored or not) through kv_empty: the producer
                    // refills a slot only after that, so no slot can complete two
                    // phases ahead of this warp (parity ABA either way).  A stored
                    // fill is released once the TMA store has read it; up to one
                    // such read stays in flight while this warp moves on, flushed
                    // before its slot comes round again.
                    const int s = kv_it % kStages;
                    if (pend == s) {
                        tma_store_wait_read();
                        mbar_arrive(&kv_empty[pend]);
                        pend = -1;
                    }
                    mbar_wait(&kv_full[s], (kv_it / kStages) & 1);
                    trace_ev(p, 2, tn, 40 + kv);
                    if (!skip_store && stores_tile(p, it, seg, row)) {
                        fence_proxy_async_smem();
                        const CUtensorMap* m = kv ? &p.tv_store : &p.tk_store;
                        for (int hf = 0; hf < D / 64; ++hf)
                            tma_store_4d(m, sKV + s * kTileBytes + hf * kHalfBytes, hf * 64, it.h, row,
                                         it.b);
                        tma_store_commit();
                        if (pend >= 0) {
                            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                            mbar_arrive(&kv_empty[pend]);
                        }
                        pend = s;
                    } else {
                        mbar_arrive(&kv_empty[s]);
                    }
                }
            }
            if (pend >= 0) {
                tma_store_wait_read();
                mbar_arrive(&kv_empty[pend]);
            }
        }
        if (lane == 0) mbar_arrive(store_idle);   // the ring is no longer read by TMA stores
        if (kMulti && p.zf_inv != nullptr) {
            // f4: zero the non-face rows of o, this CTA's share (warp-uniform branch)
            // 32 of this CTA's rows per batch: each lane loads one row's face-map
            // entry (one L2 round trip per batch, not per row), then the warp
            // zeroes the batch's non-face rows.
            const int words = p.o_H * D / 8;                  // 16-B words per token row
            const int64_t total = int64_t(p.B) * p.zf_rows;
            const uint4 z = make_uint4(0, 0, 0, 0);
            for (int64_t r0 = blockIdx.x; r0 < total; r0 += 32 * int64_t(gridDim.x)) {
                const int64_t rl = r0 + int64_t(lane) * gridDim.x;
                bool zero = false;
                if (rl < total) zero = __ldg(p.zf_inv + (p.zf_row0 + rl % p.zf_rows) % p.zf_T) < 0;
                uint32_t m = __ballot_sync(0xffffffffu, zero);
                while (m) {
                    const int k = __ffs(m) - 1;
                    m &= m - 1;
                    const int64_t r = r0 + int64_t(k) * gridDim.x;
                    const int64_t b = r / p.zf_rows, rr = p.zf_row0 + r % p.zf_rows;
                    uint4* row = reinterpret_cast<uint4*>(p.o_dst[0] + (b * p.o_bstride + rr) * int64_t(p.o_H) * D);
#pragma unroll 4
                    for (int w = lane; w < words; w += 32) __stcs(row + w, z);
                }
            }
        }
      } else if (warp == 9 || warp == 11) {
        // ------------------------------------------------ MMA issuers
        // Two independent issuers so that neither waits behind the other:
        //   warp 9   S_i(j) = Q_i K_j^T into the shared S buffer, i = 0, 1, gated
        //            by K_j landing and s_free (previous S loaded by a softmax WG);
        //   warp 11  O_i += P_i(j) V_j, gated by V_j landing and p_full_i.
        // They touch disjoint TMEM (S vs P_i / O_i) and each commits only its
        // own MMAs (tcgen05.commit tracks the issuing thread's operations).
        // A tcgen05.mma issue blocks while the tensor pipe's queue is full, so a
        // single issuer held every S behind the PV issued before it.
        // The whole warp runs its loop; one elected lane issues each group.
        const uint64_t dq = make_sdesc_sw128(smem_u32(sQ), 16, 1024);
        const uint64_t dk = make_sdesc_sw128(smem_u32(sKV), 16, 1024);
        const uint64_t dv = make_sdesc_sw128(smem_u32(sKV), kHalfBytes, 1024);
        constexpr uint32_t kTile16 = kTileBytes >> 4;      // descriptor address units
        uint32_t kv_it = 0, g = 0, n_item = 0, s_count = 0;
        int tn = 0;
        Item it;
        Cursor cu;
        for (; next_item(p, cu, it); ++n_item) {
            const int nkv = it.hi - it.lo;
            if (warp == 9) {
                for (int j = 0; j < nkv; ++j) {
                    // ring position of K_j (producer's order K0, K1, V0, K2, V1, ...)
                    const uint32_t ik = kv_it + (j == 0 ? 0 : 2 * j - 1), sk = ik % kStages;
                    mbar_wait(&kv_full[sk], (ik / kStages) & 1);
                    if (lane == 0) trace_ev(p, 1, tn, 10);
                    for (int i = 0; i < 2; ++i) {
                        if (s_count > 0) mbar_wait(s_free, (s_count - 1) & 1);
                        if (j == 0) mbar_wait(&q_full[i], n_item & 1);
                        if (lane == 0) trace_ev(p, 1, tn, 15 + i);
                        tc_fence_after();
                        static_assert(kHalfBytes >> 4 == 1024, "S k-step offsets in mma_ss_group");
                        mma_ss_group<D / 16>(tmem + kColS, dq + i * kTile16, dk + sk * kTile16, kIdescS);
                        mma_commit_w(&s_full[i]);
                        ++s_count;
                        if (lane == 0) trace_ev(p, 1, tn, 13 + i);
                        if (j == nkv - 1) mma_commit_w(&q_empty[i]);
                    }
                    mma_commit_w(&kv_empty[sk]);   // K_j free once S_0(j), S_1(j) complete
                }
            } else {
                for (int j = 0; j < nkv; ++j) {
                    const uint32_t iv = kv_it + (j == nkv - 1 ? 2 * nkv - 1 : 2 * j + 2), sv = iv % kStages;
                    mbar_wait(&kv_full[sv], (iv / kStages) & 1);
                    for (int i = 0; i < 2; ++i) {
                        mbar_wait(&p_full[i], (g + j) & 1);
                        if (j == 0 && n_item > 0) mbar_wait(&o_empty[i], (n_item - 1) & 1);
                        if (lane == 0) trace_ev(p, 3, tn, 11 + i);
                        tc_fence_after();
                        static_assert(kBN == 128 && kHalfBytes == 16384, "PV k-step offsets in mma_ts_group8");
                        mma_ts_group8(tmem + kColO + i * D, tmem + kColP + i * 64, dv + sv * kTile16,
                                      kIdescO, j > 0 ? 1u : 0u);
                        mma_commit_w(&o_done[i]);
                        if (j == nkv - 1) mma_commit_w(&o_final[i]);
                    }
                    mma_commit_w(&kv_empty[sv]);   // V_j free once PV_0(j), PV_1(j) complete
                }
            }
            kv_it += 2 * nkv;
            g += nkv;
        }
      }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsSoftmax));
        // ------------------------------------------------ softmax + epilogue (warps 0-7)
        const int i = warp >> 2, wq = warp & 3;
        const int row_in_pair = i * kBM + wq * 32 + lane;       // 0..255
        const uint32_t lane_off = uint32_t(wq * 32) << 16;
        const uint32_t tS = tmem + lane_off + kColS;
        const uint32_t tPi = tmem + lane_off + kColP + i * 64;
        const uint32_t tOi = tmem + lane_off + kColO + i * D;
        const float sl2 = p.scale_log2;
        uint32_t g = 0, n_item = 0;
        int tn = 0;
        const bool tr = (lane == 0);   // every softmax warp records (equal trace overhead)
        Item it;
        Cursor cu;
        for (; next_item(p, cu, it); ++n_item) {
#if !defined(TM_SPANS_MERGE) && !defined(TM_SPANS_MERGE2)
            if (threadIdx.x == 0 && n_item == 1) trace_span(p, 2);   // first item's epilogue done
#endif
            float m_run = -INFINITY, l = 0.f;
            for (int j = it.lo; j < it.hi; ++j, ++g) {
                int seg, row, valid;
                tile_info<kMulti>(p, it.pr, j, seg, row, valid);
                uint32_t r[kBN];
                mbar_wait(&s_full[i], g & 1);
                if (tr) trace_ev(p, 5 + warp, tn, 20);
#if !defined(TM_SPANS_MERGE) && !defined(TM_SPANS_MERGE2)
                if (threadIdx.x == 0 && g == 0) trace_span(p, 1);
#endif
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < kBN; c += 32) tmem_ld32(tS + c, r + c);
                tmem_wait_ld();
                tc_fence_before();
                mbar_arrive(s_free);          // the S buffer may be refilled
                if (tr) trace_ev(p, 5 + warp, tn, 21);
                if (valid < kBN) {
#pragma unroll
                    for (int c = 0; c < kBN; ++c)
                        if (c >= valid) r[c] = 0xff800000u;   // -inf: key beyond the segment
                }
                // The previous PV_i reads P_i: it must be complete before P_i is
                // overwritten.  Waited on only once this tile's exps are done (P is
                // held packed in registers meanwhile), so a late PV never stalls
                // the exponentials.
                bool pv_waited = (g == 0);
                auto wait_prev_pv = [&]() {
                    if (!pv_waited) {
                        mbar_wait(&o_done[i], (g - 1) & 1);
                        tc_fence_after();
                        pv_waited = true;
                    }
                };
                auto row_max = [&]() -> float {   // 3-input max tree (depth 5), ALU pipe
                    float t1[43];
#pragma unroll
                    for (int k = 0; k < 42; ++k)
                        t1[k] = max3(__uint_as_float(r[3 * k]), __uint_as_float(r[3 * k + 1]),
                                     __uint_as_float(r[3 * k + 2]));
                    t1[42] = fmaxf(__uint_as_float(r[126]), __uint_as_float(r[127]));
                    float t2[15];
#pragma unroll
                    for (int k = 0; k < 14; ++k) t2[k] = max3(t1[3 * k], t1[3 * k + 1], t1[3 * k + 2]);
                    t2[14] = t1[42];
                    float t3[5];
#pragma unroll
                    for (int k = 0; k < 5; ++k) t3[k] = max3(t2[3 * k], t2[3 * k + 1], t2[3 * k + 2]);
                    return max3(max3(t3[0], t3[1], t3[2]), t3[3], t3[4]);
                };
                // Running max with a lazy threshold: m_run (log2 units) moves only
                // when this tile's exact max exceeds it by more than kLazyLog2, so
                // every weight is <= 2^kLazyLog2 and nothing is ever recomputed.
                // O_i and l are rescaled by 2^(m_old - m_new) when it moves (exact
                // after the final O / l either way).
                const float mt = row_max() * sl2;
                const bool grow = mt > m_run + kLazyLog2;      // always on an item's first tile
                if (__any_sync(0xffffffffu, grow)) {
                    const float m_new = grow ? mt : m_run;
                    const float alpha = grow ? ex2(m_run - m_new) : 1.f;   // 0 on the first tile
                    m_run = m_new;
                    l *= alpha;
                    if (j != it.lo) {   // O_i holds PV_i(it.lo .. j-1): complete first
                        wait_prev_pv();
#pragma unroll
                        for (int c = 0; c < D; c += 16) {
                            uint32_t o[16];
                            tmem_ld16(tOi + c, o);
                            tmem_wait_ld();
#pragma unroll
                            for (int e = 0; e < 16; ++e)
                                o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
                            tmem_st16(tOi + c, o);
                        }
                    }
                }
                if (tr) trace_ev(p, 5 + warp, tn, 22);
                // p = 2^(s * scale * log2 e - m_run), kPolyMask pairs of every 16 on
                // the FMA-pipe polynomial; row sum in fp32, P rounded to bf16 (RNE).
                uint32_t pk[kBN / 2];
                float tsum;
                {
                    const float nm = (m_run == -INFINITY) ? 0.f : -m_run;
                    const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(nm, nm);
                    float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                                     make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
                    for (int e = 0; e < kBN / 2; ++e) {
                        const float2 x = ffma2(make_float2(__uint_as_float(r[2 * e]),
                                                           __uint_as_float(r[2 * e + 1])),
                                               sc2, nm2);
                        float2 pe;
                        if ((kPolyMask >> (e & 15)) & 1) {
                            pe = exp2_poly2(x);
                        } else {
                            pe.x = ex2(x.x);
                            pe.y = ex2(x.y);
                        }
                        acc[e & 3] = fadd2(acc[e & 3], pe);
                        pk[e] = pack_bf16x2(pe.x, pe.y);
                    }
                    const float2 s01 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
                    tsum = s01.x + s01.y;
                }
                wait_prev_pv();
                if (tr) trace_ev(p, 5 + warp, tn, 25);
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_st16(tPi + c * 16, pk + c * 16);
                l += tsum;
                if (tr) trace_ev(p, 5 + warp, tn, 23);
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(&p_full[i]);
                if (tr) trace_ev(p, 5 + warp, tn, 24);
            }
            // ------------------------------------------------ epilogue
            mbar_wait(&o_final[i], n_item & 1);
            tc_fence_after();
#ifdef TM_SPANS_MERGE
            if (threadIdx.x == 0) trace_span(p, 2);   // (spans A/B) this item's epilogue begins
#endif
            const int q = it.qp * 2 * kBM + row_in_pair;
            // Split units (stream-K pieces).  Each softmax warpgroup
            // (Q tile i of the unit) is its own merge participant: tile i's
            // merger keeps O_i in TMEM, waits until the unit's other pieces have
            // published their tile-i partials, merges them in piece order and
            // stores the rows; every other piece publishes its tile-i partial.
            // Tile 0 is merged by piece 0 (its CTA's last item).  With >= 3
            // pieces, piece 1 spans its CTA's whole range, so it also ends with
            // the launch: it merges tile 1 (ROW-SPLIT CO-MERGE), and piece 0
            // publishes its tile-1 partial instead.  Each leg of the chain that
            // follows the last tile -- partial write, partial reads, output store
            // -- then moves 32 KB through one SM instead of 64-128 KB.
            const bool co = it.piece && it.npieces >= 3;
            const int merger_piece = (i == 1 && co) ? 1 : 0;
            if (!it.piece || p.dbg_nomerge) {   // (dbg_nomerge: timing bound only, wrong output)
                store_rows_bf16<D, kKind>(p, p.prob[it.pr], tOi, 1.f / l, sEpi + warp * 4096, it.b, q - lane,
                                   it.h, lane);
#ifdef TM_SPANS_MERGE
                if (threadIdx.x == 0) trace_span(p, 5);
#endif
                tc_fence_before();
                mbar_arrive(&o_empty[i]);
            } else if (it.pidx != merger_piece) {
                // Publish this piece's tile-i partial: the unnormalised O row
                // scaled by 2^s into fp16 (s per row, a power of two so the
                // scaling is exact: the row's largest |O| lands in [2^14, 2^15),
                // relative rounding <= 2^-11 of it), the running max m (log2
                // units), l and m - s (the exponent of the O weight); then count
                // it in for the tile's merger.  A first item (piece >= 1) uses its
                // CTA's first-item slot; piece 0 (co-merge) the last-item slot.
#ifdef TM_SPANS_PUB
                if (threadIdx.x == 0) trace_span(p, 4);   // (spans A/B) partner's tiles done
#endif
                float* tp = part_tile<D>(p, it.blk, it.cl, it.pidx == 0 ? 2 : i);
                uint4* po = reinterpret_cast<uint4*>(tp);
                const int r = wq * 32 + lane;             // row within the tile
                uint32_t o[D];
#pragma unroll
                for (int c = 0; c < D; c += 32) tmem_ld32(tOi + c, o + c);
                tmem_wait_ld();
                tc_fence_before();
                mbar_arrive(&o_empty[i]);     // O_i read out: the next item's PV may write it
                float amax = 0.f;
#pragma unroll
                for (int c = 0; c < D; ++c) amax = fmaxf(amax, fabsf(__uint_as_float(o[c])));
                int sx = 141 - int((__float_as_uint(amax) >> 23) & 0xffu);
                sx = sx < -100 ? -100 : (sx > 100 ? 100 : sx);
                const float sc = __uint_as_float(uint32_t(127 + sx) << 23);   // 2^s exactly
#pragma unroll
                for (int c = 0; c < D; c += 8) {
                    uint4 v;
                    v.x = pack_f16x2(__uint_as_float(o[c]) * sc, __uint_as_float(o[c + 1]) * sc);
                    v.y = pack_f16x2(__uint_as_float(o[c + 2]) * sc, __uint_as_float(o[c + 3]) * sc);
                    v.z = pack_f16x2(__uint_as_float(o[c + 4]) * sc, __uint_as_float(o[c + 5]) * sc);
                    v.w = pack_f16x2(__uint_as_float(o[c + 6]) * sc, __uint_as_float(o[c + 7]) * sc);
                    po[(c >> 3) * kBM + r] = v;
                }
                tp[kTileO + r] = m_run;
                tp[kTileO + kBM + r] = l;
                tp[kTileO + 2 * kBM + r] = m_run - float(sx);
                wg_bar(i);                    // the warpgroup's partial stores precede ...
                if (wq == 0 && lane == 0) {   // ... this one release (cumulative over the barrier)
                    const int mp = (i == 1 && co) ? 1 : 0;          // the tile's merger piece
                    const int n = it.pidx < mp ? it.pidx : it.pidx - 1;   // contributor index
                    red_release_or(&p.counters[(it.blk * kMaxPersistentCtas + it.cfirst) * 2 + i], 1ull << n);
#ifdef TM_SPANS_PUB
                    trace_span(p, 6);                 // (spans A/B) partial published
#endif
                }
            } else {
                // Tile i's merger (its CTA's last item of the block), O_i in TMEM:
                // wait for the other np - 1 pieces' tile-i partials, merge them
                // in piece order (deterministic, no float atomics) and store.
                if (threadIdx.x == 0) trace_span(p, 4);
                const int np = it.npieces;
                const int nc = np - 1;            // contributors (<= 64: cached_class caps pieces)
                const int r = wq * 32 + lane;
                // contributor n (0 .. np-2) in piece order, skipping the merger
                auto contrib = [&](int n) -> const float* {
                    const int k = n < merger_piece ? n : n + 1;
                    return k == 0 ? part_tile<D>(p, it.blk, it.cfirst, 2)     // piece 0's last-item slot
                                  : part_tile<D>(p, it.blk, it.cfirst + k, i);
                };
                // If this is the CTA's last item overall (no more Q or K/V loads),
                // the contributors' O rows (32 KB each) are pulled by bulk copies
                // into three buffers of this warpgroup -- its Q tile and two ring
                // slots -- three in flight, each issued as soon as its
                // contributor's bit is in (early pieces copy while the late one
                // finishes); each thread reads its row from shared memory
                // ([d/8][128] uint4: conflict-free).  The ring is reused once both
                // tiles' last MMAs are complete (o_final of the other tile too) and
                // no append store reads it (store_idle).  Otherwise (a later
                // schedule block follows, its loads already in flight) each thread
                // loads its row from L2 directly.  Both apply the same per-element
                // update in the same piece order (merge_elem): the same bits.
                constexpr uint32_t kRowsBytes = kBM * D * 2;
                static_assert(kRowsBytes == kTileBytes && kStages >= 4, "merge buffers: Q tile + 2 ring slots");
                Cursor cpeek = cu;
                Item nx;
                const bool smem_merge = !next_item(p, cpeek, nx);
                auto buf = [&](int j) -> uint8_t* {
                    return j == 0 ? sQ + i * kTileBytes : sKV + (2 * i + j - 1) * kTileBytes;
                };
                auto issue = [&](int n) {
                    uint64_t* bar = &merge_bar[3 * i + n % 3];
                    mbar_arrive_expect_tx(bar, kRowsBytes);
                    fence_proxy_async_global();        // generic-proxy writes -> bulk-copy reads
                    bulk_g2s(buf(n % 3), contrib(n), kRowsBytes, bar);
                };
                if (wq == 0 && lane == 0) {
                    unsigned long long* vc = p.counters + (it.blk * kMaxPersistentCtas + it.cfirst) * 2 + i;
                    const unsigned long long all = nc >= 64 ? ~0ull : (1ull << nc) - 1;
                    const int pre = nc < 3 ? nc : 3;             // copies issued while waiting
                    unsigned long long issued = 0;
                    if (smem_merge) {
                        mbar_wait(&o_final[i ^ 1], n_item & 1);   // the other tile's MMAs are done too
                        mbar_wait(store_idle, 0);
                        tc_fence_after();
                    }
                    const long long t0 = clock64();
                    for (;;) {
                        const unsigned long long m = ld_acquire_u64(vc);
                        if (smem_merge) {
                            const unsigned long long nw = m & ~issued & ((1ull << pre) - 1);
                            if (nw) {
                                for (int n = 0; n < pre; ++n)
                                    if ((nw >> n) & 1) issue(n);
                                issued |= nw;
                            }
                        }
                        if (m == all) break;
                        if (clock64() - t0 > (1ll << 33)) __trap();
                    }
                    *vc = 0;                                // ready for the next launch
                }
                wg_bar(i);                    // thread 0's acquire covers the warpgroup's reads
                if (threadIdx.x == 0) trace_span(p, 5);
                float mm[8], ll[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const bool in = e < nc;
                    mm[e] = in ? __ldcg(contrib(e) + kTileO + r) : -INFINITY;
                    ll[e] = in ? __ldcg(contrib(e) + kTileO + kBM + r) : 0.f;
                }
                float mstar = m_run;
#pragma unroll
                for (int e = 0; e < 8; ++e) mstar = fmaxf(mstar, mm[e]);
                for (int k0 = 8; k0 < nc; k0 += 8) {        // more than 9 pieces (long units)
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        if (k0 + e < nc) mstar = fmaxf(mstar, __ldcg(contrib(k0 + e) + kTileO + r));
                }
                const float w0 = ex2(m_run - mstar);
                float wsum = w0 * l;
#pragma unroll
                for (int e = 0; e < 8; ++e) wsum += ex2(mm[e] - mstar) * ll[e];
                for (int k0 = 8; k0 < nc; k0 += 8) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const bool in = k0 + e < nc;
                        const float m2 = in ? __ldcg(contrib(k0 + e) + kTileO + r) : -INFINITY;
                        const float l2 = in ? __ldcg(contrib(k0 + e) + kTileO + kBM + r) : 0.f;
                        wsum += ex2(m2 - mstar) * l2;
                    }
                }
                const float inv = 1.f / wsum;
#ifdef TM_SPANS_MERGE2
                if (threadIdx.x == 0) trace_span(p, 1);      // (spans A/B) weights ready
#endif
                // O <- O * wo + wk * x per contributor; wk = 2^(m_k - s_k - m*)
                // (its fp16 rows carry 2^s_k); wo = w0 once, then 1.
                float mo_nxt = __ldcg(contrib(0) + kTileO + 2 * kBM + r);
                for (int n = 0; n < nc; ++n) {
                    const float wk = ex2(mo_nxt - mstar);
                    if (n + 1 < nc) mo_nxt = __ldcg(contrib(n + 1) + kTileO + 2 * kBM + r);
                    const float wo = n == 0 ? w0 : 1.f;
                    uint4 x[D / 8];
                    if (smem_merge) {
                        mbar_wait(&merge_bar[3 * i + n % 3], (n / 3) & 1);
#ifdef TM_SPANS_PUB
                        if (threadIdx.x == 0 && n == nc - 1) trace_span(p, 6);   // (spans A/B) last buffer landed
#endif
                        const uint4* sp = reinterpret_cast<const uint4*>(buf(n % 3));
#pragma unroll
                        for (int c = 0; c < D / 8; ++c) x[c] = sp[c * kBM + r];
                        if (n + 3 < nc) {
                            wg_bar(i);              // the warpgroup is done with this buffer
                            if (wq == 0 && lane == 0) issue(n + 3);
                        }
                    } else {
                        const uint4* gp = reinterpret_cast<const uint4*>(contrib(n));
#pragma unroll
                        for (int c = 0; c < D / 8; ++c) x[c] = __ldcg(gp + c * kBM + r);
                    }
#pragma unroll
                    for (int c = 0; c < D; c += 32) {
                        uint32_t o[32];
                        tmem_ld32(tOi + c, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const uint4 v = x[(c >> 3) + e];
                            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                            for (int t = 0; t < 4; ++t) {
                                const float2 f = unpack_f16x2(w[t]);
                                o[8 * e + 2 * t] = merge_elem(o[8 * e + 2 * t], wo, wk, f.x);
                                o[8 * e + 2 * t + 1] = merge_elem(o[8 * e + 2 * t + 1], wo, wk, f.y);
                            }
                        }
                        tmem_st32(tOi + c, o);
                    }
                }
                tmem_wait_st();
#ifdef TM_SPANS_MERGE2
                if (threadIdx.x == 0) trace_span(p, 2);      // (spans A/B) partials merged
#endif
                store_rows_bf16<D, kKind>(p, p.prob[it.pr], tOi, inv, sEpi + warp * 4096, it.b, q - lane, it.h,
                                   lane);
                tc_fence_before();
                mbar_arrive(&o_empty[i]);
            }
        }
        // The epilogue's TMA stores must have READ their staging buffers before
        // the CTA's shared memory goes away; their global writes complete with
        // the grid (what a dependent launch waits for).  exit_wait_full (A/B,
        // TM_EXIT_WAIT_FULL=1) waits for the writes themselves.
        if (lane == 0) {
            if (p.exit_wait_full) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
#ifdef TM_SPANS_MERGE
        if (threadIdx.x == 0) trace_span(p, 4);   // (spans A/B) softmax loop left, before the final barrier
#endif
        if (threadIdx.x == 0) {
#ifndef TM_SPANS_PUB
            trace_span(p, 6, g);
#endif
            uint32_t smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            trace_span(p, 7, n_item | (long long)smid << 16);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) trace_span(p, 3);
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
    // a6 fused: this rank's O rows are in the owners' windows once every CTA
    // is here; the last CTA bumps done[rank] at each owner.
    if (kPeerKind && p.signal_done) peer_signal(p.done_ctr, p.own, p.P, p.rank, 3, p.wait_done);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

// Token-major bf16 [B][L][H][d]: dims (inner first) {d, H, L, B}; box {64, 1, 128, 1}.
// `bstride` = tokens between batch elements (>= L; a sub-range of a longer sequence).
bool make_map(CUtensorMap* m, const void* base, int d, int H, int64_t L, int B, int64_t bstride = 0,
              int box_rows = 128) {
    if (bstride <= 0) bstride = L;
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[4] = {cuuint64_t(d), cuuint64_t(H), cuuint64_t(L), cuuint64_t(B)};
    cuuint64_t strides[3] = {cuuint64_t(d) * 2, cuuint64_t(H) * d * 2, cuuint64_t(bstride) * H * d * 2};
    cuuint32_t box[4] = {64, 1, cuuint32_t(box_rows), 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int D>
constexpr int smem_bytes() {
    return 1024 + (2 + kStages) * kBN * D * 2 + kEpiBytes + 512;
}

int sm_count() { return current_sm_count(); }

template <int D, uint32_t kPolyMask, int kKind>
cudaError_t launch_t(const FmhaParams& p, int grid, cudaStream_t stream) {
    // The max-dynamic-shared-memory attribute is per device: set once per
    // device ordinal (bit per device; ordinals >= 64 set it on every launch).
    static unsigned long long attr_set = 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    const unsigned long long bit = dev < 64 ? 1ull << dev : 0;
    if (!bit || !(__atomic_load_n(&attr_set, __ATOMIC_RELAXED) & bit)) {
        cudaError_t e = cudaFuncSetAttribute(fmha_sm100_kernel<D, kPolyMask, kKind>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             smem_bytes<D>());
        if (e != cudaSuccess) return e;
        __atomic_fetch_or(&attr_set, bit, __ATOMIC_RELAXED);
    }
    return launch_pdl(fmha_sm100_kernel<D, kPolyMask, kKind>, dim3(grid), dim3(kThreads), smem_bytes<D>(),
                      stream, p);
}

// Which of every 16 exp2 pairs run as the FMA-pipe polynomial (bit e set) --
// the MUFU/FMA balance.  At d = 128 the MUFU exp rate (16/clk/SM) equals the
// tensor rate in score elements, so some offload gives the softmax slack; more
// polynomial costs FMA/ALU issue and energy (the kernel is power-capped when
// sustained).  Measured (random data, independent S/PV issuers, exact tile max):
// 2/16 vs all-MUFU 1382 vs 1363 TFLOP/s burst, 1172 vs 1156 sustained;
// 3/16 = 2/16, 4/16 and more slower (profiles/README.md).  With the fused
// c_t append all-MUFU measured ~1 % better (328.3 vs 332.0 us) and zero-copy
// calls prefer 2/16 (317.8 vs 324.0; profiles/r1_poly_append_sweep.txt), but
// one split for every launch keeps the append, zero-copy, window and Ulysses
// paths bitwise identical (S:303 window == streaming).  With the v19 kernel
// (pipelined merge, L2 prefetch) all-MUFU beat 2/16 on the fused-append
// workload (bench step 1368-1369 vs 1358-1363, streaming 30.15 vs 30.53
// ms/chunk) but lost 1.7 % on the zero-copy kernel alone
// (profiles/r1_v20_poly_ab.txt); 1/16 then beat all-MUFU on every measure
// (step +0.4 %, zero-copy alone +0.9 %, streaming +0.3 %;
// profiles/r1_v21_poly_ab.txt), so the default is 1/16.
// TM_POLY selects a split for tuning: 1 = all MUFU, 2 = 2/16, 3 = 3/16,
// 4 = 4/16, 5 = 1/16 (the default, also when TM_POLY is unset).
constexpr uint32_t kPoly2of16 = 0x0808u;     // pairs {3, 11} of every 16 (TM_POLY=2)
template <int D, int kKind>
cudaError_t launch_d(const FmhaParams& p, int grid, cudaStream_t stream) {
    static int env_sel = [] {
        const char* e = getenv("TM_POLY");
        return e ? atoi(e) : 0;
    }();
    const int sel = env_sel ? env_sel : 5;
    switch (sel) {
        case 1: return launch_t<D, 0x0000u, kKind>(p, grid, stream);   // all MUFU
        case 3: return launch_t<D, 0x1084u, kKind>(p, grid, stream);   // {2,7,12}
        case 5: return launch_t<D, 0x0800u, kKind>(p, grid, stream);   // {11}: 1/16
        case 4: return launch_t<D, 0x4444u, kKind>(p, grid, stream);   // {2,6,10,14}
        default: return launch_t<D, kPoly2of16, kKind>(p, grid, stream);
    }
}

}  // namespace

// Host: cut the tail's W tiles -- runs of units, run r holding units[r]
// units of tiles[r] KV tiles each, flattened in order -- into at most C
// contiguous ranges whose cost -- tiles plus kItemCost per item after a
// range's first -- is as equal as possible (a CTA that switches to another
// unit pays its epilogue / partial write, the next Q load and pipeline
// refill, and as the unit's merger the partial reads: ~6 tiles' time
// measured, profiles/r1_v8_cta_spans.txt).  A greedy fill under budget B, the
// smallest B (bisection) that needs <= C ranges.  Pieces shorter than
// kMinPiece are not started at a range's end.  TM_SCHED_SPLIT=1 (A/B only):
// plain equal ranges.  Returns G'.
int tail_bounds_runs(int nruns, const int* units, const int* tiles, int C, int min_piece, int* bound) {
    static const float item_cost = [] {
        const char* e = getenv("TM_SCHED_ITEM_COST");
        return e ? float(atof(e)) : 3.f;
    }();
    // A range whose LAST item is a partner piece (it starts inside its unit)
    // ends with the partial write the unit's merger waits for: charged
    // write_cost tiles, so the partial is in L2 when the merger is done.
    static const float write_cost = [] {
        const char* e = getenv("TM_SCHED_WRITE_COST");
        return e ? float(atof(e)) : 0.f;
    }();
    static const bool split_sched = [] {
        const char* e = getenv("TM_SCHED_SPLIT");
        return e && *e && strcmp(e, "0") != 0;
    }();
    std::vector<long long> run0(nruns + 1, 0);
    long long T = 0;
    for (int r = 0; r < nruns; ++r) {
        run0[r + 1] = run0[r] + (long long)units[r] * tiles[r];
        T += units[r];
    }
    const int W = int(run0[nruns]);
    // end of the unit holding tile x
    auto unit_end = [&](int x) -> int {
        int r = 0;
        while (r + 1 < nruns && run0[r + 1] <= x) ++r;
        const long long off = x - run0[r];
        return int(run0[r] + (off / tiles[r] + 1) * tiles[r]);
    };
    int G = C;
    if (G > W / min_piece) G = W / min_piece;
    if (G < T) G = int(T < C ? T : C);
    if (G > C) G = C;
    if (G < 1) G = 1;
    if (split_sched || item_cost <= 0.f) {
        for (int c = 0; c <= G; ++c) bound[c] = int((long long)c * W / G);
        return G;
    }
    // At most G ranges: never more than W / min_piece (short problems would
    // otherwise be cut into 1-tile pieces whose merges cost more than the work).
    auto fill = [&](float B, int* out) -> int {   // ranges used, or G+1 if more are needed
        int x = 0, g = 0;
        if (out) out[0] = 0;
        while (x < W) {
            if (g == G) return G + 1;
            const int start = x;
            float cost = 0.f;
            while (x < W) {
                const int ue = unit_end(x);
                const float extra = x > start ? item_cost : 0.f;
                const bool partner = x > 0 && unit_end(x - 1) == ue;   // starts inside its unit
                const float avail = B - cost - extra - (partner ? write_cost : 0.f);
                int take = int(avail);
                if (take > ue - x) take = ue - x;
                if (x > start && take < min_piece && take < ue - x) break;
                if (take <= 0) {
                    if (x == start) take = 1;    // always progress
                    else break;
                }
                cost += take + extra;
                x += take;
                if (x < ue) break;               // budget ends inside this unit
            }
            ++g;
            if (out) out[g] = x;
        }
        return g;
    };
    int maxn = 1;
    for (int r = 0; r < nruns; ++r) maxn = tiles[r] > maxn ? tiles[r] : maxn;
    float lo = float(W) / G, hi = float(W) / G + item_cost * 4 + maxn;
    while (fill(hi, nullptr) > G) hi *= 2;
    for (int it = 0; it < 40; ++it) {
        const float mid = 0.5f * (lo + hi);
        if (fill(mid, nullptr) <= G) hi = mid;
        else lo = mid;
    }
    return fill(hi, bound);
}

int tail_bounds(int T, int n, int C, int min_piece, int* bound) {
    return tail_bounds_runs(1, &T, &n, C, min_piece, bound);
}

// The schedule the kernel runs: tail_bounds from kMinPiece, the minimum piece
// raised (in proportion to the excess) until no unit is cut into more than
// kMaxUnitPieces pieces (a split unit's merger tracks its contributors in a
// 64-bit mask).
int tail_bounds_capped(int T, int n, int C, int* bound) {
    constexpr int kMinPiece = 4;
    int g = 0;
    for (int min_piece = kMinPiece;;) {
        g = tail_bounds(T, n, C, min_piece, bound);
        int worst = 1;
        for (int u = 0; u < T; ++u) {
            const int first = int(std::upper_bound(bound, bound + g + 1, u * n) - bound) - 1;
            const int last = int(std::upper_bound(bound, bound + g + 1, u * n + n - 1) - bound) - 1;
            worst = std::max(worst, last - first + 1);
        }
        if (worst <= kMaxUnitPieces || min_piece >= n) break;
        min_piece = std::max(min_piece + 1, (min_piece * worst + kMaxUnitPieces - 1) / kMaxUnitPieces);
    }
    return g;
}

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("TM_PDL");
        return !(e && strcmp(e, "0") == 0);
    }();
    return on;
}

size_t fmha_sm100_scratch_bytes(int d) {
    return size_t(kMaxBlocks) * kMaxPersistentCtas * (256 * size_t(d) + 512) * 4 +
           size_t(kMaxBlocks) * kMaxPersistentCtas * 2 * 8;
}

namespace {

// KV segments of one problem: tile starts, lengths, rows and maps.
void set_segments(Prob& P, int nseg, const int64_t* len, const int64_t* row0, const int* map) {
    int tiles = 0;
    P.nseg = nseg;
    for (int s = 0; s < nseg; ++s) {
        P.seg_tile_start[s] = tiles;
        P.seg_len[s] = int(len[s]);
        P.seg_row0[s] = int(row0[s]);
        P.seg_map[s] = map[s];
        tiles += int((len[s] + kBN - 1) / kBN);
    }
    P.seg_tile_start[nseg] = tiles;
    P.n_tiles = tiles;
}

int grid_ctas(int max_ctas) {
    int C = sm_count() < kMaxPersistentCtas ? sm_count() : kMaxPersistentCtas;
    if (max_ctas > 0 && max_ctas < C) C = max_ctas;
    return C;
}

// The stream-K bounds of T tail units of n tiles over C CTAs, cached per
// (T, n, C): a shape's schedule is computed once.
bool cached_class(int T, int n, int C, SkClass& k) {
    if ((long long)T * n >= (1ll << 30)) return false;
    static std::mutex mu;
    static std::map<std::tuple<int, int, int>, std::vector<int>> cache;
    std::lock_guard<std::mutex> lock(mu);
    std::vector<int>& b = cache[std::make_tuple(T, n, C)];
    if (b.empty()) {
        b.assign(kMaxPersistentCtas + 1, 0);
        b.resize(tail_bounds_capped(T, n, C, b.data()) + 1);
    }
    const int G = int(b.size()) - 1;
    if (G <= 0) return false;
    for (int c = 0; c <= G; ++c) k.bound[c] = b[c];
    k.ctas = G;
    return true;
}

// Appends block (problem pr, heads [h0, h0 + nh)) to the launch's schedule:
// R whole rounds, then the tail's stream-K class (shared by the blocks of the
// same tail shape).  *full: the launch has no room left (the caller launches
// what it has and continues); false otherwise means an invalid shape.
bool add_block(FmhaParams& p, int pr, int h0, int nh, int C, bool* full) {
    *full = false;
    const Prob& P = p.prob[pr];
    const int U = p.B * nh * P.n_qpairs;
    const int R = U / C, T = U - R * C;
    int cls = -1;
    if (T > 0) {
        for (int i = 0; i < p.ncls; ++i)
            if (p.cls_key[i][0] == T && p.cls_key[i][1] == P.n_tiles) cls = i;
        if (cls < 0) {
            if (p.ncls == kMaxSkClasses) {
                *full = true;
                return false;
            }
            if (!cached_class(T, P.n_tiles, C, p.cls[p.ncls])) return false;
            p.cls_key[p.ncls][0] = T;
            p.cls_key[p.ncls][1] = P.n_tiles;
            cls = p.ncls++;
        }
    }
    if (p.nblk == kMaxBlocks) {
        *full = true;
        return false;
    }
    Block& b = p.blk[p.nblk];
    b.pr = pr;
    b.h0 = h0;
    b.nh = nh;
    b.rounds = R;
    b.cls = cls;
    b.tail0 = R * C;
    b.off = 0;
    if (p.nblk > 0) {
        const Block& a = p.blk[p.nblk - 1];
        b.off = (a.off + (a.cls >= 0 ? p.cls[a.cls].ctas : 0)) % C;
    }
    ++p.nblk;
    return true;
}

// Grid: C when a block has whole rounds or several blocks are rotated over
// the CTAs, else the single block's tail width.
int launch_grid(const FmhaParams& p) {
    if (p.nblk > 1) return p.ctas;
    if (p.nblk == 0) return 0;
    if (p.blk[0].rounds > 0) return p.ctas;
    return p.blk[0].cls >= 0 ? p.cls[p.blk[0].cls].ctas : 0;
}

bool exit_wait_full() {
    static const bool on = [] {
        const char* e = getenv("TM_EXIT_WAIT_FULL");
        return e && *e && strcmp(e, "0") != 0;
    }();
    return on;
}

cudaError_t finish_and_launch(FmhaParams& p, int d, int grid, void* scratch, cudaStream_t stream,
                              int* launches, unsigned long long* trace, bool peer, int kind) {
    static const int l2_prefetch_env = [] {
        const char* e = getenv("TM_L2_PREFETCH");
        return e ? atoi(e) : 2;
    }();
    // (no L2 prefetch for peer windows, filled during the launch, nor for the
    // packed f4 launches, whose operands a prep kernel just wrote: their first
    // real loads would queue behind the prefetches)
    p.l2_prefetch = (peer || p.prob[0].packed_R) ? 0 : l2_prefetch_env;
    p.exit_wait_full = exit_wait_full();
    static const bool nomerge = [] {
        const char* e = getenv("TM_DBG_NOMERGE");
        return e && *e && strcmp(e, "0") != 0;
    }();
    p.dbg_nomerge = nomerge;
    static const bool nolatestore = [] {
        const char* e = getenv("TM_DBG_NOLATESTORE");
        return e && *e && strcmp(e, "0") != 0;
    }();
    p.dbg_nolatestore = nolatestore;
    p.trace = trace;
    p.part = static_cast<float*>(scratch);
    p.counters = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(scratch) +
                                        size_t(kMaxBlocks) * kMaxPersistentCtas *
                                            (256 * size_t(d) + 512) * 4);
    if (grid <= 0) return cudaErrorInvalidValue;
    cudaError_t e;
    switch (kind) {
        case 1: e = d == 128 ? launch_d<128, 1>(p, grid, stream) : launch_d<64, 1>(p, grid, stream); break;
        case 2: e = d == 128 ? launch_d<128, 2>(p, grid, stream) : launch_d<64, 2>(p, grid, stream); break;
        default: e = d == 128 ? launch_d<128, 0>(p, grid, stream) : launch_d<64, 0>(p, grid, stream);
    }
    if (e == cudaSuccess && launches) ++*launches;
    return e;
}

bool tma_epi_enabled() {
    static const bool on = [] {
        const char* e = getenv("TM_TMA_EPI");
        return !(e && strcmp(e, "0") == 0);
    }();
    return on;
}

}  // namespace

cudaError_t launch_fmha_sm100(const AttnProblem& pr, void* scratch, cudaStream_t stream,
                              int* launches, unsigned long long* trace) {
    if (pr.d != 64 && pr.d != 128) return cudaErrorInvalidValue;
    if (pr.nseg < 1 || pr.nseg > kMaxSegments) return cudaErrorInvalidValue;
    FmhaParams p;
    memset(&p, 0, sizeof(p));
    if (!make_map(&p.tq, pr.q, pr.d, pr.H, pr.Lq, pr.B, pr.q_bstride)) return cudaErrorInvalidValue;
    int64_t len[kMaxSegments], row0[kMaxSegments];
    int map[kMaxSegments];
    for (int s = 0; s < pr.nseg; ++s) {
        if (!make_map(&p.tk[s], pr.seg[s].k, pr.d, pr.H, pr.seg[s].len, pr.B, pr.seg[s].bstride) ||
            !make_map(&p.tv[s], pr.seg[s].v, pr.d, pr.H, pr.seg[s].len, pr.B, pr.seg[s].bstride))
            return cudaErrorInvalidValue;
        len[s] = pr.seg[s].len;
        row0[s] = 0;
        map[s] = s;
    }
    p.nmaps = pr.nseg;
    p.nprob = 1;
    Prob& P = p.prob[0];
    set_segments(P, pr.nseg, len, row0, map);
    const int tiles = P.n_tiles;
    p.store_seg = -1;
    if (pr.store_k && pr.store_v) {
        const Segment& cur = pr.seg[pr.nseg - 1];
        if (!make_map(&p.tk_store, pr.store_k, pr.d, pr.H, cur.len, pr.B) ||
            !make_map(&p.tv_store, pr.store_v, pr.d, pr.H, cur.len, pr.B))
            return cudaErrorInvalidValue;
        p.store_seg = pr.nseg - 1;
    }
    P.Lq = int(pr.Lq);
    P.q_row0 = 0;
    P.o_row0 = 0;
    P.o_clip = 1;
    p.H = pr.H;
    p.B = pr.B;
    p.scale_log2 = pr.scale * 1.4426950408889634f;
    p.o_dst[0] = static_cast<uint16_t*>(pr.o);
    p.o_bstride = pr.q_bstride > 0 ? pr.q_bstride : pr.Lq;
    p.tma_epi = 0;
    if (tma_epi_enabled() && !pr.peer && make_map(&p.to, pr.o, pr.d, pr.H, pr.Lq, pr.B, p.o_bstride, 32))
        p.tma_epi = 1;
    p.o_rows = int(pr.Lq);
    p.o_H = pr.H;
    p.o_h0 = 0;
    p.wait_seg = -1;
    if (const PeerAttnArgs* pa = pr.peer) {
        if (pa->P < 1 || pa->P > kMaxPeers) return cudaErrorInvalidValue;
        for (int r = 0; r < pa->P; ++r) p.o_dst[r] = static_cast<uint16_t*>(pa->o_dst[r]);
        p.o_rows = int(pa->o_rows);
        p.o_bstride = pa->o_rows;
        p.o_H = pa->o_H;
        p.o_h0 = pa->o_h0;
        p.peer = pa->own != nullptr && pa->wait_seg >= 0;
        p.wait_seg = pa->wait_seg;
        p.src_rows = int(pa->src_rows);
        for (int t = 0; t < 3; ++t) p.epoch[t] = pa->epoch[t];
        p.own = pa->own;
        p.push = pa->push;
        p.pp = pa->pp;
        p.signal_done = pa->signal_done;
        p.wait_done = pa->wait_done;
        for (int r = 0; r < pa->P; ++r) p.done_ctr[r] = pa->done_ctr[r];
        p.P = pa->P;
        p.rank = pa->rank;
        if (p.peer && p.src_rows <= 0) return cudaErrorInvalidValue;
        if (p.push && int64_t(p.pp.B) * p.pp.Ls * p.pp.P * p.pp.W >= (int64_t(1) << 31))
            return cudaErrorInvalidValue;
    }
    const int qtiles = int((pr.Lq + kBM - 1) / kBM);
    P.n_qpairs = (qtiles + 1) / 2;
    // Persistent schedule: R whole rounds over C CTAs, then the T tail units'
    // T*n KV tiles in contiguous ranges over G' CTAs (stream-K).  P = 2, 4, 8
    // head shards leave T >= C/2 (240, 120, 60 units of 56 tiles at WAN-512),
    // where whole-unit or even-split tails idle ~19% of the machine.
    // Schedule blocks of sched_heads heads (0: all heads in one block).
    const int C = grid_ctas(pr.max_ctas);
    p.ctas = C;
    const int hb = pr.sched_heads > 0 ? pr.sched_heads : pr.H;
    if (pr.H % hb) return cudaErrorInvalidValue;
    for (int h0 = 0; h0 < pr.H; h0 += hb) {
        bool full = false;
        if (!add_block(p, 0, h0, hb, C, &full)) return cudaErrorInvalidValue;
    }
    (void)tiles;
    return finish_and_launch(p, pr.d, launch_grid(p), scratch, stream, launches, trace,
                             pr.peer != nullptr, pr.peer != nullptr ? 2 : 0);
}

// The kMulti kernel variant only for launches that use its code (packed keys,
// the f4 zero fill); the f1 window's problems run on the chunk-attention kernel
// (the extra code measured 1-3 % slower where it is compiled in but unused).
int multi_kind(const FmhaParams& p) {
    bool packed = false;
    for (int i = 0; i < p.nprob; ++i) packed |= p.prob[i].packed_R != 0;
    return (packed || p.zf_inv != nullptr) ? 1 : 0;
}

cudaError_t launch_fmha_sm100_multi(const MultiProblem& mp, void* scratch, cudaStream_t stream,
                                    int* launches, unsigned long long* trace) {
    if (mp.d != 64 && mp.d != 128) return cudaErrorInvalidValue;
    if (mp.nprob < 1 || mp.nprob > kMaxProblems) return cudaErrorInvalidValue;
    FmhaParams p;
    memset(&p, 0, sizeof(p));
    if (!make_map(&p.tq, mp.q, mp.d, mp.H, mp.q_rows, mp.B, mp.q_bstride) ||
        !make_map(&p.tk[0], mp.k, mp.d, mp.H, mp.kv_rows, mp.B, mp.kv_bstride) ||
        !make_map(&p.tv[0], mp.v, mp.d, mp.H, mp.kv_rows, mp.B, mp.kv_bstride))
        return cudaErrorInvalidValue;
    p.nmaps = 1;
    p.nprob = mp.nprob;
    p.store_seg = -1;
    p.H = mp.H;
    p.B = mp.B;
    p.scale_log2 = mp.scale * 1.4426950408889634f;
    p.o_dst[0] = static_cast<uint16_t*>(mp.o);
    p.o_bstride = mp.o_bstride > 0 ? mp.o_bstride : mp.o_rows;
    p.o_row_map = mp.o_row_map;
    p.zf_inv = mp.zero_inv;
    p.zf_T = int(mp.zero_T);
    p.zf_row0 = mp.zero_row0;
    p.zf_rows = mp.zero_rows;
    if (p.zf_inv && (p.zf_T <= 0 || p.zf_rows <= 0)) return cudaErrorInvalidValue;
    p.tma_epi = 0;
    if (tma_epi_enabled() && !mp.o_row_map &&
        make_map(&p.to, mp.o, mp.d, mp.H, mp.o_rows, mp.B, p.o_bstride, 32))
        p.tma_epi = 1;
    p.o_rows = int(1 << 30);          // one owner: every row of O is local
    p.o_H = mp.H;
    p.o_h0 = 0;
    p.wait_seg = -1;
    for (int i = 0; i < mp.nprob; ++i) {
        const SubProblem& sp = mp.prob[i];
        if (sp.nseg < 1 || sp.nseg > kMaxSegments || sp.Lq <= 0) return cudaErrorInvalidValue;
        Prob& P = p.prob[i];
        int map[kMaxSegments] = {};
        set_segments(P, sp.nseg, sp.seg_len, sp.seg_row0, map);
        P.q_row0 = int(sp.q_row0);
        P.Lq = int(sp.Lq);
        P.o_row0 = int(sp.o_row0);
        P.o_clip = !mp.o_row_map && sp.o_row0 + sp.Lq == mp.o_rows;
        P.n_qpairs = int((sp.Lq + 2 * kBM - 1) / (2 * kBM));
    }
    // Packed keys (MultiProblem::pack_keys): the largest box height R in {32,
    // 16, 8} dividing every segment length (R >= 8 keeps every box at a
    // 1024-B-aligned offset of the tile, where the 128-B swizzle repeats).
    int R = 0;
    if (mp.pack_keys) {
        R = 32;
        for (int i = 0; i < mp.nprob; ++i)
            for (int sg = 0; sg < mp.prob[i].nseg; ++sg)
                while (R >= 8 && mp.prob[i].seg_len[sg] % R) R /= 2;
        if (R < 8) R = 0;
    }
    if (R) {
        if (!make_map(&p.tk_sub, mp.k, mp.d, mp.H, mp.kv_rows, mp.B, mp.kv_bstride, R) ||
            !make_map(&p.tv_sub, mp.v, mp.d, mp.H, mp.kv_rows, mp.B, mp.kv_bstride, R))
            return cudaErrorInvalidValue;
        for (int i = 0; i < mp.nprob; ++i) {
            Prob& P = p.prob[i];
            const SubProblem& sp = mp.prob[i];
            int64_t k0 = 0;
            for (int sg = 0; sg < sp.nseg; ++sg) {
                P.seg_key0[sg] = int(k0);
                k0 += sp.seg_len[sg];
            }
            P.packed_R = R;
            P.Lk = int(k0);
            P.n_tiles = int((k0 + kBN - 1) / kBN);
        }
    }
    // Blocks: every problem x head group, in order.  A launch holds up to
    // kMaxBlocks blocks of up to kMaxSkClasses tail shapes, so a long list
    // runs as several launches (each block is scheduled as if alone anyway).
    const int C = grid_ctas(mp.max_ctas);
    p.ctas = C;
    const int hb = mp.sched_heads > 0 ? mp.sched_heads : mp.H;
    if (mp.H % hb) return cudaErrorInvalidValue;
    for (int i = 0; i < mp.nprob; ++i) {
        for (int h0 = 0; h0 < mp.H; h0 += hb) {
            bool full = false;
            if (add_block(p, i, h0, hb, C, &full)) continue;
            if (!full) return cudaErrorInvalidValue;
            cudaError_t e = finish_and_launch(p, mp.d, launch_grid(p), scratch, stream, launches,
                                              trace, false, multi_kind(p));
            if (e != cudaSuccess) return e;
            p.zf_inv = nullptr;               // the first launch zero-filled
            p.nblk = 0;
            p.ncls = 0;
            if (!add_block(p, i, h0, hb, C, &full)) return cudaErrorInvalidValue;
        }
    }
    return finish_and_launch(p, mp.d, launch_grid(p), scratch, stream, launches, trace, false, multi_kind(p));
}

}  // namespace tmk
