// peer_map.h -- index maps of the peer-memory Ulysses transport (rows a2, a6;
// DeepSpeed-Ulysses sequence parallelism), shared by the
// device code (peer.cuh push, fmha_sm100.cu epilogue) and the host routine
// tm_peer_route_host (api.cpp) that the world-size-2 gloo tests run on CPU.
//
// Rank r holds the sequence shard of global tokens [r*Ls, r*Ls + Ls) (padded
// to Ls; tokens >= L are padding) and owns heads [r*Hl, r*Hl + Hl).
//   push:  word i of a shard [B][Ls][H][d] (W 16-B words per (token, head
//          block)) goes to rank p's window [B][Lw][Hl][d], row r*Ls + t
//   out:   output row q of head h (window head h of rank r) goes to rank
//          q / Ls's O window [B][Ls][H][d], row q % Ls, head r*Hl + h
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define TM_PHD __host__ __device__ __forceinline__
#else
#define TM_PHD inline
#endif

namespace tmk {

// Push: for word i of rank `rank`'s shard, the destination rank and word offset
// in its window (false: padding token, not sent).
TM_PHD bool peer_push_route(uint32_t i, uint32_t W, uint32_t P, uint32_t Ls, int64_t L,
                            int64_t Lw, int rank, uint32_t& p, int64_t& dst) {
    const uint32_t PW = P * W;
    const uint32_t row = i / PW, k = i - row * PW;
    p = k / W;
    const uint32_t w = k - p * W;
    const uint32_t b = row / Ls, t = row - b * Ls;
    const int64_t g = int64_t(rank) * Ls + t;
    if (g >= L) return false;
    dst = (int64_t(b) * Lw + g) * W + w;
    return true;
}

// Output: owner rank and (d-element) row offset in the owner's O buffer of
// output row q, batch b, local head h.  o_bstride: rows between batches
// (o_rows for the O window; a longer sequence for sub-range problems).
TM_PHD int64_t peer_out_route(int64_t b, int64_t q, int h, int64_t o_rows, int64_t o_bstride,
                             int o_H, int o_h0, int& owner) {
    owner = int(q / o_rows);
    const int64_t r = q - int64_t(owner) * o_rows;
    return (b * o_bstride + r) * o_H + o_h0 + h;
}

}  // namespace tmk
