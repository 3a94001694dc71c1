// ulysses_map.h -- the index map of the Ulysses sequence <-> head exchange
// (DeepSpeed-Ulysses), shared by the device pack/unpack kernel
// (elementwise.cu) and the host routine tm_ulysses_shuffle_host (api.cpp) so
// that the world-size-2 gloo tests exercise the same layout code on CPU.
//
// Rows are d*esize bytes moved as W 16-byte words.  Rank r holds the sequence
// shard of global tokens [r*Ls, r*Ls + Ls) (padded to Ls; tokens >= L are
// padding) and, after the exchange, heads [r*Hl, r*Hl + Hl).
//   mode 0  pack_seq_to_peers:     src [B][Ls][H][d]      -> dst [P][B][Ls][Hl][d]
//   mode 1  unpack_peers_to_heads: src [P][B][Ls][Hl][d]  -> dst [B][L][Hl][d]   (tokens < L)
//   mode 2  pack_heads_to_peers:   src [B][L][Hl][d]      -> dst [P][B][Ls][Hl][d] (pad rows 0)
//   mode 3  unpack_peers_to_seq:   src [P][B][Ls][Hl][d]  -> dst [B][Ls][H][d]
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define TM_HD __host__ __device__ __forceinline__
#else
#define TM_HD inline
#endif

namespace tmk {

struct UlyssesShape {
    int B, P, Hl, W;    // batch, ranks, heads per rank, 16-B words per row
    int64_t Ls, L;      // shard tokens (padded), global tokens
};

// Total words of the peer-block index space [P][B][Ls][Hl][W].
TM_HD int64_t ulysses_words(const UlyssesShape& s) {
    return int64_t(s.P) * s.B * s.Ls * s.Hl * s.W;
}

// For word `idx` of the peer-block space: source / destination word offsets
// (-1 = skip the move, -2 = write zero).
TM_HD void ulysses_map(const UlyssesShape& s, int mode, int64_t idx, int64_t& src, int64_t& dst) {
    int64_t r = idx;
    const int w = int(r % s.W); r /= s.W;
    const int hl = int(r % s.Hl); r /= s.Hl;
    const int64_t t = r % s.Ls; r /= s.Ls;
    const int b = int(r % s.B); r /= s.B;
    const int p = int(r);
    const int H = s.Hl * s.P;
    const int64_t blk = idx;                                                    // [P][B][Ls][Hl]
    const int64_t seq = ((int64_t(b) * s.Ls + t) * H + p * s.Hl + hl) * s.W + w;  // [B][Ls][H]
    const int64_t g = p * s.Ls + t;                                             // global token
    const int64_t head = ((int64_t(b) * s.L + g) * s.Hl + hl) * s.W + w;        // [B][L][Hl]
    switch (mode) {
        case 0: src = seq; dst = blk; break;
        case 1: src = blk; dst = g < s.L ? head : -1; break;
        case 2: src = g < s.L ? head : -2; dst = blk; break;
        default: src = blk; dst = seq; break;
    }
}

}  // namespace tmk
