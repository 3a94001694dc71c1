// internal.h -- host-side declarations shared by the C-ABI (api.cpp) and the
// kernel launchers.  Not part of the public ABI (include/tm.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tmk {

constexpr int kMaxSegments = 5;   // {c_0, c_{t-1}, c_t}; f4 audio windows need up to 5
constexpr int kMaxPersistentCtas = 160;   // persistent grid cap (B200: 148 SMs)

// One contiguous K/V segment in token-major layout [B][len][H][d].
struct Segment {
    const void* k = nullptr;
    const void* v = nullptr;
    int64_t len = 0;               // tokens (0 = absent)
    int64_t bstride = 0;           // tokens between batch elements (0: = len)
};

// a4: the segment schedule of one chunk-attention call.
struct AttnProblem {
    const void* q = nullptr;       // [B][Lq][H][d]
    void* o = nullptr;             // [B][Lq][H][d]
    int64_t Lq = 0;
    int64_t q_bstride = 0;         // tokens between batch elements of q / o (0: = Lq)
    int B = 1, H = 1, d = 128;     // H = heads resident on this rank
    int nseg = 0;
    Segment seg[kMaxSegments];
    float scale = 0.f;             // softmax scale (1/sqrt(d), Eq 7)
    // a3 fused append (sm100 path): if set, the last segment's K/V tiles are also
    // written to these [B][len][H][d] buffers (the cache slot) by the kernel.
    void* store_k = nullptr;
    void* store_v = nullptr;
};

// Launchers; return cudaSuccess or the launch error.  `launches` is
// incremented by the number of kernels enqueued.
// `scratch` (fmha_sm100_scratch_bytes(d) bytes, zero-initialised once) holds
// the split-KV partials and merge counters; counters return to zero.
size_t fmha_sm100_scratch_bytes(int d);
// `trace` (debug, may be null): 4 x 4096 uint64 clock64 timeline of CTA 0.
cudaError_t launch_fmha_sm100(const AttnProblem& p, void* scratch, cudaStream_t s, int* launches,
                              unsigned long long* trace = nullptr);
cudaError_t launch_fmha_fp32(const AttnProblem& p, cudaStream_t s, int* launches);
cudaError_t launch_euler(float* x, const void* v, int v_is_bf16, int64_t n, float dt,
                         cudaStream_t s, int* launches);
// f2: few-step sampler entry (see elementwise.cu); eps == nullptr -> Philox noise.
cudaError_t launch_sampler(float* x, const void* v, int v_is_bf16, const float* eps, int64_t n,
                           float t_cur, float t_next, uint64_t seed, uint64_t offset,
                           void* x_bf16, cudaStream_t s, int* launches);
// f4: gather (scatter = 0) / scatter (1) of face-token rows, ids device int32.
cudaError_t launch_face_rows(const void* src, void* dst, const int32_t* ids, int64_t BF, int64_t T,
                            int64_t nf, int row_bytes, int scatter, cudaStream_t s, int* launches);
// Non-finite check: sets *flag (device int) to 1 if any element is NaN/Inf.
cudaError_t launch_nonfinite(const void* x, int is_bf16, int64_t n, int* flag, cudaStream_t s,
                             int* launches);

// Ulysses pack / unpack.  Token-major [B][L][H][d] <-> per-peer
// blocks; see ulysses.cu for the exact layouts.
cudaError_t launch_pack_seq_to_peers(const void* src, void* dst, int B, int64_t Ls, int H, int P,
                                     int d, int esize, cudaStream_t s, int* launches);
cudaError_t launch_unpack_peers_to_heads(const void* src, void* dst, int B, int64_t Ls,
                                         int64_t L, int Hl, int P, int d, int esize,
                                         cudaStream_t s, int* launches);
cudaError_t launch_pack_heads_to_peers(const void* src, void* dst, int B, int64_t Ls, int64_t L,
                                       int Hl, int P, int d, int esize, cudaStream_t s,
                                       int* launches);
cudaError_t launch_unpack_peers_to_seq(const void* src, void* dst, int B, int64_t Ls, int H,
                                       int P, int d, int esize, cudaStream_t s, int* launches);

}  // namespace tmk
