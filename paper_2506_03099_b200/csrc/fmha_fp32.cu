// fmha_fp32.cu -- fp32 validation-mode chunk attention (row a5, TM_FP32).
//
// Same segment schedule as the tcgen05 kernel (a4: only {c_0, c_{t-1}, c_t},
// P:151), fp32 throughout (no tf32: single-pass tf32 misses the 1e-4 bar,
// SURVEY.md Sec 4.4), accurate expf.  SIMT design: a CTA owns one head and
// 16 query rows (4 warps x 4 rows); 32-key K/V tiles are staged in shared
// memory; lane j computes the logit of key j, and the online softmax's row
// max / row sum are warp-shuffle reductions; for P.V each lane owns d/32
// output dims and key j's probability is broadcast with __shfl_sync.
// The logit q.k is a compensated (Ogita-Rump-Oishi "Dot2") fp32 dot product:
// with |logits| ~ 1e3 (distribution D6) a plain fp32 FMA chain loses ~6e-4
// of the softmax weights' relative accuracy, which would miss the 1e-4 bar.
#include <cuda_runtime.h>

#include <cmath>

#include "internal.h"

namespace tmk {
namespace {

constexpr int kWarps = 4;
constexpr int kRowsPerWarp = 4;
constexpr int kRows = kWarps * kRowsPerWarp;
constexpr int kKeys = 32;

struct Fp32Params {
    const float* q;
    float* o;
    const float* k[kMaxSegments];
    const float* v[kMaxSegments];
    int64_t len[kMaxSegments];
    int64_t bstride[kMaxSegments];   // tokens between batch elements of each segment
    int nseg;
    int64_t Lq;
    int64_t q_bstride;                // tokens between batch elements of q / o
    int H;
    float scale;
};

__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

template <int D>
__global__ void __launch_bounds__(kWarps * 32) fmha_fp32_kernel(const Fp32Params p) {
    constexpr int DP = D + 1;            // padded K row: lane j reads row j conflict-free
    constexpr int PER = D / 32;          // output dims per lane
    __shared__ float sq[kRows][D];
    __shared__ float sk[kKeys][DP];
    __shared__ float sv[kKeys][D];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int h = blockIdx.y, b = blockIdx.z;
    const int64_t r0 = int64_t(blockIdx.x) * kRows;
    const int H = p.H;

    for (int idx = threadIdx.x; idx < kRows * D; idx += blockDim.x) {
        const int rr = idx / D, c = idx % D;
        const int64_t q = r0 + rr;
        sq[rr][c] = q < p.Lq ? p.q[((int64_t(b) * p.q_bstride + q) * H + h) * D + c] : 0.f;
    }

    float m[kRowsPerWarp], l[kRowsPerWarp], acc[kRowsPerWarp][PER];
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) {
        m[r] = -INFINITY;
        l[r] = 0.f;
#pragma unroll
        for (int e = 0; e < PER; ++e) acc[r][e] = 0.f;
    }

    for (int s = 0; s < p.nseg; ++s) {
        const int64_t len = p.len[s];
        const int64_t bst = p.bstride[s];
        const float* K = p.k[s];
        const float* V = p.v[s];
        for (int64_t j0 = 0; j0 < len; j0 += kKeys) {
            __syncthreads();
            for (int idx = threadIdx.x; idx < kKeys * D; idx += blockDim.x) {
                const int jj = idx / D, c = idx % D;
                const int64_t j = j0 + jj;
                const bool ok = j < len;
                const int64_t g = ((int64_t(b) * bst + j) * H + h) * D + c;
                sk[jj][c] = ok ? K[g] : 0.f;
                sv[jj][c] = ok ? V[g] : 0.f;
            }
            __syncthreads();
            const bool key_ok = j0 + lane < len;
#pragma unroll
            for (int r = 0; r < kRowsPerWarp; ++r) {
                const int rr = warp * kRowsPerWarp + r;
                // Dot2: s + c carries the dot product to ~twice fp32 precision.
                float sum = 0.f, comp = 0.f;
#pragma unroll 16
                for (int c = 0; c < D; ++c) {
                    const float a = sq[rr][c], bk = sk[lane][c];
                    // _rn intrinsics: never contracted into FMAs, so the
                    // error-free transformations stay exact.
                    const float pr = __fmul_rn(a, bk);
                    const float pe = fmaf(a, bk, -pr);                  // TwoProduct error
                    const float t = __fadd_rn(sum, pr);                 // TwoSum
                    const float z = __fsub_rn(t, sum);
                    comp = __fadd_rn(comp, __fadd_rn(__fadd_rn(__fsub_rn(sum, __fsub_rn(t, z)),
                                                               __fsub_rn(pr, z)), pe));
                    sum = t;
                }
                // logit = hi + lo (unevaluated pair); the running max uses hi
                // and exp() sees (hi - m) + lo, so |logit| ~ 1e3 keeps ~1e-7
                // relative accuracy in the weights.
                const float hi = key_ok ? __fmul_rn(sum, p.scale) : -INFINITY;
                const float lo = key_ok ? fmaf(sum, p.scale, -hi) + comp * p.scale : 0.f;
                const float m_new = fmaxf(m[r], warp_max(hi));
                const float alpha = expf(m[r] - m_new);     // m = -inf at start -> 0
                const float pj = expf(__fadd_rn(__fsub_rn(hi, m_new), lo));
                l[r] = l[r] * alpha + warp_sum(pj);
                m[r] = m_new;
#pragma unroll
                for (int e = 0; e < PER; ++e) acc[r][e] *= alpha;
#pragma unroll 8
                for (int jj = 0; jj < kKeys; ++jj) {
                    const float pb = __shfl_sync(0xffffffffu, pj, jj);
#pragma unroll
                    for (int e = 0; e < PER; ++e) acc[r][e] = fmaf(pb, sv[jj][lane + 32 * e], acc[r][e]);
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) {
        const int64_t q = r0 + warp * kRowsPerWarp + r;
        if (q >= p.Lq) continue;
        const float inv = 1.f / l[r];
        float* dst = p.o + ((int64_t(b) * p.q_bstride + q) * H + h) * D;
#pragma unroll
        for (int e = 0; e < PER; ++e) dst[lane + 32 * e] = acc[r][e] * inv;
    }
}

}  // namespace

cudaError_t launch_fmha_fp32(const AttnProblem& pr, cudaStream_t stream, int* launches) {
    Fp32Params p{};
    p.q = static_cast<const float*>(pr.q);
    p.o = static_cast<float*>(pr.o);
    p.nseg = pr.nseg;
    for (int s = 0; s < pr.nseg; ++s) {
        p.k[s] = static_cast<const float*>(pr.seg[s].k);
        p.v[s] = static_cast<const float*>(pr.seg[s].v);
        p.len[s] = pr.seg[s].len;
        p.bstride[s] = pr.seg[s].bstride > 0 ? pr.seg[s].bstride : pr.seg[s].len;
    }
    p.Lq = pr.Lq;
    p.q_bstride = pr.q_bstride > 0 ? pr.q_bstride : pr.Lq;
    p.H = pr.H;
    p.scale = pr.scale;
    dim3 grid(unsigned((pr.Lq + kRows - 1) / kRows), pr.H, pr.B);
    if (pr.d == 128)
        fmha_fp32_kernel<128><<<grid, kWarps * 32, 0, stream>>>(p);
    else if (pr.d == 64)
        fmha_fp32_kernel<64><<<grid, kWarps * 32, 0, stream>>>(p);
    else
        return cudaErrorInvalidValue;
    if (launches) ++*launches;
    return cudaGetLastError();
}

}  // namespace tmk
