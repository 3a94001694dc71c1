// elementwise.cu -- HBM-bound kernels of the path:
//   a7  flow-matching Euler step x <- x + dt*v (Eqs 1-2),
//       one fp32 FMA per element (single rounding), 16-byte vector loads,
//       grid sized in multiples of the SM count;
//   a2/a6 Ulysses pack / unpack between sequence shards and head shards
//       (DeepSpeed-Ulysses), 16-byte vector moves;
//   debug finiteness check (TM_DEBUG).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"
#include "ulysses_map.h"

namespace tmk {
namespace {

int num_sms() { return current_sm_count(); }

cudaError_t finish(cudaError_t e, int* launches) {
    if (e == cudaSuccess && launches) ++*launches;
    return e;
}

unsigned grid_for(int64_t work_items, int threads, int per_sm = 8) {
    const int64_t want = (work_items + threads - 1) / threads;
    const int64_t cap = int64_t(num_sms()) * per_sm;
    return unsigned(want < cap ? (want > 0 ? want : 1) : cap);
}

// ------------------------------------------------------------------ Euler
// x: fp32 [n] (16-B aligned), v: fp32 or bf16 [n].  Each thread handles 8
// consecutive elements per iteration (2 x float4 of x, 8 v values).
template <bool kBf16>
__global__ void __launch_bounds__(256) euler_kernel(float* __restrict__ x,
                                                    const void* __restrict__ vv, int64_t n,
                                                    float dt) {
    asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: after the previous grid
    const int64_t n8 = n / 8;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n8; i += stride) {
        float4 a = reinterpret_cast<const float4*>(x)[2 * i];
        float4 c = reinterpret_cast<const float4*>(x)[2 * i + 1];
        float v[8];
        if constexpr (kBf16) {
            const uint4 w = reinterpret_cast<const uint4*>(vv)[i];
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                v[2 * e] = __uint_as_float(ws[e] << 16);
                v[2 * e + 1] = __uint_as_float(ws[e] & 0xffff0000u);
            }
        } else {
            const float4 b0 = reinterpret_cast<const float4*>(vv)[2 * i];
            const float4 b1 = reinterpret_cast<const float4*>(vv)[2 * i + 1];
            v[0] = b0.x; v[1] = b0.y; v[2] = b0.z; v[3] = b0.w;
            v[4] = b1.x; v[5] = b1.y; v[6] = b1.z; v[7] = b1.w;
        }
        a.x = __fmaf_rn(dt, v[0], a.x); a.y = __fmaf_rn(dt, v[1], a.y);
        a.z = __fmaf_rn(dt, v[2], a.z); a.w = __fmaf_rn(dt, v[3], a.w);
        c.x = __fmaf_rn(dt, v[4], c.x); c.y = __fmaf_rn(dt, v[5], c.y);
        c.z = __fmaf_rn(dt, v[6], c.z); c.w = __fmaf_rn(dt, v[7], c.w);
        reinterpret_cast<float4*>(x)[2 * i] = a;
        reinterpret_cast<float4*>(x)[2 * i + 1] = c;
    }
    // ragged tail (< 8 elements), handled by the first threads of block 0
    if (blockIdx.x == 0) {
        const int64_t t = n8 * 8 + threadIdx.x;
        if (t < n) {
            float v;
            if constexpr (kBf16)
                v = __uint_as_float(uint32_t(static_cast<const uint16_t*>(vv)[t]) << 16);
            else
                v = static_cast<const float*>(vv)[t];
            x[t] = __fmaf_rn(dt, v, x[t]);
        }
    }
}

// ------------------------------------------------------------------ f2 sampler step
// Philox4x32-10 (Salmon et al., SC'11): counter-based, so element i's noise is
// a pure function of (seed, offset, i) -- deterministic and order-free.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        // one 32x32 -> 64-bit multiply (IMAD.WIDE.U32) gives both halves
        const uint64_t p0 = uint64_t(0xD2511F53u) * c.x, p1 = uint64_t(0xCD9E8D57u) * c.z;
        const uint32_t hi0 = uint32_t(p0 >> 32), lo0 = uint32_t(p0);
        const uint32_t hi1 = uint32_t(p1 >> 32), lo1 = uint32_t(p1);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

// t = -2 ln u for u = (w + 0.5) 2^-32 with relative accuracy ~2^-21 over the
// whole range, in ~12 instructions instead of the accurate logf's ~25: MUFU
// lg2 where u <= 15/16 (|ln u| >= 0.065, so its 2^-22 relative error stays
// relative); near 1 the series -ln(1 - d) = d + d^2/2 + ... + d^6/6 with
// d = 1 - u taken from the integer ~w = 2^32 - 1 - w (no cancellation;
// truncation < 1e-8 relative for d < 1/16).  Also finite where u itself
// rounds to 1 in fp32 (d = 2^-33 for w = 2^32 - 1).
__device__ __forceinline__ float neg2_log_u(uint32_t w, float u) {
    constexpr float k32 = 2.3283064365386963e-10f;      // 2^-32
    float lg;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(u));
    const float d = fmaf(float(~w), k32, 0.5f * k32);
    float sr = fmaf(d, 1.f / 6.f, 0.2f);
    sr = fmaf(d, sr, 0.25f);
    sr = fmaf(d, sr, 1.f / 3.f);
    sr = fmaf(d, sr, 0.5f);
    sr = fmaf(d, sr, 1.f);
    return d < 0.0625f ? 2.f * d * sr : -1.3862943611198906f * lg;
}

// S:224 one schedule entry of the few-step student, fused with the
// noise draw and the bf16 cast of the next NFE's input:
//   x1_hat = x + (1 - t_cur) v ;  x <- t_next x1_hat + (1 - t_next) eps  (Eq 1)
// or x <- x1_hat for the final entry (t_next >= 1).  eps: caller's fp32 buffer
// (kEps) or N(0,1) from Philox(counter = (i/4, offset), key = seed) with the
// Box-Muller pairs (w0,w1), (w2,w3).  Each thread handles 4 elements.
template <bool kBf16V, bool kEps>
__global__ void __launch_bounds__(256) sampler_kernel(float* __restrict__ x,
                                                      const void* __restrict__ vv,
                                                      const float* __restrict__ eps, int64_t n,
                                                      float t_cur, float t_next, uint2 seed,
                                                      uint2 offset, uint16_t* __restrict__ xb) {
    const int64_t groups = (n + 3) / 4;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const bool final_step = t_next >= 1.f;
    const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(vv) |
                           reinterpret_cast<uintptr_t>(xb)) & 15) == 0;
    for (int64_t gi = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; gi < groups; gi += stride) {
        // Vector-path operands are loaded first so their latency overlaps the
        // Philox / Box-Muller arithmetic below.
        const bool vec = 4 * gi + 4 <= n && aligned;
        float4 xv = make_float4(0.f, 0.f, 0.f, 0.f);
        float vf[4] = {0.f, 0.f, 0.f, 0.f};
        if (vec) {
            xv = reinterpret_cast<const float4*>(x)[gi];
            if constexpr (kBf16V) {
                const uint2 w = reinterpret_cast<const uint2*>(vv)[gi];
                vf[0] = __uint_as_float(w.x << 16); vf[1] = __uint_as_float(w.x & 0xffff0000u);
                vf[2] = __uint_as_float(w.y << 16); vf[3] = __uint_as_float(w.y & 0xffff0000u);
            } else {
                const float4 w = reinterpret_cast<const float4*>(vv)[gi];
                vf[0] = w.x; vf[1] = w.y; vf[2] = w.z; vf[3] = w.w;
            }
        }
        float e[4] = {0.f, 0.f, 0.f, 0.f};
        if (!final_step) {
            if constexpr (kEps) {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (4 * gi + j < n) e[j] = eps[4 * gi + j];
            } else {
                const uint4 w = philox4x32_10(
                    make_uint4(uint32_t(gi), uint32_t(uint64_t(gi) >> 32), offset.x, offset.y), seed);
                const float k32 = 2.3283064365386963e-10f;      // 2^-32
                const float u0 = fmaf(float(w.x), k32, 0.5f * k32), u1 = fmaf(float(w.y), k32, 0.5f * k32);
                const float u2 = fmaf(float(w.z), k32, 0.5f * k32), u3 = fmaf(float(w.w), k32, 0.5f * k32);
                // r = sqrt(-2 ln u) as t * rsqrt(t) (MUFU, rel. error ~2^-23); t from
                // neg2_log_u (relative accuracy everywhere, also where u rounds
                // to 1 in fp32: an absolute log error would be amplified by 1/r
                // there).  The clamp keeps 0 * rsqrt(0) from being NaN.
                // The angle 2 pi u is taken as pi (2u - 1) + pi, inside MUFU
                // sin/cos's accurate range [-pi, pi] (abs. error ~2^-21), so
                // sin and cos flip sign.
                const float t0 = neg2_log_u(w.x, u0), t2 = neg2_log_u(w.z, u2);
                const float r0 = t0 * rsqrtf(fmaxf(t0, 1e-30f)), r1 = t2 * rsqrtf(fmaxf(t2, 1e-30f));
                const float a1 = 3.14159265358979f * fmaf(2.f, u1, -1.f);
                const float a3 = 3.14159265358979f * fmaf(2.f, u3, -1.f);
                float s0, c0, s1, c1;
                __sincosf(a1, &s0, &c0);
                __sincosf(a3, &s1, &c1);
                e[0] = -r0 * c0; e[1] = -r0 * s0; e[2] = -r1 * c1; e[3] = -r1 * s1;
            }
        }
        const int64_t i0 = 4 * gi;
        if (vec) {                               // vector path: 16 B x, 8 / 16 B v, 8 B bf16 out
            const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
            float xn[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float x1 = __fmaf_rn(1.f - t_cur, vf[j], xs[j]);
                xn[j] = final_step ? x1 : __fmaf_rn(t_next, x1, (1.f - t_next) * e[j]);
            }
            reinterpret_cast<float4*>(x)[gi] = make_float4(xn[0], xn[1], xn[2], xn[3]);
            if (xb) {
                const uint32_t lo = uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(xn[0]))) |
                                    (uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(xn[1]))) << 16);
                const uint32_t hi = uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(xn[2]))) |
                                    (uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(xn[3]))) << 16);
                reinterpret_cast<uint2*>(xb)[gi] = make_uint2(lo, hi);
            }
            continue;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t i = 4 * gi + j;
            if (i >= n) break;
            const float vi = kBf16V ? __uint_as_float(uint32_t(static_cast<const uint16_t*>(vv)[i]) << 16)
                                    : static_cast<const float*>(vv)[i];
            const float x1 = __fmaf_rn(1.f - t_cur, vi, x[i]);
            const float xn = final_step ? x1 : __fmaf_rn(t_next, x1, (1.f - t_next) * e[j]);
            x[i] = xn;
            if (xb) xb[i] = __bfloat16_as_ushort(__float2bfloat16_rn(xn));
        }
    }
}

// ------------------------------------------------------------------ f4 face-row gather / scatter
// Rows of W 16-byte words.  gather: dst[bf][i] = src[bf][ids[i]]  (bf = b * frames + f)
//                           scatter: dst[bf][ids[i]] = src[bf][i]
template <bool kScatter>
__global__ void __launch_bounds__(256) face_rows_kernel(const uint4* __restrict__ src,
                                                        uint4* __restrict__ dst,
                                                        const int32_t* __restrict__ ids,
                                                        int64_t BF, int64_t T, int64_t nf, int W) {
    const int64_t total = BF * nf * W;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
        const int w = int(idx % W);
        const int64_t r = idx / W;
        const int64_t i = r % nf, bf = r / nf;
        const int64_t full = (bf * T + ids[i]) * W + w;
        const int64_t comp = (bf * nf + i) * W + w;
        if (kScatter) dst[full] = src[comp];
        else dst[comp] = src[full];
    }
}

// f4 preparation: the face rows of q are gathered, qf[bf][i] = q[bf][ids[i]]
// (one warp per face row, rows of W 16-byte words), and CTA 0 writes the
// inverse map inv[t] = a face slot of token t, or -1 (ids outside [0, T) are
// ignored).  The attention launch then writes the face rows of o through ids
// and zeroes the non-face rows (inv[t] < 0: no audio update)
// with its spare warp while it attends.  Launched with PDL.
__global__ void __launch_bounds__(128) audio_prep_kernel(const uint4* __restrict__ q,
                                                         uint4* __restrict__ qf,
                                                         int32_t* __restrict__ inv_out,
                                                         const int32_t* __restrict__ ids,
                                                         int64_t BF, int T, int nf, int W) {
    extern __shared__ int inv[];
    asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: after the previous grid
    if (blockIdx.x == 0) {
        for (int t = threadIdx.x; t < T; t += blockDim.x) inv[t] = -1;
        __syncthreads();
        for (int i = threadIdx.x; i < nf; i += blockDim.x) {
            const int t = ids[i];
            if (t >= 0 && t < T) inv[t] = i;      // duplicates: any one slot (same row, same output)
        }
        __syncthreads();
        for (int t = threadIdx.x; t < T; t += blockDim.x) inv_out[t] = inv[t];
    }
    // One warp per face row; lanes stride over the row's W 16-byte words, 20
    // loads in flight per lane before the stores (a 40-head d = 128 row, 640
    // words, is one round trip).
    constexpr int kU = 20;
    const int lane = threadIdx.x & 31;
    const int64_t rows = BF * nf;
    const int64_t wstride = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += wstride) {
        const int t = ids[r % nf];
        if (t < 0 || t >= T) continue;
        const uint4* src = q + ((r / nf) * T + t) * W;
        uint4* dst = qf + r * W;
        for (int w0 = lane; w0 < W; w0 += 32 * kU) {
            uint4 v[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u)
                if (w0 + 32 * u < W) v[u] = __ldcs(src + w0 + 32 * u);
#pragma unroll
            for (int u = 0; u < kU; ++u)
                if (w0 + 32 * u < W) dst[w0 + 32 * u] = v[u];
        }
    }
}

// ------------------------------------------------------------------ finiteness
template <bool kBf16>
__global__ void nonfinite_kernel(const void* __restrict__ x, int64_t n, int* flag) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    int bad = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        float f = kBf16 ? __uint_as_float(uint32_t(static_cast<const uint16_t*>(x)[i]) << 16)
                        : static_cast<const float*>(x)[i];
        bad |= !isfinite(f);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// ------------------------------------------------------------------ Ulysses
// Index map in ulysses_map.h (shared with the host routine used by the tests).
__global__ void __launch_bounds__(256) ulysses_kernel(const uint4* __restrict__ src,
                                                      uint4* __restrict__ dst, UlyssesShape s,
                                                      int mode) {
    const int64_t total = ulysses_words(s);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
        int64_t si, di;
        ulysses_map(s, mode, idx, si, di);
        if (di < 0) continue;
        dst[di] = si == -2 ? make_uint4(0, 0, 0, 0) : src[si];
    }
}

cudaError_t launch_shuffle(const void* src, void* dst, int B, int64_t Ls, int64_t L, int Hl, int P,
                           int d, int esize, int mode, cudaStream_t st, int* launches) {
    if ((d * esize) % 16) return cudaErrorInvalidValue;
    UlyssesShape s{B, P, Hl, d * esize / 16, Ls, L};
    ulysses_kernel<<<grid_for(ulysses_words(s), 256), 256, 0, st>>>(
        static_cast<const uint4*>(src), static_cast<uint4*>(dst), s, mode);
    if (launches) ++*launches;
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_euler(float* x, const void* v, int v_is_bf16, int64_t n, float dt,
                         cudaStream_t s, int* launches) {
    if (n <= 0) return cudaSuccess;
    const unsigned grid = grid_for((n + 7) / 8, 256, 16);
    if (v_is_bf16)
        return finish(launch_pdl(euler_kernel<true>, dim3(grid), dim3(256), 0, s, x, v, n, dt),
                      launches);
    else
        return finish(launch_pdl(euler_kernel<false>, dim3(grid), dim3(256), 0, s, x, v, n, dt),
                      launches);
}

cudaError_t launch_sampler(float* x, const void* v, int v_is_bf16, const float* eps, int64_t n,
                           float t_cur, float t_next, uint64_t seed, uint64_t offset,
                           void* x_bf16, cudaStream_t s, int* launches) {
    if (n <= 0) return cudaSuccess;
    const unsigned grid = grid_for((n + 3) / 4, 256, 16);
    const uint2 sd = make_uint2(uint32_t(seed), uint32_t(seed >> 32));
    const uint2 of = make_uint2(uint32_t(offset), uint32_t(offset >> 32));
    uint16_t* xb = static_cast<uint16_t*>(x_bf16);
    if (v_is_bf16) {
        if (eps) sampler_kernel<true, true><<<grid, 256, 0, s>>>(x, v, eps, n, t_cur, t_next, sd, of, xb);
        else sampler_kernel<true, false><<<grid, 256, 0, s>>>(x, v, eps, n, t_cur, t_next, sd, of, xb);
    } else {
        if (eps) sampler_kernel<false, true><<<grid, 256, 0, s>>>(x, v, eps, n, t_cur, t_next, sd, of, xb);
        else sampler_kernel<false, false><<<grid, 256, 0, s>>>(x, v, eps, n, t_cur, t_next, sd, of, xb);
    }
    if (launches) ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_face_rows(const void* src, void* dst, const int32_t* ids, int64_t BF, int64_t T,
                            int64_t nf, int row_bytes, int scatter, cudaStream_t s, int* launches) {
    if (row_bytes % 16) return cudaErrorInvalidValue;
    const int W = row_bytes / 16;
    const unsigned grid = grid_for(BF * nf * W, 256, 8);
    if (scatter)
        face_rows_kernel<true><<<grid, 256, 0, s>>>(static_cast<const uint4*>(src),
                                                    static_cast<uint4*>(dst), ids, BF, T, nf, W);
    else
        face_rows_kernel<false><<<grid, 256, 0, s>>>(static_cast<const uint4*>(src),
                                                     static_cast<uint4*>(dst), ids, BF, T, nf, W);
    if (launches) ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_audio_prep(const void* q, void* qf, int32_t* inv, const int32_t* ids, int64_t BF,
                              int64_t T, int64_t nf, int row_bytes, cudaStream_t s, int* launches) {
    if (row_bytes % 16 || T <= 0 || T > 49152 || nf <= 0) return cudaErrorInvalidValue;
    const int W = row_bytes / 16;
    const size_t smem = size_t(T) * 4;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(audio_prep_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
    }
    // face rows over the 4 warps of <= 4 CTAs per SM (one row per warp: the
    // gather is spread over every SM)
    const unsigned grid = grid_for(BF * nf, 4, 4);
    return finish(launch_pdl(audio_prep_kernel, dim3(grid), dim3(128), smem, s,
                             static_cast<const uint4*>(q), static_cast<uint4*>(qf), inv, ids, BF,
                             int(T), int(nf), W),
                  launches);
}

cudaError_t launch_nonfinite(const void* x, int is_bf16, int64_t n, int* flag, cudaStream_t s,
                             int* launches) {
    if (n <= 0) return cudaSuccess;
    const unsigned grid = grid_for(n, 256, 4);
    if (is_bf16)
        nonfinite_kernel<true><<<grid, 256, 0, s>>>(x, n, flag);
    else
        nonfinite_kernel<false><<<grid, 256, 0, s>>>(x, n, flag);
    if (launches) ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_pack_seq_to_peers(const void* src, void* dst, int B, int64_t Ls, int H, int P,
                                     int d, int esize, cudaStream_t s, int* launches) {
    return launch_shuffle(src, dst, B, Ls, Ls * P, H / P, P, d, esize, 0, s, launches);
}
cudaError_t launch_unpack_peers_to_heads(const void* src, void* dst, int B, int64_t Ls, int64_t L,
                                         int Hl, int P, int d, int esize, cudaStream_t s,
                                         int* launches) {
    return launch_shuffle(src, dst, B, Ls, L, Hl, P, d, esize, 1, s, launches);
}
cudaError_t launch_pack_heads_to_peers(const void* src, void* dst, int B, int64_t Ls, int64_t L,
                                       int Hl, int P, int d, int esize, cudaStream_t s,
                                       int* launches) {
    return launch_shuffle(src, dst, B, Ls, L, Hl, P, d, esize, 2, s, launches);
}
cudaError_t launch_unpack_peers_to_seq(const void* src, void* dst, int B, int64_t Ls, int H,
                                       int P, int d, int esize, cudaStream_t s, int* launches) {
    return launch_shuffle(src, dst, B, Ls, Ls * P, H / P, P, d, esize, 3, s, launches);
}

}  // namespace tmk
