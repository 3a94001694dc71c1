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
// Blackwell design (one CTA = one head x two 128-row Q tiles):
//   warp 8      TMA producer: Q0,Q1 once, then K_j / V_j tiles through a
//               4-slot shared-memory ring (cp.async.bulk.tensor, 128B swizzle)
//   warp 9      tcgen05 MMA issuer (one thread) + TMEM owner:
//                 S_i = Q_i K_j^T  (SS, M=128 N=128 K=d, fp32 in TMEM)
//                 O_i += P_i V_j   (TS: P_i bf16 read from TMEM, V MN-major)
//               issue order PV0_{j-1}, S0_j, PV1_{j-1}, S1_j: the tensor core
//               works on one tile while the other tile's softmax runs.
//   warps 0-7   softmax, one warpgroup per Q tile, one thread per query row
//               (tcgen05.ld 32x32b puts a whole S row in one thread's
//               registers, so row max/sum need no shuffles); exp2 with the
//               scale*log2(e) folded into one FFMA; conditional O rescale
//               (only when the running max grows by > 8 in log2 units --
//               exact after the final 1/l); P rounded to bf16 (RNE) and
//               stored back into TMEM over S_i; epilogue O/l -> bf16.
// TMEM: S0 [0,128) S1 [128,256) O0 [256,256+d) O1 [256+d, 256+2d).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <mutex>

#include "internal.h"
#include "ptx.cuh"

namespace tmk {
namespace {

constexpr int kBM = 128;          // query rows per Q tile
constexpr int kBN = 128;          // keys per KV tile
constexpr int kStages = 4;        // K/V smem ring slots
constexpr int kThreads = 320;     // 8 softmax warps + TMA warp + MMA warp
constexpr int kHalfBytes = 128 * 128;   // one 64-column (128 B) half of a 128-row tile

struct __align__(64) FmhaParams {
    CUtensorMap tq;                   // Q [B][Lq][H][d]
    CUtensorMap tk[kMaxSegments];     // K segments [B][len][H][d]
    CUtensorMap tv[kMaxSegments];     // V segments
    int seg_tile_start[kMaxSegments + 1];
    int seg_len[kMaxSegments];
    int nseg;
    int n_tiles;
    int Lq, H, B;
    float scale_log2;                 // softmax scale * log2(e)
    uint16_t* o;                      // bf16 bits [B][Lq][H][d]
};

__device__ __forceinline__ void tile_info(const FmhaParams& p, int j, int& seg, int& row,
                                          int& valid) {
    seg = 0;
#pragma unroll
    for (int s = 1; s < kMaxSegments; ++s)
        if (s < p.nseg && j >= p.seg_tile_start[s]) seg = s;
    row = (j - p.seg_tile_start[seg]) * kBN;
    valid = min(kBN, p.seg_len[seg] - row);
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) fmha_sm100_kernel(const __grid_constant__ FmhaParams p) {
    constexpr int kTileBytes = kBN * D * 2;
    constexpr uint32_t kIdescS = make_idesc_bf16(kBM, kBN, 0, 0);   // Q, K both K-major
    constexpr uint32_t kIdescO = make_idesc_bf16(kBM, D, 0, 1);     // P (TMEM), V MN-major

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* sQ = smem;                                  // 2 tiles
    uint8_t* sKV = smem + 2 * kTileBytes;                // kStages slots
    uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + kStages * kTileBytes);
    uint64_t* q_full = bars;
    uint64_t* kv_full = bars + 1;
    uint64_t* kv_empty = kv_full + kStages;
    uint64_t* s_full = kv_empty + kStages;
    uint64_t* p_full = s_full + 2;
    uint64_t* o_final = p_full + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_final + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int h = blockIdx.y, b = blockIdx.z;
    const int q0 = blockIdx.x * 2 * kBM;
    const int n = p.n_tiles;

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 128);
            mbar_init(&o_final[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == 8 && lane == 0) {
        tma_prefetch(&p.tq);
        for (int s = 0; s < p.nseg; ++s) {
            tma_prefetch(&p.tk[s]);
            tma_prefetch(&p.tv[s]);
        }
    }
    if (warp == 9) tmem_alloc(tmem_holder, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;

    if (warp == 8) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            mbar_arrive_expect_tx(q_full, 2 * kTileBytes);
            for (int i = 0; i < 2; ++i)
                for (int hf = 0; hf < D / 64; ++hf)
                    tma_load_4d(sQ + i * kTileBytes + hf * kHalfBytes, &p.tq, q_full, hf * 64, h,
                                q0 + i * kBM, b);
            for (int it = 0; it < 2 * n; ++it) {
                const int s = it % kStages;
                mbar_wait(&kv_empty[s], ((it / kStages) & 1) ^ 1);
                int seg, row, valid;
                tile_info(p, it >> 1, seg, row, valid);
                const CUtensorMap* m = (it & 1) ? &p.tv[seg] : &p.tk[seg];
                mbar_arrive_expect_tx(&kv_full[s], kTileBytes);
                for (int hf = 0; hf < D / 64; ++hf)
                    tma_load_4d(sKV + s * kTileBytes + hf * kHalfBytes, m, &kv_full[s], hf * 64,
                                h, row, b);
            }
        }
    } else if (warp == 9) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t sQa = smem_u32(sQ), sKVa = smem_u32(sKV);
            auto issue_s = [&](int i, int slot) {
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint32_t off = (kk >> 2) * kHalfBytes + (kk & 3) * 32;
                    mma_ss(tmem + i * 128, make_sdesc_sw128(sQa + i * kTileBytes + off, 16, 1024),
                           make_sdesc_sw128(sKVa + slot * kTileBytes + off, 16, 1024), kIdescS,
                           kk > 0);
                }
            };
            auto issue_pv = [&](int i, int slot, bool acc) {
#pragma unroll
                for (int kk = 0; kk < kBN / 16; ++kk)
                    mma_ts(tmem + 256 + i * D, tmem + i * 128 + kk * 8,
                           make_sdesc_sw128(sKVa + slot * kTileBytes + kk * 2048, kHalfBytes, 1024),
                           kIdescO, (acc || kk > 0) ? 1u : 0u);
            };
            mbar_wait(q_full, 0);
            tc_fence_after();
            for (int j = 0; j < n; ++j) {
                const int ik = 2 * j, sk = ik % kStages;
                mbar_wait(&kv_full[sk], (ik / kStages) & 1);
                tc_fence_after();
                int sv = 0;
                if (j > 0) {
                    const int iv = 2 * (j - 1) + 1;
                    sv = iv % kStages;
                    mbar_wait(&kv_full[sv], (iv / kStages) & 1);
                    tc_fence_after();
                }
                for (int i = 0; i < 2; ++i) {
                    if (j > 0) {
                        mbar_wait(&p_full[i], (j - 1) & 1);
                        tc_fence_after();
                        issue_pv(i, sv, j - 1 > 0);
                    }
                    issue_s(i, sk);
                    mma_commit(&s_full[i]);
                }
                mma_commit(&kv_empty[sk]);
                if (j > 0) mma_commit(&kv_empty[sv]);
            }
            const int iv = 2 * (n - 1) + 1, sv = iv % kStages;
            mbar_wait(&kv_full[sv], (iv / kStages) & 1);
            tc_fence_after();
            for (int i = 0; i < 2; ++i) {
                mbar_wait(&p_full[i], (n - 1) & 1);
                tc_fence_after();
                issue_pv(i, sv, n - 1 > 0);
                mma_commit(&o_final[i]);
            }
            mma_commit(&kv_empty[sv]);
        }
    } else {
        // ------------------------------------------------ softmax (warps 0-7)
        const int i = warp >> 2, wq = warp & 3;
        const uint32_t lane_off = uint32_t(wq * 32) << 16;
        const uint32_t tSi = tmem + lane_off + i * 128;
        const uint32_t tOi = tmem + lane_off + 256 + i * D;
        const float sl2 = p.scale_log2;
        float m_run = -INFINITY, l = 0.f;
        uint32_t r[kBN];
        uint32_t pk[kBN / 2];
        for (int j = 0; j < n; ++j) {
            int seg, row, valid;
            tile_info(p, j, seg, row, valid);
            mbar_wait(&s_full[i], j & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < kBN; c += 32) tmem_ld32(tSi + c, r + c);
            tmem_wait_ld();
            if (valid < kBN) {
#pragma unroll
                for (int c = 0; c < kBN; ++c)
                    if (c >= valid) r[c] = 0xff800000u;   // -inf: key beyond the segment
            }
            float mx = -INFINITY;
#pragma unroll
            for (int c = 0; c < kBN; ++c) mx = fmaxf(mx, __uint_as_float(r[c]));
            const float m_new = fmaxf(m_run, mx * sl2);
            const bool need = m_new > m_run + 8.0f;
            float alpha = 1.f;
            if (need) {
                alpha = ex2(m_run - m_new);
                m_run = m_new;
            }
            l *= alpha;
            if (j > 0 && __any_sync(0xffffffffu, need)) {
                // O_i was last written by PV_i_{j-1}, complete before s_full fired.
#pragma unroll
                for (int c = 0; c < D; c += 32) {
                    uint32_t o[32];
                    tmem_ld32(tOi + c, o);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
                    tmem_st32(tOi + c, o);
                }
            }
            const float nm = (m_run == -INFINITY) ? 0.f : -m_run;
            float sum = 0.f;
#pragma unroll
            for (int c = 0; c < kBN / 2; ++c) {
                const float p0 = ex2(fmaf(__uint_as_float(r[2 * c]), sl2, nm));
                const float p1 = ex2(fmaf(__uint_as_float(r[2 * c + 1]), sl2, nm));
                sum += p0 + p1;
                pk[c] = pack_bf16x2(p0, p1);
            }
            l += sum;
            tmem_st32(tSi, pk);
            tmem_st32(tSi + 32, pk + 32);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&p_full[i]);
        }
        // ------------------------------------------------ epilogue O / l
        mbar_wait(&o_final[i], 0);
        tc_fence_after();
        const float inv_l = 1.f / l;
        const int q = q0 + i * kBM + wq * 32 + lane;
        uint16_t* dst = p.o + ((int64_t(b) * p.Lq + q) * p.H + h) * D;
#pragma unroll
        for (int c = 0; c < D; c += 32) {
            uint32_t o[32];
            tmem_ld32(tOi + c, o);
            tmem_wait_ld();
            uint32_t w[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
                w[e] = pack_bf16x2(__uint_as_float(o[2 * e]) * inv_l,
                                   __uint_as_float(o[2 * e + 1]) * inv_l);
            if (q < p.Lq) {
                uint4* d4 = reinterpret_cast<uint4*>(dst + c);
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    d4[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
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
bool make_map(CUtensorMap* m, const void* base, int d, int H, int64_t L, int B) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[4] = {cuuint64_t(d), cuuint64_t(H), cuuint64_t(L), cuuint64_t(B)};
    cuuint64_t strides[3] = {cuuint64_t(d) * 2, cuuint64_t(H) * d * 2, cuuint64_t(L) * H * d * 2};
    cuuint32_t box[4] = {64, 1, 128, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int D>
constexpr int smem_bytes() {
    return 1024 + (2 + kStages) * kBN * D * 2 + 256;
}

}  // namespace

cudaError_t launch_fmha_sm100(const AttnProblem& pr, cudaStream_t stream, int* launches) {
    if (pr.d != 64 && pr.d != 128) return cudaErrorInvalidValue;
    FmhaParams p;
    memset(&p, 0, sizeof(p));
    if (!make_map(&p.tq, pr.q, pr.d, pr.H, pr.Lq, pr.B)) return cudaErrorInvalidValue;
    int tiles = 0;
    for (int s = 0; s < pr.nseg; ++s) {
        if (!make_map(&p.tk[s], pr.seg[s].k, pr.d, pr.H, pr.seg[s].len, pr.B) ||
            !make_map(&p.tv[s], pr.seg[s].v, pr.d, pr.H, pr.seg[s].len, pr.B))
            return cudaErrorInvalidValue;
        p.seg_tile_start[s] = tiles;
        p.seg_len[s] = int(pr.seg[s].len);
        tiles += int((pr.seg[s].len + kBN - 1) / kBN);
    }
    p.seg_tile_start[pr.nseg] = tiles;
    p.nseg = pr.nseg;
    p.n_tiles = tiles;
    p.Lq = int(pr.Lq);
    p.H = pr.H;
    p.B = pr.B;
    p.scale_log2 = pr.scale * 1.4426950408889634f;
    p.o = static_cast<uint16_t*>(pr.o);
    const int qtiles = int((pr.Lq + kBM - 1) / kBM);
    dim3 grid((qtiles + 1) / 2, pr.H, pr.B);
    cudaError_t e;
    if (pr.d == 128) {
        static bool attr = false;
        if (!attr) {
            e = cudaFuncSetAttribute(fmha_sm100_kernel<128>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<128>());
            if (e != cudaSuccess) return e;
            attr = true;
        }
        fmha_sm100_kernel<128><<<grid, kThreads, smem_bytes<128>(), stream>>>(p);
    } else {
        static bool attr = false;
        if (!attr) {
            e = cudaFuncSetAttribute(fmha_sm100_kernel<64>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<64>());
            if (e != cudaSuccess) return e;
            attr = true;
        }
        fmha_sm100_kernel<64><<<grid, kThreads, smem_bytes<64>(), stream>>>(p);
    }
    if (launches) ++*launches;
    return cudaGetLastError();
}

}  // namespace tmk
