// softmax_microbench.cu -- cycles for the attention kernel's per-row exp loop
// (128 columns per thread: FFMA2 scale/subtract, MUFU.EX2 or polynomial exp2,
// FADD2 row sum, F2FP bf16 pack) in registers, one warp per SMSP, to find the
// real per-tile cost and its limiting pipe.  Variants toggle parts of the mix.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

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
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t d;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
    return d;
}
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
    constexpr float kMagic = 12582912.f;
    x.x = fmaxf(x.x, -125.f);
    x.y = fmaxf(x.y, -125.f);
    const float2 j = fadd2(x, make_float2(kMagic, kMagic));
    const float2 n = fadd2(j, make_float2(-kMagic, -kMagic));
    const float2 f = ffma2(n, make_float2(-1.f, -1.f), x);
    float2 p = ffma2(make_float2(0.055171094834804535f, 0.055171094834804535f), f,
                     make_float2(0.24260999262332916f, 0.24260999262332916f));
    p = ffma2(p, f, make_float2(0.6932609677314758f, 0.6932609677314758f));
    p = ffma2(p, f, make_float2(0.9999281167984009f, 0.9999281167984009f));
    uint32_t ex, ey;
    asm("{\n\t.reg .b32 t;\n\tshl.b32 t, %1, 23;\n\tadd.u32 %0, %2, t;\n\t}"
        : "=r"(ex) : "r"(__float_as_uint(j.x)), "r"(__float_as_uint(p.x)));
    asm("{\n\t.reg .b32 t;\n\tshl.b32 t, %1, 23;\n\tadd.u32 %0, %2, t;\n\t}"
        : "=r"(ey) : "r"(__float_as_uint(j.y)), "r"(__float_as_uint(p.y)));
    return make_float2(__uint_as_float(ex), __uint_as_float(ey));
}

// MODE bits: 1 = pack (F2FP), 2 = sum (FADD2); POLY = bitmask over 16 pairs
template <int MODE, uint32_t POLY>
__global__ void bench(const float* in, uint32_t* out, int iters, long long* cyc) {
    float r[128];
#pragma unroll
    for (int c = 0; c < 128; ++c) r[c] = in[(threadIdx.x * 7 + c) & 1023];
    uint32_t sink = 0;
    float lsum = 0.f;
    const float sl2 = 0.1275f;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const float nm = -1.5f - 0.001f * it;
        const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(nm, nm);
        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const float2 x = ffma2(make_float2(r[32 * c + 2 * e], r[32 * c + 2 * e + 1]), sc2, nm2);
                float2 pe;
                if ((POLY >> e) & 1) {
                    pe = exp2_poly2(x);
                } else {
                    pe.x = ex2(x.x);
                    pe.y = ex2(x.y);
                }
                if (MODE & 2) acc[e & 3] = fadd2(acc[e & 3], pe);
                pk[e] = (MODE & 1) ? pack_bf16x2(pe.x, pe.y) : (__float_as_uint(pe.x) ^ __float_as_uint(pe.y));
            }
#pragma unroll
            for (int e = 0; e < 16; ++e) sink += pk[e];
        }
        const float2 s01 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
        lsum += s01.x + s01.y;
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = sink + __float_as_uint(lsum);
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE, uint32_t POLY>
void run(const char* name, int warps) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* in;
    uint32_t* o;
    long long* c;
    cudaMalloc(&in, 1024 * 4);
    cudaMemset(in, 0, 1024 * 4);
    cudaMalloc(&o, sizeof(uint32_t) * sms * warps * 32);
    cudaMalloc(&c, sizeof(long long) * sms);
    const int iters = 2000;
    bench<MODE, POLY><<<sms, warps * 32>>>(in, o, iters, c);
    cudaDeviceSynchronize();
    long long h[512];
    cudaMemcpy(h, c, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < sms; ++i) m += h[i];
    m /= sms;
    printf("%-34s warps/SMSP=%d: %7.0f cycles per 128-col row-tile per warp\n", name, warps / 4,
           m / iters);
    cudaFree(in);
    cudaFree(o);
    cudaFree(c);
}

int main() {
    for (int w : {4, 8}) {
        run<3, 0x0000>("all MUFU, pack+sum", w);
        run<3, 0x4444>("4/16 poly, pack+sum", w);
        run<3, 0x2492>("5/16 poly, pack+sum", w);
        run<3, 0xA54A>("7/16 poly, pack+sum", w);
        run<3, 0xAAAA>("8/16 poly, pack+sum", w);
        run<1, 0x4444>("4/16 poly, pack, no sum", w);
        run<2, 0x4444>("4/16 poly, sum, no pack", w);
        run<0, 0x4444>("4/16 poly, no pack, no sum", w);
        run<0, 0x0000>("all MUFU, no pack, no sum", w);
        run<0, 0xFFFF>("all poly, no pack, no sum", w);
    }
    return 0;
}
