// pipe_microbench.cu -- per-SMSP throughput of the softmax instructions on
// this B200: MUFU.EX2, FFMA, FFMA2, FADD2, F2FP (cvt.rn.bf16x2.f32), FMNMX3,
// integer shift+add.  8 independent chains per thread, W warps per CTA, one
// CTA per SM.  Reports cycles per warp-instruction per SMSP.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void bench(float* out, int iters, long long* cyc) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = 0.001f * (threadIdx.x + i);
    uint64_t b[8];
    for (int i = 0; i < 8; ++i) b[i] = (uint64_t(__float_as_uint(a[i])) << 32) | __float_as_uint(a[i] + 1);
    const uint64_t c2 = (uint64_t(__float_as_uint(0.999f)) << 32) | __float_as_uint(0.999f);
    const uint64_t d2 = (uint64_t(__float_as_uint(1e-7f)) << 32) | __float_as_uint(1e-7f);
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
            if (OP == 1) asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, 0f33D6BF95;" : "+f"(a[i]));
            if (OP == 2) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(b[i]) : "l"(c2), "l"(d2));
            if (OP == 3) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(b[i]) : "l"(d2));
            if (OP == 4) {
                uint32_t r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
                a[i] = __uint_as_float(r);
            }
            if (OP == 5) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 3) & 7]), "f"(a[(i + 5) & 7]));
            if (OP == 6) {
                uint32_t x = __float_as_uint(a[i]);
                asm volatile("{.reg .b32 t; shl.b32 t, %0, 23; add.u32 %0, %0, t;}" : "+r"(x));
                a[i] = __uint_as_float(x);
            }
            if (OP == 7) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]), "f"(a[(i + 2) & 7]));
        }
    }
    const long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(uint32_t(b[i]));
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* o;
    long long* c;
    cudaMalloc(&o, sizeof(float) * sms * warps * 32);
    cudaMalloc(&c, sizeof(long long) * sms);
    const int iters = 4096;
    bench<OP><<<sms, warps * 32>>>(o, iters, c);
    cudaDeviceSynchronize();
    long long h[512];
    cudaMemcpy(h, c, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < sms; ++i) m += h[i];
    m /= sms;
    // warp-instructions per SMSP = iters * 8 * (warps / 4)
    const double per = m / (iters * 8.0 * (warps / 4.0));
    printf("%-22s warps/CTA=%2d: %6.2f cycles per warp-instr per SMSP\n", name, warps, per);
    cudaFree(o);
    cudaFree(c);
}

int main() {
    for (int w : {4, 8, 16}) {
        run<0>("MUFU.EX2", w);
        run<1>("FFMA (imm)", w);
        run<7>("FFMA (3 reg)", w);
        run<2>("FFMA2", w);
        run<3>("FADD2", w);
        run<4>("F2FP bf16x2", w);
        run<5>("FMNMX3", w);
        run<6>("SHL+IADD (2 instr)", w);
    }
    return 0;
}
