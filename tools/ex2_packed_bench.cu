// ex2_packed_bench.cu -- throughput of packed exp2 (bf16x2 / f16x2) vs fp32
// MUFU.EX2 on this B200, cycles per warp-instruction per SMSP, and the error of
// each form vs fp64 exp2 over x in [-20, 0].
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

template <int OP>
__global__ void bench(uint32_t* out, int iters, long long* cyc) {
    uint32_t a[8];
    for (int i = 0; i < 8; ++i) a[i] = 0xBF00BF00u + threadIdx.x + i;   // ~ -0.5 in bf16
    float f[8];
    for (int i = 0; i < 8; ++i) f[i] = -0.5f - 0.001f * (threadIdx.x + i);
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
            if (OP == 1) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
            if (OP == 2) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
        }
    }
    const long long t1 = clock64();
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s += a[i] + __float_as_uint(f[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void accuracy(float* err_bf, float* err_h, float* err_f, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float x = -20.f * (i + 0.5f) / n;
    uint32_t xb, xh, yb, yh;
    asm("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(xb) : "f"(x));
    asm("cvt.rn.f16x2.f32 %0, %1, %1;" : "=r"(xh) : "f"(x));
    asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(yb) : "r"(xb));
    asm("ex2.approx.f16x2 %0, %1;" : "=r"(yh) : "r"(xh));
    float yf;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"(x));
    const float pb = __uint_as_float((yb & 0xffffu) << 16);
    float ph;
    asm("{ .reg .f16 h; mov.b32 {h, _}, %1; cvt.f32.f16 %0, h; }" : "=f"(ph) : "r"(yh));
    const double ref = exp2((double)x);
    err_bf[i] = (float)fabs((pb - ref) / ref);
    err_h[i] = (float)fabs((ph - ref) / ref);
    err_f[i] = (float)fabs((yf - ref) / ref);
}

template <int OP>
void run(const char* name) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* o;
    long long* c;
    cudaMalloc(&o, sizeof(uint32_t) * sms * 256);
    cudaMalloc(&c, sizeof(long long) * sms);
    const int iters = 4096;
    bench<OP><<<sms, 256>>>(o, iters, c);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[512];
    cudaMemcpy(h, c, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < sms; ++i) m += h[i];
    m /= sms;
    printf("%-16s %6.2f cycles per warp-instr per SMSP (8 warps/CTA) [%s]\n", name,
           m / (iters * 8.0 * 2.0), cudaGetErrorString(e));
    cudaFree(o);
    cudaFree(c);
}

int main() {
    run<0>("ex2 f32");
    run<1>("ex2 bf16x2");
    run<2>("ex2 f16x2");
    const int n = 1 << 20;
    float *a, *b, *c;
    cudaMallocManaged(&a, n * 4);
    cudaMallocManaged(&b, n * 4);
    cudaMallocManaged(&c, n * 4);
    accuracy<<<n / 256, 256>>>(a, b, c, n);
    cudaDeviceSynchronize();
    // max relative error by x band
    const float bands[] = {0, -2, -4, -8, -12, -16, -20};
    for (int k = 0; k + 1 < 7; ++k) {
        float mb = 0, mh = 0, mf = 0;
        for (int i = 0; i < n; ++i) {
            const float x = -20.f * (i + 0.5f) / n;
            if (x <= bands[k] && x > bands[k + 1]) {
                mb = fmaxf(mb, a[i]); mh = fmaxf(mh, b[i]); mf = fmaxf(mf, c[i]);
            }
        }
        printf("x in (%5.0f, %5.0f]: max rel err bf16x2 %.2e  f16x2 %.2e  f32 %.2e\n", bands[k + 1],
               bands[k], mb, mh, mf);
    }
    return 0;
}
