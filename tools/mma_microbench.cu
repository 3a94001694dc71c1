// mma_microbench.cu -- calibrate tcgen05.mma throughput on this B200:
// back-to-back kind::f16 MMAs (bf16 in, fp32 accumulate) from one thread per
// CTA, one CTA per SM, operands resident in shared memory (SWIZZLE_128B
// K-major layout as in the attention kernel).  Reports cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2506_03099_b200/csrc \
//        mma_microbench.cu -o mma_microbench
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace tmk;

template <int MODE, int N>
__global__ void __launch_bounds__(128, 1) bench(long long* out, int iters) {
    // MODE 0: SS (A, B smem), MODE 1: TS (A tmem, B smem MN-major), MODE 2: SS with B MN-major
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar[2];
    __shared__ uint32_t holder;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u * ((i & 7) == 0);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(&holder, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = holder;
    if (warp == 0) {        // whole warp converged; one elected lane issues
        const uint32_t base = smem_u32(smem);
        constexpr uint32_t idesc_kk = make_idesc_bf16(128, N, 0, 0);
        constexpr uint32_t idesc_kmn = make_idesc_bf16(128, N, 0, 1);
        const uint64_t da = make_sdesc_sw128(base, 16, 1024);
        const uint64_t db = make_sdesc_sw128(base + 32768, 16, 1024);
        const uint64_t dbmn = make_sdesc_sw128(base + 32768, 16384, 1024);
        long long t0 = 0;
        for (int it = -2; it < iters; ++it) {
            if (it == 0) t0 = clock64();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                if (MODE == 0)
                    mma_ss_w(tmem + 256, da + (kk & 3) * 2, db + (kk & 3) * 2, idesc_kk, 1);
                else if (MODE == 1)
                    mma_ts_w(tmem + 256, tmem + kk * 8, dbmn + kk * 128, idesc_kmn, 1);
                else
                    mma_ss_w(tmem + 256, da + (kk & 3) * 2, dbmn + kk * 128, idesc_kmn, 1);
            }
            // keep one group of 8 queued: wait for the previous group only
            mma_commit_w(&bar[it & 1]);
            if (it > -2) mbar_wait(&bar[(it - 1) & 1], (((it + 2) - 1) >> 1) & 1);
        }
        const long long t1 = clock64();
        const int nl = iters + 1;   // last group's index
        mbar_wait(&bar[nl & 1], (nl >> 1) & 1);
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int MODE, int N>
void run(const char* name, int sms) {
    long long* d;
    cudaMalloc(&d, sizeof(long long) * sms);
    const int iters = 2000;
    cudaFuncSetAttribute(bench<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    bench<MODE, N><<<sms, 128, 100 * 1024>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[256];
    cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += h[i];
    mean /= sms;
    const double per = mean / (iters * 8.0);
    const double macs = 128.0 * N * 16;
    printf("%-28s N=%3d: %7.1f cycles/MMA, %6.0f MAC/clk/SM (%.0f%% of 4096)  [%s]\n", name, N, per,
           macs / per, 100 * macs / per / 4096, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int s : {1, sms}) {
        printf("--- %d CTA(s)\n", s);
        run<0, 128>("SS K-major/K-major", s);
        run<0, 256>("SS K-major/K-major", s);
        run<1, 128>("TS A=tmem, B MN-major", s);
        run<1, 256>("TS A=tmem, B MN-major", s);
        run<2, 128>("SS K-major/B MN-major", s);
        run<0, 64>("SS K-major/K-major", s);
    }
    return 0;
}
