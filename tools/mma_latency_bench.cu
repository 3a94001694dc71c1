// mma_latency_bench.cu -- tcgen05 issue cost and issue-to-completion latency
// into an IDLE tensor pipe (the situation of the attention kernel's S MMAs
// after a wait), and TS-MMA throughput while other warps stream tcgen05.ld
// out of TMEM (the softmax loading S while PV runs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2506_03099_b200/csrc \
//        mma_latency_bench.cu -o mma_latency_bench
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace tmk;

// MODE 0: 8 SS MMAs (per-MMA elect), 1: 8 SS MMAs (one asm group),
//      2: 8 TS MMAs (group), 3: 1 SS MMA.  LOADERS: warps 4..7 stream
//      tcgen05.ld 32x32b.x32 over TMEM columns [0,128) during the timed loop.
template <int MODE, bool LOADERS>
__global__ void __launch_bounds__(256, 1) lat(long long* out, int reps) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    __shared__ volatile int stop;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u * ((i & 7) == 0);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        stop = 0;
    }
    if (warp == 0) tmem_alloc(&holder, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = holder;
    if (warp == 0) {
        const uint32_t base = smem_u32(smem);
        constexpr uint32_t idesc_kk = make_idesc_bf16(128, 128, 0, 0);
        constexpr uint32_t idesc_kmn = make_idesc_bf16(128, 128, 0, 1);
        const uint64_t da = make_sdesc_sw128(base, 16, 1024);
        const uint64_t db = make_sdesc_sw128(base + 32768, 16, 1024);
        const uint64_t dbmn = make_sdesc_sw128(base + 32768, 16384, 1024);
        long long iss = 0, done = 0;
        for (int r = 0; r < reps; ++r) {
            const long long t0 = clock64();
            if (MODE == 0) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ss_w(tmem + 256, da + (kk & 3) * 2, db + (kk & 3) * 2, idesc_kk, kk > 0);
            } else if (MODE == 1) {
                mma_ss_group<8>(tmem + 256, da, db, idesc_kk);
            } else if (MODE == 2) {
                mma_ts_group8(tmem + 256, tmem + 128, dbmn, idesc_kmn, 0);
            } else {
                mma_ss_w(tmem + 256, da, db, idesc_kk, 0);
            }
            const long long t1 = clock64();
            mma_commit_w(&bar);
            mbar_wait(&bar, r & 1);
            const long long t2 = clock64();
            if (r >= 4) { iss += t1 - t0; done += t2 - t0; }
            __syncwarp();
        }
        if (threadIdx.x == 0) {
            out[2 * blockIdx.x] = iss / (reps - 4);
            out[2 * blockIdx.x + 1] = done / (reps - 4);
            stop = 1;
        }
    } else if (LOADERS && warp >= 4) {
        const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
        uint32_t r[32];
        uint32_t acc = 0;
        while (!stop) {
#pragma unroll
            for (int c = 0; c < 128; c += 32) {
                tmem_ld32(tmem + lane_off + c, r);
                tmem_wait_ld();
                acc += r[0] + r[31];
            }
        }
        if (acc == 0x12345678u) out[0] = acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int MODE, bool LOADERS>
void run(const char* name) {
    long long* d;
    cudaMalloc(&d, sizeof(long long) * 2 * 148);
    cudaFuncSetAttribute(lat<MODE, LOADERS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    lat<MODE, LOADERS><<<148, 256, 100 * 1024>>>(d, 200);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> h(2 * 148);
    cudaMemcpy(h.data(), d, sizeof(long long) * 2 * 148, cudaMemcpyDeviceToHost);
    std::vector<long long> a, b;
    for (int i = 0; i < 148; ++i) { a.push_back(h[2 * i]); b.push_back(h[2 * i + 1]); }
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    printf("%-40s issue %5lld cyc, issue->commit observed %5lld cyc  [%s]\n", name, a[74], b[74],
           cudaGetErrorString(e));
    cudaFree(d);
}

// tcgen05.ld throughput of 4 warps (each 128 columns x 32 lanes = 16 KB per
// pass, as the softmax loading S), with warp 0 keeping the tensor pipe busy
// with TS MMAs accumulating into other TMEM columns (MMA=true) or idle.
template <bool MMA>
__global__ void __launch_bounds__(256, 1) ldbw(long long* out, int passes) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar[2];
    __shared__ uint32_t holder;
    __shared__ volatile int stop;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u * ((i & 7) == 0);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
        stop = 0;
    }
    if (warp == 0) tmem_alloc(&holder, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = holder;
    if (warp == 0) {
        if (MMA) {
            const uint32_t base = smem_u32(smem);
            constexpr uint32_t idesc_kmn = make_idesc_bf16(128, 128, 0, 1);
            const uint64_t dbmn = make_sdesc_sw128(base + 32768, 16384, 1024);
            for (int it = 0; !stop; ++it) {
                mma_ts_group8(tmem + 256, tmem + 128, dbmn, idesc_kmn, 1);
                mma_commit_w(&bar[it & 1]);
                if (it > 0) mbar_wait(&bar[(it - 1) & 1], ((it - 1) >> 1) & 1);
            }
        }
    } else if (warp >= 4) {
        const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
        uint32_t r[128];
        uint32_t acc = 0;
        for (int w = 0; w < 4; ++w) {   // warm-up
#pragma unroll
            for (int c = 0; c < 128; c += 32) tmem_ld32(tmem + lane_off + c, r + c);
            tmem_wait_ld();
        }
        const long long t0 = clock64();
        for (int ps = 0; ps < passes; ++ps) {
#pragma unroll
            for (int c = 0; c < 128; c += 32) tmem_ld32(tmem + lane_off + c, r + c);
            tmem_wait_ld();
            acc += r[0] ^ r[37] ^ r[127];
        }
        const long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) out[blockIdx.x * 4 + (warp & 3)] = t1 - t0;
        if (acc == 0x12345678u) out[0] = acc;
        asm volatile("bar.sync 1, 128;");
        if (threadIdx.x == 128) stop = 1;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <bool MMA>
void run_ld(const char* name) {
    long long* d;
    cudaMalloc(&d, sizeof(long long) * 4 * 148);
    cudaFuncSetAttribute(ldbw<MMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int passes = 400;
    ldbw<MMA><<<148, 256, 100 * 1024>>>(d, passes);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> h(4 * 148);
    cudaMemcpy(h.data(), d, sizeof(long long) * 4 * 148, cudaMemcpyDeviceToHost);
    std::sort(h.begin(), h.end());
    printf("%-40s %6.1f cyc per 16 KB warp load (median), max %6.1f  [%s]\n", name,
           h[h.size() / 2] / double(passes), h.back() / double(passes), cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<3, false>("1 SS MMA, idle pipe");
    run<0, false>("8 SS MMAs per-MMA elect, idle pipe");
    run<1, false>("8 SS MMAs one asm group, idle pipe");
    run<2, false>("8 TS MMAs one asm group, idle pipe");
    run<1, true>("8 SS MMAs group + 4 warps tcgen05.ld");
    run<2, true>("8 TS MMAs group + 4 warps tcgen05.ld");
    run_ld<false>("4 warps tcgen05.ld, tensor pipe idle");
    run_ld<true>("4 warps tcgen05.ld, TS MMAs running");
    return 0;
}
