// Single-SM (and few-SM) L2 transfer rates: what one CTA can move between L2
// and shared memory / registers, the budget of the stream-K merge chain
// (partner partial write, merger reads, output store).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sm_l2_bw tools/sm_l2_bw.cu && /tmp/sm_l2_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// mode 0: bulk copies (cp.async.bulk) of `chunk` bytes, `inflight` outstanding, total `bytes` per CTA
// mode 1: per-thread 16-B loads (ld.global.cg), 16 in flight per thread
// mode 2: per-thread 16-B stores (st.global) then __threadfence
__global__ void __launch_bounds__(256, 1) k(const uint8_t* src, uint8_t* dst, int mode, int bytes, int chunk,
                                           int inflight, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[4];
    const uint8_t* s = src + (size_t)blockIdx.x * bytes;
    uint8_t* d = dst + (size_t)blockIdx.x * bytes;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    uint4 acc = make_uint4(0, 0, 0, 0);
    if (mode == 0) {
        if (threadIdx.x == 0) {
            const int n = bytes / chunk;
            for (int j = 0; j < n; ++j) {
                const int b = j % inflight;
                if (j >= inflight) {
                    const uint32_t ph = ((j / inflight) - 1) & 1;
                    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(&bar[b])), "r"(ph));
                }
                asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bar[b])), "r"(chunk));
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(su32(sm + b * chunk)), "l"(s + (size_t)j * chunk), "r"(chunk), "r"(su32(&bar[b])) : "memory");
            }
            for (int j = n - inflight < 0 ? 0 : n - inflight; j < n; ++j) {
                const int b = j % inflight;
                const uint32_t ph = (j / inflight) & 1;
                asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(&bar[b])), "r"(ph));
            }
        }
    } else if (mode == 1) {
        const uint4* g = reinterpret_cast<const uint4*>(s);
        const int n = bytes / 16;
        for (int i = threadIdx.x; i < n; i += 256 * 16) {
            uint4 v[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = i + e * 256 < n ? __ldcg(g + i + e * 256) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int e = 0; e < 16; ++e) { acc.x ^= v[e].x; acc.y ^= v[e].y; acc.z ^= v[e].z; acc.w ^= v[e].w; }
        }
    } else if (mode == 3) {
        // bulk smem -> global stores of `chunk` bytes, then wait for the writes and fence
        if (threadIdx.x == 0) {
            for (int j = 0; j < bytes / chunk; ++j)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                             ::"l"(d + (size_t)j * chunk), "r"(su32(sm + (j % 3) * chunk)), "r"(chunk) : "memory");
            asm volatile("cp.async.bulk.commit_group;");
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            __threadfence();
        }
    } else if (mode == 4) {
        uint4* g = reinterpret_cast<uint4*>(d);
        const int n = bytes / 16;
        for (int i = threadIdx.x; i < n; i += 256) g[i] = make_uint4(i, 1, 2, 3);
    } else {
        uint4* g = reinterpret_cast<uint4*>(d);
        const int n = bytes / 16;
        for (int i = threadIdx.x; i < n; i += 256) g[i] = make_uint4(i, 1, 2, 3);
        __threadfence();
    }
    __syncthreads();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc.x == 0x12345678) out[gridDim.x] = acc.y;
}

int main() {
    const size_t N = 256 << 20;
    uint8_t *src, *dst;
    unsigned long long* out;
    cudaMalloc(&src, N);
    cudaMalloc(&dst, N);
    cudaMalloc(&out, 4096 * 8);
    cudaMemset(src, 1, N);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const char* names[5] = {"bulk g2s", "ldg.cg 16B", "st.global+fence", "bulk s2g+wait", "st.global only"};
    for (int mode = 0; mode < 5; ++mode)
        for (int ctas : {1, 60, 148})
            for (int bytes : {32768, 65536, 131072}) {
                const int chunks[2] = {16384, 65536};
                for (int ci = 0; ci < (mode == 0 || mode == 3 ? 2 : 1); ++ci) {
                    const int chunk = mode == 0 || mode == 3 ? (chunks[ci] > bytes ? bytes : chunks[ci]) : 0;
                    const int inflight = mode == 0 ? (chunk == 65536 ? 3 : 4) : 0;
                    unsigned long long h[148];
                    double best = 1e30;
                    for (int rep = 0; rep < 5; ++rep) {
                        // warm the source into L2 (it was just read / written) -- read it once
                        k<<<ctas, 256, 200 * 1024>>>(src, dst, 1, bytes, chunk, inflight, out);
                        k<<<ctas, 256, 200 * 1024>>>(src, dst, mode, bytes, chunk, inflight, out);
                        cudaMemcpy(h, out, ctas * 8, cudaMemcpyDeviceToHost);
                        double mx = 0;
                        for (int c = 0; c < ctas; ++c) mx = h[c] > mx ? h[c] : mx;
                        best = mx < best ? mx : best;
                    }
                    printf("%-16s ctas %3d bytes/CTA %7d chunk %6d: %7.2f us  %7.1f GB/s per CTA\n", names[mode], ctas,
                           bytes, chunk, best / 1e3, bytes / best);
                }
            }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
}
