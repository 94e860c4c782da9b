// Microbenchmark: issue cost of 2-SM tcgen05.mma (cta_group::2, M = 256)
// against the 1-SM M = 128 instruction (mma_lat.cu), K = 16 bf16: the question
// for small-head attention is whether an M=256 pair instruction costs about
// the same as an M=128 one (halving MMA issue per score).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o mma2_lat mma2_lat.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2412_16481_b200/csrc/tc_common.cuh"
using namespace f3d::tc;

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N, int CHAINS>
__global__ void __cluster_dims__(2, 1, 1) k2(long long* out, int iters) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&slot)), "r"(512) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    fence_proxy_async(); tc_fence_before(); __syncthreads(); tc_fence_after();
    cluster_sync_all();
    const uint32_t tmem = slot;
    const uint32_t a = saddr(sm), b = saddr(sm) + 32768;
    if (cta_rank() == 0 && threadIdx.x == 0) {
        constexpr uint32_t id = idesc_bf16(256, N, 0, 0);
        const uint64_t da = smem_desc(a, 128, 512), db = smem_desc(b, 128, 256);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int c = 0; c < CHAINS; ++c)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(tmem + c * N), "l"(da), "l"(db), "r"(id), "r"(1u) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(saddr(&bar)), "h"((unsigned short)3) : "memory");
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        out[0] = t1 - t0;
    }
    if (cta_rank() == 1 && threadIdx.x == 0) mbar_wait(&bar, 0);   // the multicast arrive lands here too
    tc_fence_before(); __syncthreads();
    cluster_sync_all();
    if (threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

template <int N, int CH>
void run() {
    long long* d; cudaMalloc(&d, 8);
    auto kern = k2<N, CH>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const int iters = 256;
    kern<<<2, 128, 65536>>>(d, iters);
    kern<<<2, 128, 65536>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double per = (double)h / (iters * CH);
    const double flop = 2.0 * 256 * N * 16;
    printf("cta_group::2 M=256 N=%3d chains=%d: %7.1f clk/mma  %6.0f flop/clk per pair (%s)\n", N, CH, per, flop / per, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<64, 4>();
    run<64, 8>();
    run<32, 8>();
    run<128, 4>();
    run<256, 2>();
    return 0;
}
