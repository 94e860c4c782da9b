// Microbenchmark: tcgen05.mma issue-to-completion cost for attention-sized
// shapes (M=128, K=16 bf16), dependent chains vs independent accumulators.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o mma_lat mma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2412_16481_b200/csrc/tc_common.cuh"
using namespace f3d::tc;

template <int N, int CHAINS>
__global__ void k(long long* out, int iters, int ts) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (threadIdx.x < 32) { tmem_alloc(&slot, 512); tmem_relinquish(); }
    fence_proxy_async(); tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t a = saddr(sm), b = saddr(sm) + 32768;
    if (threadIdx.x == 0) {
        constexpr uint32_t id = idesc_bf16(128, N, 0, 0);
        long long t0 = clock64();
        const uint64_t da = smem_desc(a, 128, 512), db = smem_desc(b, 128, 256);
        if (ts == 2) {
            for (int it = 0; it < iters; ++it) {
#pragma unroll
                for (int c = 0; c < CHAINS; ++c) umma_f16(tmem + c * N, da, db, id, 1);
            }
        } else
        for (int it = 0; it < iters; ++it) {
            for (int c = 0; c < CHAINS; ++c) {
                const uint32_t d = tmem + (ts ? 0 : c * N);
                if (ts) umma_f16_ts(tmem + 256 + c * 8 % 256, tmem + (c * 32) % 128, smem_desc(b, 128, 256), id, 1);
                else umma_f16(d, smem_desc(a + (c % 4) * 256, 128, 512), smem_desc(b, 128, 256), id, 1);
            }
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        out[0] = t1 - t0;
    }
    tc_fence_before(); __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int N, int CH>
void run(const char* name, int ts) {
    long long* d; cudaMalloc(&d, 8);
    auto kern = k<N, CH>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const int iters = 256;
    kern<<<1, 128, 65536>>>(d, iters, ts);
    kern<<<1, 128, 65536>>>(d, iters, ts);
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    const double per = (double)h / (iters * CH);
    const double flop = 2.0 * 128 * N * 16;
    printf("%-28s N=%3d chains=%d: %7.1f clk/mma  %6.0f flop/clk (%s)\n", name, N, CH, per, flop / per, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<64, 4>("SS hoisted desc", 2);
    run<64, 8>("SS hoisted desc", 2);
    run<128, 4>("SS hoisted desc", 2);
    run<256, 2>("SS hoisted desc", 2);
    run<32, 8>("SS hoisted desc", 2);
    run<64, 1>("SS dependent (same D)", 0);
    run<64, 4>("SS 4 independent D", 0);
    run<128, 1>("SS dependent", 0);
    run<128, 4>("SS 4 independent D", 0);
    run<256, 1>("SS dependent", 0);
    run<256, 2>("SS 2 independent D", 0);
    run<32, 1>("SS dependent", 0);
    run<32, 4>("SS 4 independent", 0);
    run<32, 4>("TS (A in TMEM)", 1);
    run<128, 4>("TS (A in TMEM)", 1);
    run<64, 4>("TS (A in TMEM)", 1);
    return 0;
}
