// Microbenchmark: is small-N tcgen05.mma bound by the shared-memory operand
// reads (A 4 KB + B N*32 B per M128 K16 instruction at ~128 B/clk) or by a
// fixed per-instruction cost?  SS (A and B from smem) vs TS (A from TMEM),
// N = 32 / 64 / 128, one or two issuing warps (independent accumulators).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o mma_ts mma_ts.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2412_16481_b200/csrc/tc_common.cuh"
using namespace f3d::tc;

template <int N, int CH, int TS, int NI>
__global__ void k(long long* out, int iters) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar[2];
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_mbar_init(); }
    if (threadIdx.x < 32) { tmem_alloc(&slot, 512); tmem_relinquish(); }
    fence_proxy_async(); tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t a = saddr(sm), b = saddr(sm) + 32768;
    const int w = threadIdx.x >> 5;
    if (w < NI && (threadIdx.x & 31) == 0) {
        constexpr uint32_t id = idesc_bf16(128, N, 0, 0);
        const uint64_t da = smem_desc(a + w * 8192, 128, 512), db = smem_desc(b + w * 8192, 128, 256);
        // accumulators: issuer w uses columns [w*256, w*256 + CH*N) (CH*N <= 224 for TS: A at 224..255)
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const uint32_t d = tmem + w * 256 + c * N;
                if (TS) umma_f16_ts(d, tmem + w * 256 + 248, db, id, 1);
                else umma_f16(d, da, db, id, 1);
            }
        }
        umma_commit(&bar[w]);
        mbar_wait(&bar[w], 0);
        long long t1 = clock64();
        out[w] = t1 - t0;
    }
    tc_fence_before(); __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int N, int CH, int TS, int NI>
void run() {
    long long* d; cudaMalloc(&d, 16);
    auto kern = k<N, CH, TS, NI>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const int iters = 512;
    kern<<<1, 128, 65536>>>(d, iters);
    kern<<<1, 128, 65536>>>(d, iters);
    long long h[2] = {0, 0}; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    const long long t = h[0] > h[1] ? h[0] : h[1];
    const double per = (double)t / (iters * CH * NI);      // SM clk per MMA (all issuers)
    printf("%s N=%3d chains=%d issuers=%d: %6.1f clk/mma per SM  %6.0f flop/clk (%s)\n", TS ? "TS" : "SS", N, CH,
           NI, per, 2.0 * 128 * N * 16 / per, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<32, 4, 0, 1>(); run<32, 4, 1, 1>(); run<32, 4, 0, 2>(); run<32, 4, 1, 2>();
    run<64, 3, 0, 1>(); run<64, 3, 1, 1>(); run<64, 3, 0, 2>(); run<64, 3, 1, 2>();
    run<128, 1, 0, 1>(); run<128, 1, 1, 1>(); run<128, 1, 0, 2>(); run<128, 1, 1, 2>();
    run<16, 8, 0, 1>(); run<16, 8, 1, 1>();
    return 0;
}
