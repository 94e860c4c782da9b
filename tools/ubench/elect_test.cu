#include <cstdio>
#include "../../paper_2412_16481_b200/csrc/tc_common.cuh"
using namespace f3d::tc;
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
    return pred != 0;
}
__global__ void k(const int* __restrict__ work, int n, uint32_t tmem, uint32_t sm) {
    const uint64_t dK = smem_desc(sm, 128, 2048), dQ = smem_desc(sm + 65536, 128, 2048);
    int kv = 0;
    for (int item = 0; item < n; ++item) {
        const int nt = __ldg(work + item);
        for (int j = 0; j < nt; ++j, ++kv) {
            const uint32_t s = kv % 5;
            const uint64_t dk = dK + (uint64_t)(s * 2048);
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    umma_f16(tmem + (j & 1) * 64, dQ + 16 * kk, dk + 16 * kk, idesc_bf16(128, 64, 0, 0), kk > 0);
            }
            __syncwarp();
        }
    }
}
