// Shared device helpers for libf3d (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/f3d.h"

#define F3D_CUDA_TRY(expr)                                  \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) {                            \
            f3d_set_last_cuda_error(_e);                    \
            return F3D_ERR_CUDA;                            \
        }                                                   \
    } while (0)

#define F3D_LAUNCH_CHECK() F3D_CUDA_TRY(cudaGetLastError())

void f3d_set_last_cuda_error(cudaError_t e);
int f3d_num_sms();
// Zero n int32 words with a kernel: a memset node in a CUDA graph may run on a
// copy engine and then queues behind concurrent H2D/D2H traffic (measured:
// 40 us stalls per step in the pipelined host loop).
cudaError_t f3d_zero_i32(int32_t* p, int64_t n, cudaStream_t st);

namespace f3d {

constexpr int kWarp = 32;

// hash kinds: hashing.py:19 HASH_KINDS order
enum HashKind : int { XOR_MOD = 0, XOR_DIV = 1, ZORDER_MOD = 2, ZORDER_DIV = 3 };

// Place bit k of a (< 2^21) at bit 3k — magic-number bit spread.
__host__ __device__ __forceinline__ uint64_t spread3(uint64_t a) {
    a &= 0x1FFFFFull;
    a = (a | (a << 32)) & 0x1F00000000FFFFull;
    a = (a | (a << 16)) & 0x1F0000FF0000FFull;
    a = (a | (a << 8)) & 0x100F00F00F00F00Full;
    a = (a | (a << 4)) & 0x10C30C30C30C30C3ull;
    a = (a | (a << 2)) & 0x1249249249249249ull;
    return a;
}

// _kernels.py:17-24: x at bit 3k, y at 3k+1, z at 3k+2 (inputs < 2^bits).
__host__ __device__ __forceinline__ int64_t morton3(int64_t x, int64_t y, int64_t z) {
    return (int64_t)(spread3((uint64_t)x) | (spread3((uint64_t)y) << 1) |
                     (spread3((uint64_t)z) << 2));
}

// 10-bit fast path: 30-bit code in 32-bit arithmetic.
__host__ __device__ __forceinline__ uint32_t spread3_10(uint32_t a) {
    a &= 0x3FFu;
    a = (a | (a << 16)) & 0x030000FFu;
    a = (a | (a << 8)) & 0x0300F00Fu;
    a = (a | (a << 4)) & 0x030C30C3u;
    a = (a | (a << 2)) & 0x09249249u;
    return a;
}

struct HashParams {
    int kind;
    int K;
    int64_t S_div;
    int bits;
    int strict;
};

// _kernels.py:27-38: bucket id, or -1 when strict div rejects the quotient.
__device__ __forceinline__ int hash_bucket1(int x, int y, int z, const HashParams& hp) {
    int64_t key;
    if (hp.kind <= XOR_DIV) {
        key = (int64_t)(x ^ y ^ z);
    } else if (hp.bits <= 10) {
        key = (int64_t)(spread3_10(x) | (spread3_10(y) << 1) | (spread3_10(z) << 2));
    } else {
        key = morton3(x, y, z);
    }
    if (hp.kind == XOR_DIV || hp.kind == ZORDER_DIV) {
        if (key < 0x7FFFFFFFll && hp.S_div < 0x7FFFFFFFll) {
            key = (int64_t)((uint32_t)key / (uint32_t)hp.S_div);
        } else {
            key = key / hp.S_div;
        }
        if (hp.strict && key >= hp.K) return -1;
    }
    if (key < 0x7FFFFFFFll) return (int)((uint32_t)key % (uint32_t)hp.K);
    return (int)(key % hp.K);
}

// Packed fp32 pairs (sm_100 FFMA2/FADD2/FMUL2: two lanes' worth of fp32 math
// per issue slot; softmax and GELU are issue-bound).
__device__ __forceinline__ uint64_t f2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2_split(uint64_t v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

inline int cdiv(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }
__device__ __forceinline__ int cdiv_dev(int a, int b) { return (a + b - 1) / b; }

// Row count of a launch sized for capacity n: min(n, *n_dev) when the count
// lives on the device (sync-free / graph-captured pipelines), else n.
__device__ __forceinline__ int64_t dyn_n(int64_t n, const int32_t* n_dev) {
    if (n_dev == nullptr) return n;
    const int64_t d = *n_dev;
    return d < n ? (d < 0 ? 0 : d) : n;
}

}  // namespace f3d
