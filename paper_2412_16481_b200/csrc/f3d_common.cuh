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
cudaError_t f3d_zero_i32x2(int32_t* p, int n, int32_t* q, int m, cudaStream_t st);   // n, m <= 32
// Programmatic dependent launch (F3D_PDL, default on): the hot-path kernels
// are launched with programmatic stream serialisation, so a kernel's CTAs are
// scheduled (and run their prologue: barriers, TMEM, smem set-up) while the
// previous kernel's last CTAs finish; each such kernel executes
// f3d::pdl_wait() before its first global read of anything a predecessor
// wrote.  (In a kernel launched without the attribute the wait is a no-op.)
bool f3d_pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t f3d_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = f3d_pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

namespace f3d {

constexpr int kWarp = 32;

// wait for the grids this one programmatically depends on (griddepcontrol)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

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

// floor(RN(RN(c - o) / vs)) -- numpy's floor((c - o) / voxel) -- with the
// division off the common path: q = RN(x * RN(1/vs)) lies within 1.5 ulp of the
// rounded quotient, so when q's fractional part is farther than 2^-40 (|q| + 1)
// from 0 and 1, the rounded quotient has the same floor as q; otherwise (a
// quotient within ~1e-12 of an integer, |q| >= 2^52, non-finite) the exact
// IEEE division decides.  inv = __drcp_rn(vs), once per thread.
__device__ __forceinline__ long long vox_floor_inv(double c, double o, double vs, double inv) {
    const double x = __dsub_rn(c, o);
    const double q = __dmul_rn(x, inv);
    const double f = floor(q);
    const double fr = __dsub_rn(q, f);
    const double tol = __fma_rn(fabs(q), 0x1p-40, 0x1p-40);
    if (fr > tol && fr < 1.0 - tol) return (long long)f;
    return (long long)floor(__ddiv_rn(x, vs));
}

// Division by a run-time constant d in [1, 2^31) for dividends n < 2^31:
// q = umulhi(n, m) >> s with m = ceil(2^(31+L) / d), s = L - 1, L = ceil(log2 d)
// (the round-up method; exact for every n < 2^31), d = 1 handled as m = 0.
struct FastDiv {
    uint32_t d, m, s;
    __host__ __device__ static FastDiv make(uint32_t d) {
        FastDiv f{d, 0u, 0u};
        if (d > 1) {
            uint32_t L = 0;
            while ((1ull << L) < d) ++L;
            f.m = (uint32_t)(((1ull << (31 + L)) + d - 1) / d);
            f.s = L - 1;
        }
        return f;
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        return m ? (__umulhi(n, m) >> s) : n;
    }
    __device__ __forceinline__ uint32_t mod(uint32_t n) const { return n - div(n) * d; }
};

struct HashParams {
    int kind;
    int K;
    int64_t S_div;
    int bits;
    int strict;
    FastDiv fdiv, fk;   // S_div and K (set by hash_params)
};

__host__ __device__ inline HashParams hash_params(int kind, int K, int64_t S_div, int bits,
                                                  int strict) {
    HashParams hp{kind, K, S_div, bits, strict, FastDiv::make(1u), FastDiv::make((uint32_t)K)};
    if (S_div < 0x7FFFFFFFll) hp.fdiv = FastDiv::make((uint32_t)S_div);
    return hp;
}

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
            key = (int64_t)hp.fdiv.div((uint32_t)key);
        } else {
            key = key / hp.S_div;
        }
        if (hp.strict && key >= hp.K) return -1;
    }
    if (key < 0x7FFFFFFFll) return (int)hp.fk.mod((uint32_t)key);
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

// GELU, exact-erf form (bw/stage.py:91-92), on a packed pair: erf via
// Abramowitz & Stegun 7.1.26 (|error| <= 1.5e-7, below the bf16 rounding of
// the result), MUFU rcp/ex2, the FMA/FMUL work issued as f32x2.  Written as
//   GELU(x) = 0.5 (x + |x|) + 0.5 |x| (erf(|x|/sqrt2) - 1)
// (x erf(x/sqrt2) = |x| erf(|x|/sqrt2)): no sign transfer, and for x < 0 the
// result is a single product (0.5 (x + |x|) = 0 exactly) instead of the
// difference 1 - erf of two numbers near 1.
__device__ __forceinline__ float2 gelu2(float x0, float x1) {
    const uint64_t ax = f2(fabsf(x0), fabsf(x1));
    // z = |x| / sqrt2 enters only as p z and z^2: both constants folded in
    // (p / sqrt2 = 0.2316418883, log2(e) / 2)
    float d0, d1, t0, t1;
    f2_split(ffma2(f2(0.23164188826636f, 0.23164188826636f), ax, f2(1.f, 1.f)), d0, d1);
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t0) : "f"(d0));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t1) : "f"(d1));
    const uint64_t t = f2(t0, t1);
    // pn = -(a1 t + ... + a5 t^5)
    uint64_t pn = ffma2(f2(-1.061405429f, -1.061405429f), t, f2(1.453152027f, 1.453152027f));
    pn = ffma2(pn, t, f2(-1.421413741f, -1.421413741f));
    pn = ffma2(pn, t, f2(0.284496736f, 0.284496736f));
    pn = ffma2(pn, t, f2(-0.254829592f, -0.254829592f));
    pn = fmul2(pn, t);
    float a0, a1, e0, e1;
    f2_split(fmul2(fmul2(ax, ax), f2(-0.7213475204444817f, -0.7213475204444817f)), a0, a1);
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(a0));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(a1));
    const uint64_t rneg = fmul2(pn, f2(e0, e1));          // erf(|x|/sqrt2) - 1
    const uint64_t h = fmul2(ax, f2(0.5f, 0.5f));
    const uint64_t base = ffma2(f2(0.5f, 0.5f), f2(x0, x1), h);   // 0.5 (x + |x|)
    float o0, o1;
    f2_split(ffma2(h, rneg, base), o0, o1);
    return make_float2(o0, o1);
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
