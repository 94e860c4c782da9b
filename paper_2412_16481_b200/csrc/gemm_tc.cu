// Stage projections on 5th-generation tensor cores (bw/stage.py:135-138, 146-158):
//
//     Y[n x N] = X[n x K] W[K x N] + bias        (optionally GELU-erf, bf16 out)
//
// the QKV, O and MLP GEMMs of a round (replacing the library GEMMs).  One
// persistent CTA per SM walks (128-row block, BN-column tile) work items:
//   * warp 0 streams X and W^T k-blocks by TMA (K-major, 128/64-byte swizzle)
//     through an S-deep ring of shared-memory stages;
//   * warp 1 (one elected lane) issues tcgen05.mma M=128 N=BN K=16 into one
//     of two TMEM accumulators (2 x BN <= 512 columns), so the next tile's
//     MMAs overlap this tile's epilogue;
//   * two epilogue warpgroups split the tile's columns: tcgen05.ld 16 columns
//     at a time (the next chunk's load in flight), + bias (+ packed-pair GELU),
//     bf16, staged in shared memory (padded rows: conflict-free), released
//     TMEM, then coalesced 16-byte stores of whole row segments.
// N is split into equal tiles of at most 256 columns (a multiple of 16);
// K is a multiple of 32 (BK = 64 with 128-byte swizzle when K % 64 == 0,
// else BK = 32 with 64-byte swizzle).  Rows past n (device count n_dev) are
// computed from whatever the buffer holds and never stored.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>

#include "f3d_common.cuh"
#include "tc_common.cuh"

namespace f3d {
namespace gm {

using namespace f3d::tc;

constexpr int kBM = 128;
constexpr int kThreads = 384;      // warp 0 TMA, warp 1 MMA, warps 4-11 epilogue (2 WGs)
constexpr int kMaxStages = 8;
constexpr int kSmemLimit = 227 * 1024;

struct Args {
    int64_t n;
    const int32_t* n_dev;
    int K, N, BN, nt, S, csplit;
    const float* bias;       // (N) fp32, nullable
    int gelu;
    __nv_bfloat16* y;
    int64_t ldy;
    // shared-memory layout (bytes from the 1024-aligned base)
    int off_stage, stage_bytes, a_bytes, off_st0, off_st1, st_stride0, st_stride1, off_bias,
        off_bar;
};

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int BK>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const Args A, const __grid_constant__ CUtensorMap amap,
                const __grid_constant__ CUtensorMap bmap) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem =
        (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);   // swizzle atoms
    const int S = A.S, BN = A.BN;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + A.off_bar);
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* acc_full = bars + 2 * S;
    uint64_t* acc_empty = acc_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
    float* s_bias = reinterpret_cast<float*>(smem + A.off_bias);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t n = dyn_n(A.n, A.n_dev);
    const int mblocks = (int)((n + kBM - 1) / kBM);
    const int ntiles = mblocks * A.nt;
    const int nk = A.K / BK;

    for (int i = tid; i < A.N; i += kThreads) s_bias[i] = A.bias ? A.bias[i] : 0.f;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(acc_full + b, 1);
            mbar_init(acc_empty + b, 256);
        }
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sbase = saddr(smem);

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        int kc = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int m = t / A.nt, j = t - m * A.nt;
            for (int ks = 0; ks < nk; ++ks, ++kc) {
                const int s = kc % S;
                if (kc >= S) mbar_wait(empty + s, ((kc / S) - 1) & 1);
                if (lane == 0) {
                    const uint32_t dst = sbase + A.off_stage + s * A.stage_bytes;
                    mbar_arrive_expect(full + s, A.stage_bytes);
                    tma_2d(dst, &amap, full + s, ks * BK, m * kBM);
                    tma_2d(dst + A.a_bytes, &bmap, full + s, ks * BK, j * BN);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        constexpr uint32_t kLt = BK == 64 ? 2u : 4u;          // SWIZZLE_128B / SWIZZLE_64B
        constexpr uint32_t kSbo = BK == 64 ? 1024u : 512u;    // 8 rows x row bytes
        const uint32_t idesc = idesc_bf16(kBM, BN, 0, 0);
        int kc = 0, it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int buf = it & 1;
            if (it >= 2) mbar_wait(acc_empty + buf, ((it >> 1) - 1) & 1);
            tc_fence_after();
            const uint32_t d = tmem + buf * BN;
            for (int ks = 0; ks < nk; ++ks, ++kc) {
                const int s = kc % S;
                mbar_wait(full + s, (kc / S) & 1);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t a0 = sbase + A.off_stage + s * A.stage_bytes;
                    const uint64_t da = sw_desc(a0, 16, kSbo, kLt);
                    const uint64_t db = sw_desc(a0 + A.a_bytes, 16, kSbo, kLt);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk)      // +32 B per K=16 step
                        umma_f16(d, da + (uint64_t)(2 * kk), db + (uint64_t)(2 * kk), idesc,
                                 (ks | kk) != 0);
                    umma_commit(empty + s);
                }
                __syncwarp();
            }
            if (elect_one()) umma_commit(acc_full + buf);
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue
        const int g = (warp >> 2) - 1;                         // warpgroup 0 / 1
        const int c_lo = g == 0 ? 0 : A.csplit, c_hi = g == 0 ? A.csplit : BN;
        const int stride = g == 0 ? A.st_stride0 : A.st_stride1;
        unsigned char* stage = smem + (g == 0 ? A.off_st0 : A.off_st1);
        const int r = (warp & 3) * 32 + lane;                  // tile row = TMEM lane
        const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
        unsigned char* strow = stage + r * stride;
        const int chunks = (c_hi - c_lo) / 8;                  // 16-byte chunks per row
        const int tq = tid & 127;
        int it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int m = t / A.nt, j = t - m * A.nt;
            const int buf = it & 1;
            mbar_wait(acc_full + buf, (it >> 1) & 1);
            tc_fence_after();
            const uint32_t c0 = tmem + lb + buf * BN;
            const float* bj = s_bias + j * BN;
            if (c_hi > c_lo) {
                uint32_t v[16], nv[16];
                tmem_ld16(c0 + c_lo, v);
                tmem_wait_ld();
#pragma unroll 1
                for (int cc = c_lo; cc < c_hi; cc += 16) {
                    const bool more = cc + 16 < c_hi;
                    if (more) tmem_ld16(c0 + cc + 16, nv);     // next chunk in flight
                    uint32_t pk[8];
#pragma unroll
                    for (int e = 0; e < 16; e += 2) {
                        float2 f = make_float2(__uint_as_float(v[e]) + bj[cc + e],
                                               __uint_as_float(v[e + 1]) + bj[cc + e + 1]);
                        if (A.gelu) f = gelu2(f.x, f.y);
                        __nv_bfloat162 h2 = __floats2bfloat162_rn(f.x, f.y);
                        pk[e >> 1] = *reinterpret_cast<uint32_t*>(&h2);
                    }
                    uint4* dst = reinterpret_cast<uint4*>(strow + (cc - c_lo) * 2);
                    dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                    dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                    if (more) {
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 16; ++e) v[e] = nv[e];
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(acc_empty + buf);                      // accumulator free
            named_bar(1 + g, 128);                             // staging tile complete
            const int64_t r0 = (int64_t)m * kBM;
            __nv_bfloat16* yb = A.y + j * BN + c_lo;
            for (int i = tq; i < kBM * chunks; i += 128) {
                const int rr = i / chunks, ch = i - rr * chunks;
                if (r0 + rr < n)
                    *reinterpret_cast<uint4*>(yb + (r0 + rr) * A.ldy + ch * 8) =
                        *reinterpret_cast<const uint4*>(stage + rr * stride + ch * 16);
            }
            named_bar(1 + g, 128);                             // staging free again
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

struct Plan {
    int BK, BN, nt, S, csplit;
    Args a;
    size_t smem;
};

static bool plan(int K, int N, Plan& p) {
    if (K < 32 || K % 32 || N < 16 || N % 16 || N > 4096) return false;
    p.BK = (K % 64 == 0) ? 64 : 32;
    int nt = (N + 255) / 256;
    while (nt <= N / 16 && (N % nt || (N / nt) % 16)) ++nt;
    if (nt > N / 16) return false;
    p.nt = nt;
    p.BN = N / nt;
    p.csplit = std::min(p.BN, ((p.BN / 2 + 15) / 16) * 16);
    Args& a = p.a;
    a.K = K;
    a.N = N;
    a.BN = p.BN;
    a.nt = nt;
    a.csplit = p.csplit;
    a.a_bytes = kBM * p.BK * 2;
    a.stage_bytes = (kBM + p.BN) * p.BK * 2;
    a.st_stride0 = p.csplit * 2 + 16;
    a.st_stride1 = (p.BN - p.csplit) * 2 + 16;
    const int staging = kBM * (a.st_stride0 + a.st_stride1);
    const int fixed = 1024 /* base alignment */ + staging + ((N * 4 + 15) & ~15) + 256;
    const int S = std::min(kMaxStages, (kSmemLimit - fixed) / a.stage_bytes);
    if (S < 2) return false;
    p.S = a.S = S;
    a.off_stage = 0;
    a.off_st0 = S * a.stage_bytes;
    a.off_st1 = a.off_st0 + kBM * a.st_stride0;
    a.off_bias = a.off_st1 + kBM * a.st_stride1;
    a.off_bar = (a.off_bias + N * 4 + 15) & ~15;
    p.smem = (size_t)a.off_bar + (2 * S + 4) * 8 + 16 + 1024;
    return p.smem <= (size_t)kSmemLimit;
}

}  // namespace gm
}  // namespace f3d

using namespace f3d;

extern "C" int f3d_gemm_supported(int K, int N) {
    gm::Plan p;
    return gm::plan(K, N, p) ? 1 : 0;
}

extern "C" int f3d_gemm(const void* x, int64_t ldx, int64_t n, int K, const void* w_t, int N,
                        const float* bias, int gelu, void* y, int64_t ldy, const int32_t* n_dev,
                        void* stream) {
    gm::Plan p;
    if (!gm::plan(K, N, p) || n < 0 || (ldx & 7) || (ldy & 7) || ldx < K || ldy < N ||
        (((uintptr_t)x | (uintptr_t)w_t | (uintptr_t)y) & 15))
        return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    cudaStream_t st = (cudaStream_t)stream;
    CUtensorMap amap, bmap;
    memset(&amap, 0, sizeof(amap));
    memset(&bmap, 0, sizeof(bmap));
    const int sw = p.BK * 2;
    if (!tc::make_map(&amap, x, ldx, K, n, p.BK, sw, gm::kBM) ||
        !tc::make_map(&bmap, w_t, K, K, N, p.BK, sw, p.BN)) {
        f3d_set_last_cuda_error(cudaErrorNotSupported);
        return F3D_ERR_CUDA;
    }
    gm::Args a = p.a;
    a.n = n;
    a.n_dev = n_dev;
    a.bias = bias;
    a.gelu = gelu;
    a.y = (__nv_bfloat16*)y;
    a.ldy = ldy;
    auto kern = p.BK == 64 ? gm::gemm_kernel<64> : gm::gemm_kernel<32>;
    static int attr[2] = {0, 0};
    int& at = attr[p.BK == 64];
    if ((int)p.smem > at) {
        F3D_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)p.smem));
        at = (int)p.smem;
    }
    const int64_t tiles = ((n + gm::kBM - 1) / gm::kBM) * p.nt;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, f3d_num_sms()));
    kern<<<grid, gm::kThreads, p.smem, st>>>(a, amap, bmap);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}
