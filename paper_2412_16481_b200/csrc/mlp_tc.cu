// Fused stage MLP on 5th-generation tensor cores (bw/stage.py:146-158):
//
//     F[r] += gelu(x[r] W_in + b_in) W_out + b_out
//     x_next[r] = LN1(F[r]) * g + b + PE(coords[r])      (optional: next round)
//
// One persistent CTA per SM walks 128-row tiles.  W_in^T and W_out^T stay in
// shared memory for the whole launch (K-major UMMA operands, SWIZZLE_NONE
// core-matrix layout); x tiles are double-buffered with cp.async.
//   * warp 0 loads x tiles; warp 1 (one elected lane) issues tcgen05.mma:
//     GEMM1 D1[128 x 4d] = X W_in (three N = 4d/3 parts) into TMEM, then
//     GEMM2 D2[128 x d] = G W_out with G read from TMEM (TS MMA);
//   * three epilogue warpgroups, one per part of D1's columns: +b_in,
//     exact-erf GELU (Abramowitz-Stegun 7.1.26, |err| <= 1.5e-7), bf16 pairs
//     packed in place (part p: columns [p*4d/3, +4d/3) -> [p*4d/3, +2d/3)), so
//     GEMM2 reads G from TMEM without an HBM round trip of the hidden rows;
//   * the three warpgroups then stage D2 (bf16, as the unfused GEMM output) in
//     shared memory and run the row epilogue with lanes over columns: F += y +
//     b_out in fp32, LayerNorm + PE of the updated row for the next round.
// The hidden columns are split in thirds (one epilogue warpgroup each, GEMM2
// k-steps of a third issued as soon as it is packed).
// TMEM: D1 at columns [0, 4d), D2 at [4d, 5d); 5d <= 512 (d <= 96 here).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>
#include <cfloat>

#include "f3d_common.cuh"
#include "tc_common.cuh"

namespace f3d {
namespace mlp {

using namespace f3d::tc;

constexpr int kBM = 128;
constexpr int kParts = 3;                  // hidden columns split in thirds, one epilogue WG each
constexpr int kThreads = (1 + kParts) * 128;   // WG0: loader (warp 0) + MMA (warp 1)

template <int D>
struct Cfg {
    static constexpr int H = 4 * D;                       // hidden width
    static constexpr int HP = H / kParts;                 // hidden columns per part
    static constexpr int kWinBytes = H * D * 2;           // W_in^T  (H rows x D cols)
    static constexpr int kWoutBytes = D * H * 2;          // W_out^T (D rows x H cols)
    static constexpr int kXBytes = kBM * D * 2;           // one x tile
    static constexpr int kOffWin = 0;
    static constexpr int kOffWout = kOffWin + kWinBytes;
    static constexpr int kOffX = kOffWout + kWoutBytes;   // 2 buffers
    static constexpr int kYStride = 2 * D + 16;            // y tile row stride (bytes, padded)
    static constexpr int kOffY = kOffX + 2 * kXBytes;     // y = D2 rounded to bf16, 128 rows
    static constexpr int kOffBias = kOffY + kBM * kYStride;   // b_in (H) + b_out (D) floats
    static constexpr int kOffBar = kOffBias + (H + D) * 4;
    static constexpr int kNumBars = 2 + 2 + 2 * kParts + 1;   // x_full[2], x_empty[2], d1[P], g[P], d2
    static constexpr int kSmem = kOffBar + kNumBars * 8 + 16;
    static constexpr int kTmemD2 = H;
    static_assert(5 * D <= 512, "TMEM: D1 (4d) + D2 (d) columns");
    static_assert(HP % 32 == 0 && HP <= 256 && D % 32 == 0, "column chunks / MMA N");
    static_assert(kSmem <= 227 * 1024, "smem budget");
};

// byte offset of 16-byte chunk c of row r in an R x C core-matrix tile
template <int C>
__device__ __forceinline__ uint32_t core_off(int r, int c) {
    return (uint32_t)((r >> 3) * (16 * C) + c * 128 + (r & 7) * 16);
}

struct Args {
    const __nv_bfloat16* x;
    int64_t ldx;
    int64_t n;
    const int32_t* n_dev;
    const __nv_bfloat16* w_in_t;    // (4d, d) row-major = W_in^T
    const float* b_in;              // (4d)
    const __nv_bfloat16* w_out_t;   // (d, 4d) row-major = W_out^T
    const float* b_out;             // (d)
    float* F;
    int64_t ldf;
    const float* ln_g;              // LN of the updated row (nullable: no x_next)
    const float* ln_b;
    const double* pec;              // PE coordinates (nullable)
    const double* lo_ext;
    float pl2;                      // log2(pe base)
    __nv_bfloat16* x_next;
    int64_t ldxn;
    float eps;
};

__device__ __forceinline__ float gelu_as(float x) {
    const float z = fabsf(x) * 0.70710678118654752f;
    float t;   // MUFU reciprocal / exp2 (approx): 1-2 ulp, far inside the 1.5e-7 formula error
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, z, 1.f)));
    float pl = fmaf(1.061405429f, t, -1.453152027f);
    pl = fmaf(pl, t, 1.421413741f);
    pl = fmaf(pl, t, -0.284496736f);
    pl = fmaf(pl, t, 0.254829592f);
    pl *= t;
    float ez;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ez) : "f"(-z * z * 1.4426950408889634f));
    const float e = 1.f - pl * ez;
    return 0.5f * x * (1.f + copysignf(e, x));
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Rows [r0, r0+128) of the tile: epilogue warp w (0..11) takes blocks of 8 rows (all loads of a
// block in flight before its reductions); lane q owns
// columns [4q, 4q+4) (q < D/4).  F += y + b_out (fp32); x_next = LN(F)*g + b
// (+ PE) in bf16 -- the arithmetic of f3d_row_ln (bw/stage.py:84-88, 157-158).
template <int D>
__device__ __forceinline__ void row_epilogue(const Args& A, const unsigned char* ytile,
                                             const float* s_bout, int64_t r0, int64_t n, int w,
                                             int lane) {
    constexpr int kYStride = 2 * D + 16;
    const bool act = lane < D / 4;
    const int c0 = 4 * lane;
    const float4 bo = act ? *reinterpret_cast<const float4*>(s_bout + c0) : make_float4(0, 0, 0, 0);
    float4 gg = make_float4(0, 0, 0, 0), bb = gg;
    if (A.x_next && act) {
        gg = __ldg(reinterpret_cast<const float4*>(A.ln_g + c0));
        bb = __ldg(reinterpret_cast<const float4*>(A.ln_b + c0));
    }
    constexpr int npair = D / 6, blk = 2 * npair;
    int pa[2], pj[2];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const int c = c0 + 2 * p;
        pa[p] = c / blk;
        pj[p] = (c - pa[p] * blk) >> 1;
    }
    constexpr int RB = 8;                        // rows in flight per warp
#pragma unroll 1
    for (int rb = w * RB; rb < kBM; rb += kParts * 4 * RB) {
        float4 v[RB];
        double pc[RB][3];
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            const int64_t row = r0 + rb + i;
            const bool ok = act && row < n;
            v[i] = ok ? *reinterpret_cast<const float4*>(A.F + row * A.ldf + c0) : make_float4(0, 0, 0, 0);
            if (A.pec && A.x_next)
#pragma unroll
                for (int a = 0; a < 3; ++a) pc[i][a] = row < n ? A.pec[3 * row + a] : 0.0;
        }
        float s[RB], q[RB];
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            const int64_t row = r0 + rb + i;
            if (act) {
                const uint2 yy = *reinterpret_cast<const uint2*>(ytile + (rb + i) * kYStride + c0 * 2);
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&yy);
                const float2 y01 = __bfloat1622float2(h[0]), y23 = __bfloat1622float2(h[1]);
                v[i].x += y01.x + bo.x;
                v[i].y += y01.y + bo.y;
                v[i].z += y23.x + bo.z;
                v[i].w += y23.y + bo.w;
                if (row < n) *reinterpret_cast<float4*>(A.F + row * A.ldf + c0) = v[i];
            }
            s[i] = (v[i].x + v[i].y) + (v[i].z + v[i].w);
        }
        if (!A.x_next) continue;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int i = 0; i < RB; ++i) s[i] += __shfl_xor_sync(0xffffffffu, s[i], o);
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            const float m = s[i] * (1.f / D);
            const float a = act ? v[i].x - m : 0.f, b = act ? v[i].y - m : 0.f;
            const float c = act ? v[i].z - m : 0.f, e = act ? v[i].w - m : 0.f;
            q[i] = (a * a + b * b) + (c * c + e * e);
            s[i] = m;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int i = 0; i < RB; ++i) q[i] += __shfl_xor_sync(0xffffffffu, q[i], o);
        if (!act) continue;
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            const int64_t row = r0 + rb + i;
            if (row >= n) break;
            const float m = s[i];
            const float rstd = rsqrtf(q[i] * (1.f / D) + A.eps);
            float o0 = (v[i].x - m) * rstd * gg.x + bb.x, o1 = (v[i].y - m) * rstd * gg.y + bb.y;
            float o2 = (v[i].z - m) * rstd * gg.z + bb.z, o3 = (v[i].w - m) * rstd * gg.w + bb.w;
            if (A.pec) {
                float sn[2], cs[2];
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    double x = pc[i][pa[p]];
                    if (A.lo_ext) x = __ddiv_rn(__dsub_rn(x, A.lo_ext[pa[p]]), A.lo_ext[3 + pa[p]]);
                    __sincosf((float)x * exp2f(-(float)pj[p] / (float)npair * A.pl2), &sn[p], &cs[p]);
                }
                o0 += sn[0];
                o1 += cs[0];
                o2 += sn[1];
                o3 += cs[1];
            }
            __nv_bfloat162 h0 = __floats2bfloat162_rn(o0, o1), h1 = __floats2bfloat162_rn(o2, o3);
            uint2 wv;
            wv.x = *reinterpret_cast<uint32_t*>(&h0);
            wv.y = *reinterpret_cast<uint32_t*>(&h1);
            *reinterpret_cast<uint2*>(A.x_next + row * A.ldxn + c0) = wv;
        }
    }
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) mlp_tc_kernel(const Args A) {
    using C = Cfg<D>;
    constexpr int H = C::H, HP = C::HP;
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    uint64_t* x_full = bars;                 // [2] loader -> MMA
    uint64_t* x_empty = bars + 2;            // [2] MMA (GEMM1 done) -> loader
    uint64_t* d1_full = bars + 4;            // [P] MMA -> epilogue WG p (its third of D1)
    uint64_t* g_full = d1_full + kParts;     // [P] epilogue WG p (128) -> MMA (G third packed)
    uint64_t* d2_full = g_full + kParts;     // MMA -> WG1 (residual epilogue)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::kNumBars);
    float* s_bin = reinterpret_cast<float*>(smem + C::kOffBias);
    float* s_bout = s_bin + H;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t n = dyn_n(A.n, A.n_dev);
    const int ntiles = (int)((n + kBM - 1) / kBM);

    // weights and biases -> smem once (all threads; 16-byte chunks)
    for (int i = tid; i < H * (D / 8); i += kThreads) {
        const int r = i / (D / 8), c = i - r * (D / 8);
        *reinterpret_cast<uint4*>(smem + C::kOffWin + core_off<D>(r, c)) =
            __ldg(reinterpret_cast<const uint4*>(A.w_in_t + (int64_t)r * D) + c);
    }
    for (int i = tid; i < D * (H / 8); i += kThreads) {
        const int r = i / (H / 8), c = i - r * (H / 8);
        *reinterpret_cast<uint4*>(smem + C::kOffWout + core_off<H>(r, c)) =
            __ldg(reinterpret_cast<const uint4*>(A.w_out_t + (int64_t)r * H) + c);
    }
    for (int i = tid; i < H; i += kThreads) s_bin[i] = A.b_in[i];
    for (int i = tid; i < D; i += kThreads) s_bout[i] = A.b_out[i];
    if (tid == 0) {
        mbar_init(x_full, 32);
        mbar_init(x_full + 1, 32);
        mbar_init(x_empty, 1);
        mbar_init(x_empty + 1, 1);
        for (int p = 0; p < kParts; ++p) {
            mbar_init(d1_full + p, 1);
            mbar_init(g_full + p, 128);
        }
        mbar_init(d2_full, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sm_base = saddr(smem);

    if (warp == 0) {
        // ------------------------------------------------ x tile loader
        int it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int b = it & 1;
            mbar_wait(x_empty + b, ((it >> 1) & 1) ^ 1);
            const uint32_t dst = sm_base + C::kOffX + b * C::kXBytes;
            const int64_t r0 = (int64_t)tile * kBM;
            for (int i = lane; i < kBM * (D / 8); i += 32) {
                const int r = i / (D / 8), c = i - r * (D / 8);
                const bool ok = r0 + r < n;
                const __nv_bfloat16* src = ok ? A.x + (r0 + r) * A.ldx + c * 8 : A.x;
                cp_async16z(dst + core_off<D>(r, c), src, ok);
            }
            cp_async_arrive(x_full + b);
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA warp
        // GEMM1 third p -> D1[:, p*HP, +HP); GEMM2 k-steps of third p as soon
        // as its G is packed (G elements [p*HP, +HP) at columns [p*HP, +HP/2)).
        constexpr uint32_t id1 = idesc_bf16(kBM, HP, 0, 0);
        constexpr uint32_t id2 = idesc_bf16(kBM, D, 0, 0);
        const uint64_t dW1 = smem_desc(sm_base + C::kOffWin, 128, 16 * D);
        const uint64_t dW2 = smem_desc(sm_base + C::kOffWout, 128, 16 * H);
        const uint64_t dX = smem_desc(sm_base + C::kOffX, 128, 16 * D);
        constexpr uint32_t kXD = C::kXBytes >> 4;
        constexpr uint32_t kPartD = ((HP / 8) * 16 * D) >> 4;   // W_in^T rows [p*HP, ...)
        int it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int b = it & 1;
            mbar_wait(x_full + b, (it >> 1) & 1);
            tc_fence_after();
            const uint64_t dx = dX + (uint64_t)(b * kXD);
            if (elect_one()) {
#pragma unroll
                for (int p = 0; p < kParts; ++p) {
#pragma unroll
                    for (int k = 0; k < D / 16; ++k)
                        umma_f16(tmem + p * HP, dx + (uint64_t)(16 * k),
                                 dW1 + (uint64_t)(p * kPartD + 16 * k), id1, k > 0);
                    umma_commit(d1_full + p);
                }
                umma_commit(x_empty + b);
            }
            __syncwarp();
#pragma unroll
            for (int p = 0; p < kParts; ++p) {
                mbar_wait(g_full + p, it & 1);
                tc_fence_after();
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < HP / 16; ++kk) {
                        const int k = p * (HP / 16) + kk;                // global K-step
                        umma_f16_ts(tmem + C::kTmemD2, tmem + p * HP + 8 * kk,
                                    dW2 + (uint64_t)(16 * k), id2, k > 0);
                    }
                    if (p == kParts - 1) umma_commit(d2_full);
                }
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue warpgroups
        const int p = (warp >> 2) - 1;                      // hidden third of this WG
        const int r = (warp & 3) * 32 + lane;               // row in tile = TMEM lane
        const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t c0 = tmem + lb + p * HP;
        const float* bin = s_bin + p * HP;
        int it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            mbar_wait(d1_full + p, it & 1);
            tc_fence_after();
#pragma unroll 1
            for (int cc = 0; cc < HP; cc += 32) {
                uint32_t v[32];
                tmem_ld32(c0 + cc, v);
                tmem_wait_ld();
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 32; e += 2) {
                    const float2 bb = *reinterpret_cast<const float2*>(bin + cc + e);
                    const float g0 = gelu_as(__uint_as_float(v[e]) + bb.x);
                    const float g1 = gelu_as(__uint_as_float(v[e + 1]) + bb.y);
                    __nv_bfloat162 h2 = __floats2bfloat162_rn(g0, g1);
                    pk[e >> 1] = *reinterpret_cast<uint32_t*>(&h2);
                }
                tmem_st16(c0 + cc / 2, pk);      // packed in place (columns already read)
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(g_full + p);
            // ---- all three WGs: y = D2 -> bf16 tile in smem (WG p copies
            // columns [32p, 32p+32) of its lane quarter), then row-parallel
            // F += y + b_out and LayerNorm (+PE) with lanes over columns
            // (coalesced F / x_next traffic, like f3d_row_ln)
            mbar_wait(d2_full, it & 1);
            tc_fence_after();
            named_bar_sync(1, kParts * 128);               // previous tile's y reads done
            unsigned char* yrow = smem + C::kOffY + r * C::kYStride;
#pragma unroll 1
            for (int c = 32 * p; c < D; c += 32 * kParts) {
                uint32_t v[32];
                tmem_ld32(tmem + lb + C::kTmemD2 + c, v);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 32; e += 8) {
                    uint4 w;
                    uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(v[e + 2 * q]),
                                                                  __uint_as_float(v[e + 2 * q + 1]));
                        wp[q] = *reinterpret_cast<uint32_t*>(&h2);
                    }
                    *reinterpret_cast<uint4*>(yrow + (c + e) * 2) = w;
                }
            }
            named_bar_sync(1, kParts * 128);               // y tile complete
            row_epilogue<D>(A, smem + C::kOffY, s_bout, (int64_t)tile * kBM, n, warp - 4, lane);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int D>
int launch(const Args& A, cudaStream_t st) {
    using C = Cfg<D>;
    auto kern = mlp_tc_kernel<D>;
    static bool attr = false;
    if (!attr) {
        F3D_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          C::kSmem));
        attr = true;
    }
    const int64_t tiles = (A.n + kBM - 1) / kBM;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, f3d_num_sms()));
    kern<<<grid, kThreads, C::kSmem, st>>>(A);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}


// ---------------------------------------------------------------------------
// u = GELU(x W_in + b_in) -> bf16 rows (the MLP's first half, bw/stage.py:91-92,
// 153-156), replacing cuBLAS GEMM + f3d_bias_gelu: the fp32 products never
// leave TMEM and u is written once.  One persistent CTA per SM:
//   * warp 0 loads x tiles (cp.async, 3 buffers); warp 1 (elected lane)
//     issues D[:, q*QP, +QP) = X W_in^T[q*QP, +QP)^T for the four column
//     quarters q into TMEM (4 x QP = 4d <= 512 columns);
//   * warpgroups 1-4 own one quarter each: tcgen05.ld 32 columns (the next
//     chunk's load in flight while the current one is processed), + b_in,
//     packed-pair GELU, bf16, 16-byte stores of the row; the quarter's TMEM is
//     released after its last load, so the next tile's MMA overlaps the tail.
namespace gg {
#ifndef F3D_GG_NOGELU
#define F3D_GG_NOGELU 0    // A/B only: bias epilogue without the GELU
#endif
#ifndef F3D_GG_PARTS
#define F3D_GG_PARTS 4
#endif
constexpr int kQ = F3D_GG_PARTS;               // column parts = epilogue warpgroups
constexpr int kThreads = (1 + kQ) * 128;
constexpr int kNX = 2;                         // x tile buffers

template <int D>
struct Cfg {
    static constexpr int H = 4 * D;
    static constexpr int QP = H / kQ;          // = D columns per quarter
    static constexpr int kWBytes = H * D * 2;
    static constexpr int kXBytes = kBM * D * 2;
    static constexpr int kOffW = 0;
    static constexpr int kOffX = kOffW + kWBytes;
    // per-part output staging: 128 rows x QP bf16, row stride padded by 16 B
    // (conflict-free 16-byte row writes), copied out with coalesced stores
    static constexpr int kStStride = QP * 2 + 16;
    static constexpr int kOffSt = kOffX + kNX * kXBytes;
    static constexpr int kOffBias = kOffSt + kQ * kBM * kStStride;
    static constexpr int kOffBar = kOffBias + H * 4;
    static constexpr int kNumBars = 2 * kNX + 2 * kQ;   // x_full, x_empty, d_full, d_empty
    static constexpr int kSmem = kOffBar + kNumBars * 8 + 16;
    static_assert(QP % 16 == 0 && QP * kQ == H && QP <= 256 && H <= 512,
                  "parts: 16-column chunks, MMA N");
    static_assert(kSmem <= 227 * 1024, "smem budget");
};

struct Args {
    const __nv_bfloat16* x;
    int64_t ldx;
    int64_t n;
    const int32_t* n_dev;
    const __nv_bfloat16* w_in_t;    // (4d, d) = W_in^T
    const float* b_in;
    __nv_bfloat16* u;               // (n, 4d) out
    int64_t ldu;
};

#ifndef F3D_GG_TMA
#define F3D_GG_TMA 1       // x tiles by TMA (SW64 K-major); 0: cp.async core-matrix tiles
#endif
// SW64 K-major operand: 32-column blocks of 64-byte swizzled rows (R rows per
// block); byte offset of 16-byte chunk c of row r
template <int R>
__device__ __forceinline__ uint32_t sw64_off(int r, int c) {
    const int b = c >> 2, cc = c & 3;
    uint32_t o = (uint32_t)(r * 64 + cc * 16);
    o ^= ((o >> 7) & 3) << 4;
    return (uint32_t)(b * R * 64) + o;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) gemm_gelu_kernel(const Args A,
                                                                const __grid_constant__ CUtensorMap xmap) {
    using C = Cfg<D>;
    constexpr int H = C::H, QP = C::QP;
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    uint64_t* x_full = bars;
    uint64_t* x_empty = bars + kNX;
    uint64_t* d_full = bars + 2 * kNX;
    uint64_t* d_empty = d_full + kQ;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::kNumBars);
    float* s_b = reinterpret_cast<float*>(smem + C::kOffBias);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t n = dyn_n(A.n, A.n_dev);
    const int ntiles = (int)((n + kBM - 1) / kBM);

    for (int i = tid; i < H * (D / 8); i += kThreads) {
        const int r = i / (D / 8), c = i - r * (D / 8);
#if F3D_GG_TMA
        const uint32_t wo = sw64_off<H>(r, c);
#else
        const uint32_t wo = core_off<D>(r, c);
#endif
        *reinterpret_cast<uint4*>(smem + C::kOffW + wo) =
            __ldg(reinterpret_cast<const uint4*>(A.w_in_t + (int64_t)r * D) + c);
    }
    for (int i = tid; i < H; i += kThreads) s_b[i] = A.b_in[i];
    if (tid == 0) {
        for (int b = 0; b < kNX; ++b) {
            mbar_init(x_full + b, F3D_GG_TMA ? 1 : 32);
            mbar_init(x_empty + b, 1);
        }
        for (int q = 0; q < kQ; ++q) {
            mbar_init(d_full + q, 1);
            mbar_init(d_empty + q, 128);
        }
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sm_base = saddr(smem);

    if (warp == 0) {
        int it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int b = it % kNX;
            mbar_wait(x_empty + b, ((it / kNX) & 1) ^ 1);
            const uint32_t dst = sm_base + C::kOffX + b * C::kXBytes;
            const int64_t r0 = (int64_t)tile * kBM;
#if F3D_GG_TMA
            if (lane == 0) {           // three 32-column boxes; rows past n zero-filled
                mbar_arrive_expect(x_full + b, C::kXBytes);
#pragma unroll
                for (int blk = 0; blk < D / 32; ++blk)
                    tma_2d(dst + blk * kBM * 64, &xmap, x_full + b, blk * 32, (int)r0);
            }
            __syncwarp();
#else
            for (int i = lane; i < kBM * (D / 8); i += 32) {
                const int r = i / (D / 8), c = i - r * (D / 8);
                const bool ok = r0 + r < n;
                const __nv_bfloat16* src = ok ? A.x + (r0 + r) * A.ldx + c * 8 : A.x;
                cp_async16z(dst + core_off<D>(r, c), src, ok);
            }
            cp_async_arrive(x_full + b);
#endif
        }
    } else if (warp == 1) {
        constexpr uint32_t id = idesc_bf16(kBM, QP, 0, 0);
#if F3D_GG_TMA
        // SW64 K-major: SBO = 8 rows x 64 B; K-step k = block k/2, +32 B inside it
        const uint64_t dW = sw_desc(sm_base + C::kOffW, 16, 512, 4);
        const uint64_t dX = sw_desc(sm_base + C::kOffX, 16, 512, 4);
        constexpr uint32_t kXD = C::kXBytes >> 4;
        constexpr uint32_t kQD = (QP * 64) >> 4;             // W_in^T rows [q*QP, ...)
        auto xk = [](int k) { return (uint32_t)(((k >> 1) * kBM * 64 + (k & 1) * 32) >> 4); };
        auto wk = [](int k) { return (uint32_t)(((k >> 1) * H * 64 + (k & 1) * 32) >> 4); };
#else
        const uint64_t dW = smem_desc(sm_base + C::kOffW, 128, 16 * D);
        const uint64_t dX = smem_desc(sm_base + C::kOffX, 128, 16 * D);
        constexpr uint32_t kXD = C::kXBytes >> 4;
        constexpr uint32_t kQD = ((QP / 8) * 16 * D) >> 4;   // W_in^T rows [q*QP, ...)
        auto xk = [](int k) { return (uint32_t)(16 * k); };
        auto wk = [](int k) { return (uint32_t)(16 * k); };
#endif
        int it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int b = it % kNX;
            mbar_wait(x_full + b, (it / kNX) & 1);
            tc_fence_after();
            const uint64_t dx = dX + (uint64_t)(b * kXD);
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
                if (it > 0) mbar_wait(d_empty + q, (it - 1) & 1);   // quarter q of tile it-1 read
                tc_fence_after();
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < D / 16; ++k)
                        umma_f16(tmem + q * QP, dx + (uint64_t)xk(k),
                                 dW + (uint64_t)(q * kQD + wk(k)), id, k > 0);
                    umma_commit(d_full + q);
                }
                __syncwarp();
            }
            if (elect_one()) umma_commit(x_empty + b);
            __syncwarp();
        }
    } else if (warp >= 4) {
        const int q = (warp >> 2) - 1;                      // column quarter of this WG
        const int r = (warp & 3) * 32 + lane;               // row in tile = TMEM lane
        const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t c0 = tmem + lb + q * QP;
        const float* bq = s_b + q * QP;
        unsigned char* stage = smem + C::kOffSt + q * kBM * C::kStStride;
        int it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            mbar_wait(d_full + q, it & 1);
            tc_fence_after();
            const int64_t r0 = (int64_t)tile * kBM;
            unsigned char* strow = stage + r * C::kStStride;
            constexpr int CW = 16;                          // columns per TMEM load
            uint32_t v[CW], nv[CW];
            tmem_ld16(c0, v);
            tmem_wait_ld();
#pragma unroll 1
            for (int cc = 0; cc < QP; cc += CW) {
                const bool more = cc + CW < QP;
                if (more) tmem_ld16(c0 + cc + CW, nv);      // next chunk in flight
                else {
                    tc_fence_before();
                    mbar_arrive(d_empty + q);               // part fully read
                }
                uint32_t pk[CW / 2];
#pragma unroll
                for (int e = 0; e < CW; e += 2) {
                    const float2 bb = *reinterpret_cast<const float2*>(bq + cc + e);
#if F3D_GG_NOGELU
                    const float2 g = make_float2(__uint_as_float(v[e]) + bb.x,
                                                 __uint_as_float(v[e + 1]) + bb.y);
#else
                    const float2 g = gelu2(__uint_as_float(v[e]) + bb.x,
                                           __uint_as_float(v[e + 1]) + bb.y);
#endif
                    __nv_bfloat162 h2 = __floats2bfloat162_rn(g.x, g.y);
                    pk[e >> 1] = *reinterpret_cast<uint32_t*>(&h2);
                }
#pragma unroll
                for (int e = 0; e < CW / 2; e += 4)
                    *reinterpret_cast<uint4*>(strow + (cc + 2 * e) * 2) =
                        make_uint4(pk[e], pk[e + 1], pk[e + 2], pk[e + 3]);
                if (more) {
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < CW; ++e) v[e] = nv[e];
                }
            }
            named_bar_sync(1 + q, 128);                     // staging tile complete
            // coalesced copy-out: consecutive threads take consecutive 16 B of a row
            constexpr int kChunks = QP * 2 / 16;            // 16-byte chunks per row
            const int tq = tid & 127;
            for (int i = tq; i < kBM * kChunks; i += 128) {
                const int rr = i / kChunks, ch = i - rr * kChunks;
                if (r0 + rr < n)
                    *reinterpret_cast<uint4*>(A.u + (r0 + rr) * A.ldu + q * QP + ch * 8) =
                        *reinterpret_cast<const uint4*>(stage + rr * C::kStStride + ch * 16);
            }
            named_bar_sync(1 + q, 128);                     // staging free for the next tile
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int D>
int launch(const Args& A, cudaStream_t st) {
    using C = Cfg<D>;
    auto kern = gemm_gelu_kernel<D>;
    static bool attr = false;
    if (!attr) {
        F3D_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          C::kSmem));
        attr = true;
    }
    CUtensorMap xmap;
    memset(&xmap, 0, sizeof(xmap));
#if F3D_GG_TMA
    if (!make_map(&xmap, A.x, A.ldx, D, A.n, 32, 64, kBM)) {
        f3d_set_last_cuda_error(cudaErrorNotSupported);   // no cuTensorMapEncodeTiled
        return F3D_ERR_CUDA;
    }
#endif
    const int64_t tiles = (A.n + kBM - 1) / kBM;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, f3d_num_sms()));
    kern<<<grid, kThreads, C::kSmem, st>>>(A, xmap);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}
}  // namespace gg

// ---------------------------------------------------------------------------
// Projection + residual + LayerNorm: F += X W + bias (X: n x K bf16, W: K x D),
// then x_next = LN(F) * g + b (+ PE) in bf16 -- the cuBLAS GEMM + f3d_row_ln
// pair of the stage (O projection -> LN2, bw/stage.py:146-152; MLP output ->
// LN1 + PE of the next round, :153-158) in one pass: the fp32 products go
// TMEM -> bf16 smem tile (the unfused path's bf16 GEMM output) -> row
// epilogue with lanes over columns (coalesced F / x_next), the arithmetic of
// row_ln_vec_kernel.
//   * warp 0 streams X in 96-column K chunks (cp.async, kNC-deep ring), W^T
//     stays in smem; warp 1 (elected lane) accumulates each tile into one of
//     two TMEM buffers (D columns each);
//   * two epilogue warpgroups copy a tile's accumulator rows to the smem y
//     tile (releasing the TMEM buffer), then run the row epilogue.
namespace gl {
constexpr int kKC = 96;                        // K columns per streamed chunk
constexpr int kNC = 4;                         // chunk ring depth
constexpr int kEW = 8;                         // epilogue warps (2 warpgroups)
constexpr int kThreads = 128 + kEW * 32;

template <int D, int K>
struct Cfg {
    static constexpr int kChunks = K / kKC;
    static constexpr int kWBytes = D * K * 2;                 // W^T: D rows x K cols
    static constexpr int kCBytes = kBM * kKC * 2;             // one X chunk
    static constexpr int kYStride = 2 * D + 16;
    static constexpr int kOffW = 0;
    static constexpr int kOffC = kOffW + kWBytes;
    static constexpr int kOffY = kOffC + kNC * kCBytes;
    static constexpr int kOffBias = kOffY + kBM * kYStride;
    static constexpr int kOffBar = kOffBias + D * 4;
    static constexpr int kNumBars = 2 * kNC + 4;              // c_full, c_empty, d_full[2], d_empty[2]
    static constexpr int kSmem = kOffBar + kNumBars * 8 + 16;
    static_assert(K % kKC == 0 && D % 32 == 0 && D <= 128, "shapes");
    static_assert(kSmem <= 227 * 1024, "smem budget");
};

struct Args {
    const __nv_bfloat16* x;
    int64_t ldx;
    int64_t n;
    const int32_t* n_dev;
    const __nv_bfloat16* w_t;       // (D, K) row-major = W^T
    const float* bias;              // (D)
    float* F;
    int64_t ldf;
    const float* ln_g;              // nullable: residual only
    const float* ln_b;
    const double* pec;              // nullable: no PE
    const double* lo_ext;
    float pl2;
    __nv_bfloat16* x_next;
    int64_t ldxn;
    float eps;
};

// rows [r0, r0 + 128): warp w of kEW takes 8-row blocks; lane q owns columns
// [4q, 4q + 4) (q < D/4) -- f3d_row_ln's vector arithmetic and PE.
template <int D>
__device__ __forceinline__ void row_epi(const Args& A, const unsigned char* ytile,
                                        const float* s_bias, int64_t r0, int64_t n, int w,
                                        int lane) {
    constexpr int kYStride = 2 * D + 16;
    const bool act = lane < D / 4;
    const int c0 = 4 * lane;
    const float4 bo = act ? *reinterpret_cast<const float4*>(s_bias + c0) : make_float4(0, 0, 0, 0);
    float4 gg = make_float4(0, 0, 0, 0), bb = gg;
    if (A.ln_g && act) {
        gg = __ldg(reinterpret_cast<const float4*>(A.ln_g + c0));
        bb = __ldg(reinterpret_cast<const float4*>(A.ln_b + c0));
    }
    constexpr int npair = D / 6, blk = 2 * npair;
    int pa[2];
    float fq[2], pinv[2];
    double plo[2];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const int c = c0 + 2 * p;
        pa[p] = c / blk;
        const int pj = (c - pa[p] * blk) >> 1;
        fq[p] = exp2f(-(float)pj / (float)npair * A.pl2);
        plo[p] = (A.pec && A.lo_ext) ? A.lo_ext[pa[p]] : 0.0;
        pinv[p] = (A.pec && A.lo_ext) ? (float)(1.0 / A.lo_ext[3 + pa[p]]) : 1.f;
    }
    constexpr int RB = 8;
#pragma unroll 1
    for (int rb = w * RB; rb < kBM; rb += kEW * RB) {
        float4 v[RB];
        double pc[RB][3];
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            const int64_t row = r0 + rb + i;
            const bool ok = act && row < n;
            v[i] = ok ? *reinterpret_cast<const float4*>(A.F + row * A.ldf + c0) : make_float4(0, 0, 0, 0);
            if (A.pec && A.ln_g)
#pragma unroll
                for (int a = 0; a < 3; ++a) pc[i][a] = row < n ? A.pec[3 * row + a] : 0.0;
        }
        float s[RB], q[RB];
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            const int64_t row = r0 + rb + i;
            if (act) {
                const uint2 yy = *reinterpret_cast<const uint2*>(ytile + (rb + i) * kYStride + c0 * 2);
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&yy);
                const float2 y01 = __bfloat1622float2(h[0]), y23 = __bfloat1622float2(h[1]);
                v[i].x += y01.x + bo.x;
                v[i].y += y01.y + bo.y;
                v[i].z += y23.x + bo.z;
                v[i].w += y23.y + bo.w;
                if (row < n) *reinterpret_cast<float4*>(A.F + row * A.ldf + c0) = v[i];
            }
            s[i] = (v[i].x + v[i].y) + (v[i].z + v[i].w);
        }
        if (!A.ln_g) continue;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int i = 0; i < RB; ++i) s[i] += __shfl_xor_sync(0xffffffffu, s[i], o);
        const float inv_d = 1.f / (float)D;
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            const float m = s[i] * inv_d;
            const float a = act ? v[i].x - m : 0.f, b = act ? v[i].y - m : 0.f;
            const float c = act ? v[i].z - m : 0.f, e = act ? v[i].w - m : 0.f;
            q[i] = (a * a + b * b) + (c * c + e * e);
            s[i] = m;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int i = 0; i < RB; ++i) q[i] += __shfl_xor_sync(0xffffffffu, q[i], o);
        if (!act) continue;
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            const int64_t row = r0 + rb + i;
            if (row >= n) break;
            const float rstd = rsqrtf(q[i] * inv_d + A.eps);
            const float m = s[i];
            float o0 = (v[i].x - m) * rstd * gg.x + bb.x;
            float o1 = (v[i].y - m) * rstd * gg.y + bb.y;
            float o2 = (v[i].z - m) * rstd * gg.z + bb.z;
            float o3 = (v[i].w - m) * rstd * gg.w + bb.w;
            if (A.pec) {
                float sn[2], cs[2];
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    // select the axis without dynamic register-array indexing
                    const double cv = pa[p] == 0 ? pc[i][0] : (pa[p] == 1 ? pc[i][1] : pc[i][2]);
                    const float xn = (float)__dsub_rn(cv, plo[p]) * pinv[p];
                    __sincosf(xn * fq[p], &sn[p], &cs[p]);
                }
                o0 += sn[0];
                o1 += cs[0];
                o2 += sn[1];
                o3 += cs[1];
            }
            __nv_bfloat162 h0 = __floats2bfloat162_rn(o0, o1), h1 = __floats2bfloat162_rn(o2, o3);
            uint2 wv;
            wv.x = *reinterpret_cast<uint32_t*>(&h0);
            wv.y = *reinterpret_cast<uint32_t*>(&h1);
            *reinterpret_cast<uint2*>(A.x_next + row * A.ldxn + c0) = wv;
        }
    }
}

template <int D, int K>
__global__ void __launch_bounds__(kThreads, 1) gemm_ln_kernel(const Args A) {
    using C = Cfg<D, K>;
    constexpr int NCH = C::kChunks;
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    uint64_t* c_full = bars;
    uint64_t* c_empty = bars + kNC;
    uint64_t* d_full = bars + 2 * kNC;
    uint64_t* d_empty = d_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::kNumBars);
    float* s_bias = reinterpret_cast<float*>(smem + C::kOffBias);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t n = dyn_n(A.n, A.n_dev);
    const int ntiles = (int)((n + kBM - 1) / kBM);

    for (int i = tid; i < D * (K / 8); i += kThreads) {
        const int r = i / (K / 8), c = i - r * (K / 8);
        *reinterpret_cast<uint4*>(smem + C::kOffW + core_off<K>(r, c)) =
            __ldg(reinterpret_cast<const uint4*>(A.w_t + (int64_t)r * K) + c);
    }
    for (int i = tid; i < D; i += kThreads) s_bias[i] = A.bias[i];
    if (tid == 0) {
        for (int b = 0; b < kNC; ++b) {
            mbar_init(c_full + b, 32);
            mbar_init(c_empty + b, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(d_full + b, 1);
            mbar_init(d_empty + b, kEW * 32);
        }
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(tmem_slot, 256);
        tmem_relinquish();
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sm_base = saddr(smem);

    if (warp == 0) {
        int ci = 0;                                          // chunk counter
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int64_t r0 = (int64_t)tile * kBM;
            for (int kc = 0; kc < NCH; ++kc, ++ci) {
                const int b = ci % kNC;
                mbar_wait(c_empty + b, ((ci / kNC) & 1) ^ 1);
                const uint32_t dst = sm_base + C::kOffC + b * C::kCBytes;
                for (int i = lane; i < kBM * (kKC / 8); i += 32) {
                    const int r = i / (kKC / 8), c = i - r * (kKC / 8);
                    const bool ok = r0 + r < n;
                    const __nv_bfloat16* src = ok ? A.x + (r0 + r) * A.ldx + kc * kKC + c * 8 : A.x;
                    cp_async16z(dst + core_off<kKC>(r, c), src, ok);
                }
                cp_async_arrive(c_full + b);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t id = idesc_bf16(kBM, D, 0, 0);
        const uint64_t dW = smem_desc(sm_base + C::kOffW, 128, 16 * K);
        const uint64_t dC = smem_desc(sm_base + C::kOffC, 128, 16 * kKC);
        constexpr uint32_t kCD = C::kCBytes >> 4;
        int ci = 0, it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int db = it & 1;
            if (it >= 2) mbar_wait(d_empty + db, ((it >> 1) - 1) & 1);   // buffer read out
            tc_fence_after();
            for (int kc = 0; kc < NCH; ++kc, ++ci) {
                const int b = ci % kNC;
                mbar_wait(c_full + b, (ci / kNC) & 1);
                tc_fence_after();
                if (elect_one()) {
                    const uint64_t dc = dC + (uint64_t)(b * kCD);
#pragma unroll
                    for (int k = 0; k < kKC / 16; ++k)
                        umma_f16(tmem + db * D, dc + (uint64_t)(16 * k),
                                 dW + (uint64_t)(16 * (kc * (kKC / 16) + k)), id,
                                 (kc > 0 || k > 0) ? 1u : 0u);
                    umma_commit(c_empty + b);
                    if (kc == NCH - 1) umma_commit(d_full + db);
                }
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        const int e = warp - 4;                              // 0 .. kEW-1
        const int r = (warp & 3) * 32 + lane;                // TMEM lane = tile row
        const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
        const int half = e >> 2;                             // column half of the copy
        unsigned char* yrow = smem + C::kOffY + r * C::kYStride;
        int it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int db = it & 1;
            mbar_wait(d_full + db, (it >> 1) & 1);
            tc_fence_after();
            named_bar_sync(5, kEW * 32);                     // previous tile's y reads done
#pragma unroll
            for (int c = half * (D / 2); c < (half + 1) * (D / 2); c += 16) {
                uint32_t v[16];
                tmem_ld16(tmem + lb + db * D + c, v);
                tmem_wait_ld();
                uint4 w0, w1;
                uint32_t* p0 = reinterpret_cast<uint32_t*>(&w0);
                uint32_t* p1 = reinterpret_cast<uint32_t*>(&w1);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[2 * q]),
                                                             __uint_as_float(v[2 * q + 1]));
                    p0[q] = *reinterpret_cast<uint32_t*>(&h);
                    h = __floats2bfloat162_rn(__uint_as_float(v[8 + 2 * q]),
                                              __uint_as_float(v[9 + 2 * q]));
                    p1[q] = *reinterpret_cast<uint32_t*>(&h);
                }
                *reinterpret_cast<uint4*>(yrow + c * 2) = w0;
                *reinterpret_cast<uint4*>(yrow + c * 2 + 16) = w1;
            }
            tc_fence_before();
            mbar_arrive(d_empty + db);                       // TMEM buffer free
            named_bar_sync(5, kEW * 32);                     // y tile complete
            row_epi<D>(A, smem + C::kOffY, s_bias, (int64_t)tile * kBM, n, e, lane);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
}

template <int D, int K>
int launch(const Args& A, cudaStream_t st) {
    using C = Cfg<D, K>;
    auto kern = gemm_ln_kernel<D, K>;
    static bool attr = false;
    if (!attr) {
        F3D_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          C::kSmem));
        attr = true;
    }
    const int64_t tiles = (A.n + kBM - 1) / kBM;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, f3d_num_sms()));
    kern<<<grid, kThreads, C::kSmem, st>>>(A);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}
}  // namespace gl
}  // namespace mlp
}  // namespace f3d

using namespace f3d;

extern "C" int f3d_mlp_supported(int d) { return d == 96 ? 1 : 0; }

extern "C" int f3d_mlp_fused(const void* x, int64_t ldx, int64_t n, int d, const void* w_in_t,
                             const float* b_in, const void* w_out_t, const float* b_out, float* F,
                             int64_t ldf, const float* ln_g, const float* ln_b,
                             const double* pe_coords, const double* lo_ext, double pe_base,
                             void* x_next, int64_t ldxn, double eps, const int32_t* n_dev,
                             void* stream) {
    if (!f3d_mlp_supported(d) || n < 0 || (ldx & 7) || (ldf & 3) || (x_next && (ldxn & 7)))
        return F3D_ERR_CONFIG;
    if (x_next && (!ln_g || !ln_b)) return F3D_ERR_CONFIG;
    if (pe_coords && (d % 6)) return F3D_ERR_CONFIG;
    if (((uintptr_t)x | (uintptr_t)w_in_t | (uintptr_t)w_out_t | (uintptr_t)F |
         (uintptr_t)x_next) & 15)
        return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    mlp::Args A;
    A.x = (const __nv_bfloat16*)x;
    A.ldx = ldx;
    A.n = n;
    A.n_dev = n_dev;
    A.w_in_t = (const __nv_bfloat16*)w_in_t;
    A.b_in = b_in;
    A.w_out_t = (const __nv_bfloat16*)w_out_t;
    A.b_out = b_out;
    A.F = F;
    A.ldf = ldf;
    A.ln_g = ln_g;
    A.ln_b = ln_b;
    A.pec = pe_coords;
    A.lo_ext = lo_ext;
    A.pl2 = pe_coords ? (float)log2(pe_base) : 0.f;
    A.x_next = (__nv_bfloat16*)x_next;
    A.ldxn = ldxn;
    A.eps = (float)eps;
    cudaStream_t st = (cudaStream_t)stream;
    return mlp::launch<96>(A, st);
}

extern "C" int f3d_gemm_gelu_supported(int d) {
    return (d == 96 || (d == 64 && (4 * 64) % (16 * mlp::gg::kQ) == 0)) ? 1 : 0;
}

extern "C" int f3d_gemm_gelu(const void* x, int64_t ldx, int64_t n, int d, const void* w_in_t,
                             const float* b_in, void* u, int64_t ldu, const int32_t* n_dev,
                             void* stream) {
    if (!f3d_gemm_gelu_supported(d) || n < 0 || (ldx & 7) || (ldu & 7)) return F3D_ERR_CONFIG;
    if (((uintptr_t)x | (uintptr_t)w_in_t | (uintptr_t)u) & 15) return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    mlp::gg::Args A;
    A.x = (const __nv_bfloat16*)x;
    A.ldx = ldx;
    A.n = n;
    A.n_dev = n_dev;
    A.w_in_t = (const __nv_bfloat16*)w_in_t;
    A.b_in = b_in;
    A.u = (__nv_bfloat16*)u;
    A.ldu = ldu;
    cudaStream_t st = (cudaStream_t)stream;
#if F3D_GG_PARTS == 4
    return d == 96 ? mlp::gg::launch<96>(A, st) : mlp::gg::launch<64>(A, st);
#else
    return mlp::gg::launch<96>(A, st);
#endif
}

extern "C" int f3d_gemm_ln_supported(int d, int k) { return (d == 96 && (k == 96 || k == 384)) ? 1 : 0; }

extern "C" int f3d_gemm_ln(const void* x, int64_t ldx, int64_t n, int d, int k, const void* w_t,
                           const float* bias, float* F, int64_t ldf, const float* ln_g,
                           const float* ln_b, const double* pe_coords, const double* lo_ext,
                           double pe_base, void* x_next, int64_t ldxn, double eps,
                           const int32_t* n_dev, void* stream) {
    if (!f3d_gemm_ln_supported(d, k) || n < 0 || (ldx & 7) || (ldf & 3) || (x_next && (ldxn & 7)))
        return F3D_ERR_CONFIG;
    if ((ln_g != nullptr) != (x_next != nullptr) || (ln_g && !ln_b)) return F3D_ERR_CONFIG;
    if (pe_coords && (!ln_g || d % 6)) return F3D_ERR_CONFIG;
    if (((uintptr_t)x | (uintptr_t)w_t | (uintptr_t)F | (uintptr_t)x_next | (uintptr_t)bias) & 15)
        return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    mlp::gl::Args A;
    A.x = (const __nv_bfloat16*)x;
    A.ldx = ldx;
    A.n = n;
    A.n_dev = n_dev;
    A.w_t = (const __nv_bfloat16*)w_t;
    A.bias = bias;
    A.F = F;
    A.ldf = ldf;
    A.ln_g = ln_g;
    A.ln_b = ln_b;
    A.pec = pe_coords;
    A.lo_ext = lo_ext;
    A.pl2 = pe_coords ? (float)log2(pe_base) : 0.f;
    A.x_next = (__nv_bfloat16*)x_next;
    A.ldxn = ldxn;
    A.eps = (float)eps;
    cudaStream_t st = (cudaStream_t)stream;
    return k == 96 ? mlp::gl::launch<96, 96>(A, st) : mlp::gl::launch<96, 384>(A, st);
}
