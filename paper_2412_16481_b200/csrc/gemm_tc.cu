// Stage projections on 5th-generation tensor cores (bw/stage.py:135-138, 146-158):
//
//     Y[n x N] = X[n x K] W[K x N] + bias        (optionally GELU-erf, bf16 out)
//
// the QKV, O and MLP GEMMs of a round (replacing the library GEMMs).  One
// persistent CTA per SM walks (128-row block, BN-column tile) work items:
//   * warp 0 streams X and W^T k-blocks by TMA (K-major, 128/64-byte swizzle)
//     through an S-deep ring of shared-memory stages;
//   * warp 1 (one elected lane) issues tcgen05.mma M=128 N=BN K=16 into one
//     of NB TMEM accumulators (NB x BN <= 512 columns, NB <= 4);
//   * NB epilogue warpgroups take the tiles round robin, one whole tile each
//     (WG g drains accumulator g), so NB tiles' epilogues overlap each other
//     and the next tiles' MMAs: tcgen05.ld 4 x 16 columns per wait, + bias
//     (+ packed-pair GELU), bf16, staged in shared memory (padded rows:
//     conflict-free), then coalesced 16-byte stores of whole row segments.
// N is split into equal tiles of at most 256 columns (a multiple of 16);
// K is a multiple of 32 (BK = 64 with 128-byte swizzle when K % 64 == 0,
// else BK = 32 with 64-byte swizzle).  Rows past n (device count n_dev) are
// computed from whatever the buffer holds and never stored.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "f3d_common.cuh"
#include "tc_common.cuh"

namespace f3d {
namespace gm {

using namespace f3d::tc;

constexpr int kBM = 128;
#ifndef F3D_GEMM_MAXWG
#define F3D_GEMM_MAXWG 3
#endif
constexpr int kMaxWG = F3D_GEMM_MAXWG;   // epilogue warpgroups (one tile each, round robin); 3: 512 threads, 128 registers
constexpr int kThreads = (1 + kMaxWG) * 128;   // warp 0 TMA, warp 1 MMA, warps 4.. epilogue
constexpr int kMaxStages = 8;
constexpr int kSmemLimit = 227 * 1024;

struct Args {
    int64_t n;
    const int32_t* n_dev;
    int K, N, BN, nt, S, nbuf;     // nbuf: TMEM accumulators = active epilogue WGs
    const float* bias;       // (N) fp32, nullable
    int gelu;
    int dbg;                 // A/B only: 1 = epilogue skips its work, 2 = no copy-out
    __nv_bfloat16* y;
    int64_t ldy;
    // shared-memory layout (bytes from the 1024-aligned base)
    int off_stage, stage_bytes, a_bytes, off_st, st_stride, off_bias, off_bar;
    int resident, off_w, w_bytes;   // resident: all of W^T stays in smem (loaded once)
    // swz: the plain epilogue stages its tile as BN/32 boxes of 32 columns in the
    // TMA 64-byte swizzle (conflict-free 16-byte shared stores; the dense
    // 2*BN-byte rows put 16 rows on the same banks at BN = 96)
    int swz;
    // residual + LayerNorm (+PE) epilogue (LN > 0; N == BN, N % 32 == 0):
    //   F[r] += Y[r] + bias;  y[r] = LN(F[r]) * gain + beta (+ PE(coords[r]))
    float* F;
    int64_t ldf;
    const float *gain, *beta;
    const double *pec, *lo_ext;     // PE: (n,3) coordinates, bbox [lo x,y,z, ext x,y,z]
    float pl2, eps;
    int off_f, off_gb;              // NB fp32 F tiles (128B-swizzled boxes of 32 columns); gain, beta, freq
};

// mbarrier wait expanded at the call site (so profiles attribute the spin to
// the waiting role's source line)
#define GM_WAIT(bar, parity)                                                   \
    asm volatile(                                                              \
        "{\n\t.reg .pred p;\n"                                                 \
        "W_%=:\n\t"                                                            \
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"           \
        "@!p bra W_%=;\n\t"                                                    \
        "}" ::"r"(saddr(bar)), "r"((uint32_t)(parity)) : "memory")

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// LN: 0 plain output y = XW + b (+GELU); 1 residual only (F += XW + b);
// 2 residual + LayerNorm -> y (bf16); 3 the same + positional encoding.
template <int BK, bool GELU, bool BIAS, int LN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const Args A, const __grid_constant__ CUtensorMap amap,
                const __grid_constant__ CUtensorMap bmap, const __grid_constant__ CUtensorMap ymap,
                const __grid_constant__ CUtensorMap fmap) {
    extern __shared__ unsigned char smem_raw[];
    // 1024-byte aligned base for the swizzle atoms, derived from the shared
    // array itself so every access below stays a shared-space (STS/LDS) one
    unsigned char* smem = smem_raw + ((1024 - (saddr(smem_raw) & 1023)) & 1023);
    const int S = A.S, BN = A.BN, NB = A.nbuf;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + A.off_bar);
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* acc_full = bars + 2 * S;
    uint64_t* acc_empty = acc_full + kMaxWG;
    uint64_t* w_full = acc_empty + kMaxWG;
    uint64_t* f_full = w_full + 1;             // [kMaxWG] F tile landed (TMA)
    uint64_t* f_empty = f_full + kMaxWG;       // [kMaxWG] F tile stored back (smem free)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(f_empty + kMaxWG);
    float* s_bias = reinterpret_cast<float*>(smem + A.off_bias);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nk = (A.K + BK - 1) / BK;        // a partial last k-block is zero-filled by TMA

    float* s_gain = reinterpret_cast<float*>(smem + A.off_gb);
    float* s_beta = s_gain + A.N;
    float* s_fq = s_beta + A.N;                // PE frequency of pair j (N/2)
    float* s_pe = s_fq + A.N / 2;              // PE: 1/ext x,y,z
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int b = 0; b < kMaxWG; ++b) {
            mbar_init(acc_full + b, 1);
            mbar_init(acc_empty + b, 128);
        }
        mbar_init(w_full, 1);
        for (int b = 0; b < kMaxWG; ++b) {
            mbar_init(f_full + b, 1);
            mbar_init(f_empty + b, 1);
        }
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    // everything above is local set-up: with programmatic dependent launch it
    // overlaps the previous kernel's tail; from here on inputs are read
    pdl_wait();
    const int64_t n = dyn_n(A.n, A.n_dev);
    const int mblocks = (int)((n + kBM - 1) / kBM);
    const int ntiles = mblocks * A.nt;
    for (int i = tid; i < A.N; i += kThreads) s_bias[i] = A.bias ? A.bias[i] : 0.f;
    if constexpr (LN >= 2) {
        for (int i = tid; i < A.N; i += kThreads) {
            s_gain[i] = A.gain[i];
            s_beta[i] = A.beta[i];
        }
        if constexpr (LN == 3) {
            const int npair = A.N / 6;
            for (int i = tid; i < A.N / 2; i += kThreads) {
                const int blk = 2 * npair, c = 2 * i, ax = c / blk, pj = (c - ax * blk) >> 1;
                s_fq[i] = exp2f(-(float)pj / (float)npair * A.pl2);
            }
            if (tid < 3) s_pe[tid] = A.lo_ext ? (float)(1.0 / A.lo_ext[3 + tid]) : 1.f;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sbase = saddr(smem);

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (A.resident && lane == 0) {
            // W^T once: box (j, ks) at off_w + (j * nk + ks) * BN * BK * 2
            mbar_arrive_expect(w_full, A.w_bytes);
            for (int j = 0; j < A.nt; ++j)
                for (int ks = 0; ks < nk; ++ks)
                    tma_2d(sbase + A.off_w + (j * nk + ks) * BN * BK * 2, &bmap, w_full, ks * BK,
                           j * BN);
        }
        int kc = 0, it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int m = t / A.nt, j = t - m * A.nt;
            if constexpr (LN > 0) {
                // the residual tile of epilogue group it % NB, ahead of the MMAs
                const int g = it % NB, use = it / NB;
                if (use >= 1) GM_WAIT(f_empty + g, (use - 1) & 1);
                if (lane == 0) {
                    mbar_arrive_expect(f_full + g, kBM * A.N * 4);
                    for (int b = 0; b < A.N / 32; ++b)
                        tma_2d(sbase + A.off_f + g * kBM * A.N * 4 + b * kBM * 128, &fmap, f_full + g,
                               b * 32, m * kBM);
                }
                __syncwarp();
            }
            for (int ks = 0; ks < nk; ++ks, ++kc) {
                const int s = kc % S;
                if (kc >= S) GM_WAIT(empty + s, ((kc / S) - 1) & 1);
                if (lane == 0) {
                    const uint32_t dst = sbase + A.off_stage + s * A.stage_bytes;
                    mbar_arrive_expect(full + s, A.stage_bytes);
                    tma_2d(dst, &amap, full + s, ks * BK, m * kBM);
                    if (!A.resident) tma_2d(dst + A.a_bytes, &bmap, full + s, ks * BK, j * BN);
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
        if (A.resident) GM_WAIT(w_full, 0);
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int jt = t % A.nt;
            const int buf = it % NB, use = it / NB;
            if (use >= 1) GM_WAIT(acc_empty + buf, (use - 1) & 1);
            tc_fence_after();
            const uint32_t d = tmem + buf * BN;
            for (int ks = 0; ks < nk; ++ks, ++kc) {
                const int s = kc % S;
                GM_WAIT(full + s, (kc / S) & 1);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t a0 = sbase + A.off_stage + s * A.stage_bytes;
                    const uint64_t da = sw_desc(a0, 16, kSbo, kLt);
                    const uint32_t b0 = A.resident
                                            ? sbase + A.off_w + (jt * nk + ks) * BN * BK * 2
                                            : a0 + A.a_bytes;
                    const uint64_t db = sw_desc(b0, 16, kSbo, kLt);
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
    } else if (LN > 0 && warp >= 4 && (warp >> 2) - 1 < NB) {
        // ------------------------------------------------ residual + LN epilogue
        // WG g takes tiles it = g, g + NB, ...; thread = tile row = TMEM lane.
        // Pass 1: F += acc + bias in the swizzled smem F tile (TMA-loaded),
        // row sum; pass 2: centred sum of squares; pass 3: LN (+PE) -> bf16
        // staging row.  Full tiles leave by TMA stores (F and y); the tile
        // holding row n stores its real rows directly.
        const int g = (warp >> 2) - 1;
        const int wq = warp & 3;
        const int r = wq * 32 + lane;
        const uint32_t lb = (uint32_t)(wq * 32) << 16;
        const int N = A.N;
        const int nch = N / 16;
        const float inv_n = 1.f / (float)N;
        unsigned char* ftile = smem + A.off_f + g * kBM * N * 4;
        unsigned char* stage = smem + A.off_st + g * kBM * A.st_stride;
        unsigned char* strow = stage + r * A.st_stride;
        const int tq = tid & 127;
        const uint32_t tbase = tmem + lb + g * N;
        // float4 q (4 columns) of this row: box q / 8, 16-byte chunk (q % 8) ^ (r % 8)
        auto fp = [&](int q) -> float4* {
            return reinterpret_cast<float4*>(ftile + (q >> 3) * kBM * 128 + r * 128 +
                                             ((((q & 7) ^ (r & 7))) << 4));
        };
        int u = 0;
        for (int t = blockIdx.x + g * gridDim.x; t < ntiles; t += NB * gridDim.x, ++u) {
            const int m = t;
            const int64_t r0 = (int64_t)m * kBM;
            const int64_t row = r0 + r;
            const bool full_tile = r0 + kBM <= n;
            GM_WAIT(acc_full + g, u & 1);
            GM_WAIT(f_full + g, u & 1);
            tc_fence_after();
            float s = 0.f;
            uint32_t v[4][16];
            for (int c0 = 0; c0 < nch; c0 += 4) {
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c0 + c < nch) tmem_ld16(tbase + 16 * (c0 + c), v[c]);
                tmem_wait_ld();
                if (c0 + 4 >= nch) {
                    tc_fence_before();
                    mbar_arrive(acc_empty + g);        // accumulator free
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (c0 + c >= nch) break;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int col = 16 * (c0 + c) + 4 * q;
                        float4 f = *fp(col >> 2);
                        f.x += __uint_as_float(v[c][4 * q]) + s_bias[col];
                        f.y += __uint_as_float(v[c][4 * q + 1]) + s_bias[col + 1];
                        f.z += __uint_as_float(v[c][4 * q + 2]) + s_bias[col + 2];
                        f.w += __uint_as_float(v[c][4 * q + 3]) + s_bias[col + 3];
                        *fp(col >> 2) = f;
                        s += (f.x + f.y) + (f.z + f.w);
                    }
                }
            }
            if constexpr (LN >= 2) {
                const float mean = s * inv_n;
                float qv = 0.f;
                for (int q = 0; q < N / 4; ++q) {
                    const float4 f = *fp(q);
                    const float a = f.x - mean, b = f.y - mean, c = f.z - mean, e = f.w - mean;
                    qv += (a * a + b * b) + (c * c + e * e);
                }
                const float rstd = rsqrtf(qv * inv_n + A.eps);
                double pc[3] = {0.0, 0.0, 0.0};
                if constexpr (LN == 3) {
                    if (row < n)
#pragma unroll
                        for (int a = 0; a < 3; ++a) pc[a] = A.pec[3 * row + a];
                }
                if (tq == 0) bulk_wait_read0();        // previous tile's y store left smem
                named_bar(1 + g, 128);
                const int blk = N / 3;
                for (int q = 0; q < N / 4; ++q) {
                    const int col = 4 * q;
                    const float4 f = *fp(q);
                    float o0 = (f.x - mean) * rstd * s_gain[col] + s_beta[col];
                    float o1 = (f.y - mean) * rstd * s_gain[col + 1] + s_beta[col + 1];
                    float o2 = (f.z - mean) * rstd * s_gain[col + 2] + s_beta[col + 2];
                    float o3 = (f.w - mean) * rstd * s_gain[col + 3] + s_beta[col + 3];
                    if constexpr (LN == 3) {
                        // (sin, cos) pairs (col, col+1), (col+2, col+3): the arithmetic
                        // of row_ln_vec_kernel (bw/attention.py:271-288)
                        float sn[2], cs[2];
#pragma unroll
                        for (int p2 = 0; p2 < 2; ++p2) {
                            const int c = col + 2 * p2, ax = c / blk;
                            const double lo = A.lo_ext ? A.lo_ext[ax] : 0.0;
                            const float xn = (float)__dsub_rn(pc[ax], lo) * s_pe[ax];
                            __sincosf(xn * s_fq[c >> 1], &sn[p2], &cs[p2]);
                        }
                        o0 += sn[0];
                        o1 += cs[0];
                        o2 += sn[1];
                        o3 += cs[1];
                    }
                    __nv_bfloat162 h0 = __floats2bfloat162_rn(o0, o1), h1 = __floats2bfloat162_rn(o2, o3);
                    *reinterpret_cast<uint2*>(strow + 8 * q) =
                        make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
                }
            }
            if (full_tile) {
                fence_proxy_async();                   // STS visible to the TMA stores
                named_bar(1 + g, 128);
                if (tq == 0) {
                    for (int b = 0; b < N / 32; ++b)
                        tma_store_2d(&fmap, saddr(ftile + b * kBM * 128), b * 32, (int)r0);
                    if constexpr (LN >= 2) tma_store_2d(&ymap, saddr(stage), 0, (int)r0);
                    bulk_commit();
                    bulk_wait_read0();                 // F tile read: the producer may refill it
                    mbar_arrive(f_empty + g);
                }
                continue;
            }
            // the tile holding row n: real rows only, straight from this thread
            if (row < n) {
                float* fr = A.F + row * A.ldf;
                for (int q = 0; q < N / 4; ++q) reinterpret_cast<float4*>(fr)[q] = *fp(q);
                if constexpr (LN >= 2) {
                    uint4* yr = reinterpret_cast<uint4*>(A.y + row * A.ldy);
                    const uint4* sr = reinterpret_cast<const uint4*>(strow);
                    for (int q = 0; q < N / 8; ++q) yr[q] = sr[q];
                }
            }
            named_bar(1 + g, 128);                     // every row read the tiles
            if (tq == 0) mbar_arrive(f_empty + g);
        }
        if (tq == 0) bulk_wait_read0();
    } else if (LN == 0 && warp >= 4 && (warp >> 2) - 1 < NB) {
        // ------------------------------------------------ epilogue
        // WG g takes the tiles it = g, g + NB, ... of this CTA (TMEM buffer g)
        // whole: tcgen05.ld 4 x 16 columns per wait, + bias (+ GELU), bf16
        // into its padded staging tile, then coalesced row-segment stores.
        const int g = (warp >> 2) - 1;
        const int wq = warp & 3;
        const int r = wq * 32 + lane;                          // tile row = TMEM lane
        const uint32_t lb = (uint32_t)(wq * 32) << 16;
        const int stride = A.st_stride;
        unsigned char* stage = smem + A.off_st + g * kBM * stride;
        unsigned char* strow = stage + r * stride;
        const int nch = BN / 16;
        const int cpr = BN / 8;                                // 16-byte chunks per row
        const uint32_t inv_cpr = ((1u << 20) + cpr - 1) / cpr;  // exact i / cpr for i < 4096
        const int tq = tid & 127;
        const uint32_t tbase = tmem + lb + g * BN;
        int u = 0;
        for (int t = blockIdx.x + g * gridDim.x; t < ntiles; t += NB * gridDim.x, ++u) {
            const int m = t / A.nt, j = t - m * A.nt;
            GM_WAIT(acc_full + g, u & 1);
            tc_fence_after();
            const float* bj = s_bias + j * BN;
            if (A.dbg == 1) {
                tc_fence_before();
                mbar_arrive(acc_empty + g);
                continue;
            }
            const int64_t r0 = (int64_t)m * kBM;
            const bool full_tile = r0 + kBM <= n;
            uint32_t v[4][16];
#pragma unroll
            for (int c = 0; c < 4; ++c)                        // first four chunks in flight
                if (c < nch) tmem_ld16(tbase + 16 * c, v[c]);
            if (tq == 0) bulk_wait_read0();                    // previous tile's store left smem
            named_bar(1 + g, 128);
            for (int c0 = 0; c0 < nch; c0 += 4) {
                if (c0 > 0) {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (c0 + c < nch) tmem_ld16(tbase + 16 * (c0 + c), v[c]);
                }
                tmem_wait_ld();
                if (c0 + 4 >= nch) {
                    tc_fence_before();
                    mbar_arrive(acc_empty + g);                // accumulator free
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (c0 + c >= nch) break;
                    float bv[16];
                    if (BIAS) {                                // 4 vector loads per chunk
                        const float4* bc = reinterpret_cast<const float4*>(bj + 16 * (c0 + c));
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float4 b4 = bc[q];
                            bv[4 * q] = b4.x;
                            bv[4 * q + 1] = b4.y;
                            bv[4 * q + 2] = b4.z;
                            bv[4 * q + 3] = b4.w;
                        }
                    }
                    uint32_t pk[8];
#pragma unroll
                    for (int e = 0; e < 16; e += 2) {
                        float2 f = make_float2(__uint_as_float(v[c][e]), __uint_as_float(v[c][e + 1]));
                        if (BIAS)   // one packed add per pair
                            f2_split(fadd2(f2(f.x, f.y), f2(bv[e], bv[e + 1])), f.x, f.y);
                        if (GELU) f = gelu2(f.x, f.y);
                        __nv_bfloat162 h2 = __floats2bfloat162_rn(f.x, f.y);
                        pk[e >> 1] = *reinterpret_cast<uint32_t*>(&h2);
                    }
                    if (A.swz) {
                        // 16-byte chunks 2cc, 2cc+1: box cc/2, chunks q0, q0+1 of the row
                        const int cc = c0 + c, q0 = (2 * cc) & 3, sw = (r >> 1) & 3;
                        unsigned char* brow = stage + (cc >> 1) * (kBM * 64) + r * 64;
                        *reinterpret_cast<uint4*>(brow + ((q0 ^ sw) << 4)) =
                            make_uint4(pk[0], pk[1], pk[2], pk[3]);
                        *reinterpret_cast<uint4*>(brow + (((q0 + 1) ^ sw) << 4)) =
                            make_uint4(pk[4], pk[5], pk[6], pk[7]);
                    } else {
                        uint4* dst = reinterpret_cast<uint4*>(strow + 32 * (c0 + c));
                        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                    }
                }
            }
            if (full_tile) fence_proxy_async();                // STS visible to the TMA store
            named_bar(1 + g, 128);                             // staging tile complete
            if (A.dbg == 2) continue;
            if (full_tile) {
                // one bulk tensor store of the whole 128 x BN tile
                if (tq == 0) {
                    if (A.swz) {
                        for (int b = 0; b < BN / 32; ++b)
                            tma_store_2d(&ymap, saddr(stage + b * (kBM * 64)), j * BN + b * 32,
                                         (int)r0);
                    } else {
                        tma_store_2d(&ymap, saddr(stage), j * BN, (int)r0);
                    }
                    bulk_commit();
                }
                continue;
            }
            // the tile holding row n: coalesced 16-byte stores of the real rows only
            const int rows = (int)(n - r0);
            const int total = rows * cpr;
            __nv_bfloat16* yb = A.y + j * BN;
            for (int i0 = tq; i0 < total; i0 += 4 * 128) {
                uint4 val[4];
                int rr[4], cc[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int i = i0 + k * 128;
                    rr[k] = (int)(((uint32_t)i * inv_cpr) >> 20);  // i / cpr (i < 2^12, cpr <= 32)
                    cc[k] = i - rr[k] * cpr;
                    if (i < total)
                        val[k] = *reinterpret_cast<const uint4*>(
                            A.swz ? stage + (cc[k] >> 2) * (kBM * 64) + rr[k] * 64 +
                                        (((cc[k] & 3) ^ ((rr[k] >> 1) & 3)) << 4)
                                  : stage + rr[k] * stride + cc[k] * 16);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (i0 + k * 128 < total)
                        *reinterpret_cast<uint4*>(yb + (r0 + rr[k]) * A.ldy + cc[k] * 8) = val[k];
            }
            named_bar(1 + g, 128);                             // staging free again
        }
        if (tq == 0) bulk_wait_read0();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

struct Plan {
    int BK, BN, nt, S;
    Args a;
    size_t smem;
};

// ln: 0 plain; 1..3 the residual (+LN, +PE) epilogue (one column tile, N % 32 == 0)
static bool plan(int K, int N, Plan& p, int ln = 0, bool gelu = false) {
    if (K < 32 || K % 32 || N < 16 || N % 16 || N > 4096) return false;
    if (ln && (N % 32 || N > 256)) return false;
    // BK = 64 (128-byte rows, SWIZZLE_128B) unless F3D_GEMM_BK32 asks for 32 when K % 64 != 0
    p.BK = (K % 64 == 0 || !getenv("F3D_GEMM_BK32")) ? 64 : 32;
    // Column tile: at most 256 wide; with the GELU epilogue at most 96 wide, so
    // that three epilogue warpgroups (TMEM accumulators) work on separate tiles
    // (measured, tools/gemm_bench.py, 100K x 96 -> 384: 44.7 us at 192-wide
    // tiles with two epilogue groups, 35.3 us at 96; config-B step 1.034 ->
    // 1.000 ms).  F3D_GEMM_BN_MAX / F3D_GEMM_BN_GELU override (A/B).
    int bn_max = gelu ? 96 : 256;
    if (const char* e = getenv(gelu ? "F3D_GEMM_BN_GELU" : "F3D_GEMM_BN_MAX"))
        bn_max = std::max(16, atoi(e));
    int nt = (N + bn_max - 1) / bn_max;
    while (nt <= N / 16 && (N % nt || (N / nt) % 16)) ++nt;
    if (nt > N / 16) return false;
    p.nt = nt;
    p.BN = N / nt;
    Args& a = p.a;
    a.K = K;
    a.N = N;
    a.BN = p.BN;
    a.nt = nt;
    a.a_bytes = kBM * p.BK * 2;
    // dense rows: the TMA store box layout (the LN epilogue stages y only with LN)
    a.st_stride = (ln == 1) ? 0 : 2 * p.BN;
    a.swz = (ln == 0 && p.BN % 32 == 0 && !getenv("F3D_GEMM_DENSE_STAGE")) ? 1 : 0;
    const int ftile = ln ? kBM * N * 4 : 0;        // per epilogue WG: the fp32 residual tile
    const int bias_bytes = (N * 4 + 15) & ~15;
    const int gb_bytes = ln ? ((2 * N + N / 2 + 4) * 4 + 15) & ~15 : 0;
    // W^T resident in shared memory when it is small (d <= ~128 projections):
    // only X streams, and no tile re-reads the weights from L2
    a.w_bytes = N * ((K + p.BK - 1) / p.BK) * p.BK * 2;
    // measured (tools/gemm_bench.py, d = 96): resident wins for the 55 KB QKV
    // weights (18.8 vs 20.8 us streaming), streaming for the 74 KB MLP ones
    // (the resident copy costs pipeline stages)
    int wmax = 64 * 1024;
    if (const char* e = getenv("F3D_GEMM_WRES_KB")) wmax = atoi(e) * 1024;
    a.resident = a.w_bytes <= wmax;
    a.stage_bytes = a.resident ? a.a_bytes : (kBM + p.BN) * p.BK * 2;
    const int wres = a.resident ? a.w_bytes : 0;
    // as many TMEM accumulators / epilogue WGs as fit, keeping >= 3 stages (>= 2 at worst)
    int nb = std::min(kMaxWG, 512 / p.BN);
    if (const char* e = getenv("F3D_GEMM_NB")) nb = std::max(1, std::min(nb, atoi(e)));
    int S = 0;
    if (ln && !getenv("F3D_GEMM_NB")) nb = std::min(nb, 2);
    for (; nb >= 1; --nb) {
        const int fixed = 1024 + wres + nb * (kBM * a.st_stride + ftile) + bias_bytes + gb_bytes +
                          512;
        S = std::min(kMaxStages, (kSmemLimit - fixed) / a.stage_bytes);
        // the LN epilogue is the heavy part: two epilogue groups even at 2 stages
        if (S >= 3 || (nb == 1 && S >= 2) || (ln && S >= 2)) break;
    }
    if (nb < 1 || S < 2) return false;
    a.nbuf = nb;
    p.S = a.S = S;
    a.off_w = 0;
    a.off_stage = wres;
    a.off_f = a.off_stage + S * a.stage_bytes;                 // 1024-aligned: stage sizes are
    a.off_st = a.off_f + nb * ftile;
    a.off_bias = a.off_st + nb * kBM * a.st_stride;
    a.off_gb = a.off_bias + bias_bytes;
    a.off_bar = (a.off_gb + gb_bytes + 15) & ~15;
    p.smem = (size_t)a.off_bar + (2 * S + 4 * kMaxWG + 1) * 8 + 16 + 1024;
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
    if (!gm::plan(K, N, p, 0, gelu != 0) || n < 0 || (ldx & 7) || (ldy & 7) || ldx < K || ldy < N ||
        (((uintptr_t)x | (uintptr_t)w_t | (uintptr_t)y) & 15))
        return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    cudaStream_t st = (cudaStream_t)stream;
    CUtensorMap amap, bmap, ymap;
    memset(&amap, 0, sizeof(amap));
    memset(&bmap, 0, sizeof(bmap));
    memset(&ymap, 0, sizeof(ymap));
    const int sw = p.BK * 2;
    if (!tc::make_map(&amap, x, ldx, K, n, p.BK, sw, gm::kBM) ||
        !tc::make_map(&bmap, w_t, K, K, N, p.BK, sw, p.BN) ||
        !(p.a.swz ? tc::make_map(&ymap, y, ldy, N, n, 32, 64, gm::kBM)
                  : tc::make_map(&ymap, y, ldy, N, n, p.BN, 0, gm::kBM))) {
        f3d_set_last_cuda_error(cudaErrorNotSupported);
        return F3D_ERR_CUDA;
    }
    gm::Args a = p.a;
    a.n = n;
    a.n_dev = n_dev;
    a.bias = bias;
    a.gelu = gelu;
    {
        const char* e = getenv("F3D_GEMM_DBG");
        a.dbg = e ? atoi(e) : 0;
    }
    a.y = (__nv_bfloat16*)y;
    a.ldy = ldy;
    using Kern = void (*)(const gm::Args, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                          const CUtensorMap);
    static const Kern kerns[8] = {
        gm::gemm_kernel<32, false, false, 0>, gm::gemm_kernel<32, false, true, 0>,
        gm::gemm_kernel<32, true, false, 0>,  gm::gemm_kernel<32, true, true, 0>,
        gm::gemm_kernel<64, false, false, 0>, gm::gemm_kernel<64, false, true, 0>,
        gm::gemm_kernel<64, true, false, 0>,  gm::gemm_kernel<64, true, true, 0>};
    const int ki = 4 * (p.BK == 64) + 2 * (gelu != 0) + (bias != nullptr);
    const Kern kern = kerns[ki];
    static int attr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int& at = attr[ki];
    if ((int)p.smem > at) {
        F3D_CUDA_TRY(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)p.smem));
        at = (int)p.smem;
    }
    const int64_t tiles = ((n + gm::kBM - 1) / gm::kBM) * p.nt;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, f3d_num_sms()));
    F3D_CUDA_TRY(f3d_launch(kern, dim3(grid), dim3(gm::kThreads), p.smem, st, a, amap, bmap, ymap,
                            ymap));
    return F3D_OK;
}

extern "C" int f3d_gemm_res_ln_supported(int K, int N) {
    gm::Plan p;
    return gm::plan(K, N, p, 2) ? 1 : 0;
}

// F[r] += X[r] W + bias (fp32 residual, in place); with gain/beta:
// y[r] = LayerNorm(F[r]) * gain + beta (+ PE) as bf16 (bw/stage.py:134-158: the
// O projection -> LN2 and the MLP output -> next round's LN1 + PE).
extern "C" int f3d_gemm_res_ln(const void* x, int64_t ldx, int64_t n, int K, const void* w_t,
                               int N, const float* bias, float* F, int64_t ldf, const float* gain,
                               const float* beta, const double* pe_coords, const double* lo_ext,
                               double pe_base, double eps, void* y, int64_t ldy,
                               const int32_t* n_dev, void* stream) {
    const int ln = gain ? (pe_coords ? 3 : 2) : 1;
    gm::Plan p;
    if (!gm::plan(K, N, p, ln) || n < 0 || (ldx & 7) || ldx < K || ldf < N || (ldf & 3) ||
        (((uintptr_t)x | (uintptr_t)w_t | (uintptr_t)F) & 15) || (gain && !beta) ||
        (pe_coords && (N % 6)))
        return F3D_ERR_CONFIG;
    if (ln >= 2 && (!y || (ldy & 7) || ldy < N || ((uintptr_t)y & 15))) return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    cudaStream_t st = (cudaStream_t)stream;
    CUtensorMap amap, bmap, ymap, fmap;
    memset(&amap, 0, sizeof(amap));
    memset(&bmap, 0, sizeof(bmap));
    memset(&ymap, 0, sizeof(ymap));
    memset(&fmap, 0, sizeof(fmap));
    const int sw = p.BK * 2;
    if (!tc::make_map(&amap, x, ldx, K, n, p.BK, sw, gm::kBM) ||
        !tc::make_map(&bmap, w_t, K, K, N, p.BK, sw, p.BN) ||
        !tc::make_map_f32(&fmap, F, ldf, N, n, 32, 128, gm::kBM) ||
        (ln >= 2 && !tc::make_map(&ymap, y, ldy, N, n, N, 0, gm::kBM))) {
        f3d_set_last_cuda_error(cudaErrorNotSupported);
        return F3D_ERR_CUDA;
    }
    gm::Args a = p.a;
    a.n = n;
    a.n_dev = n_dev;
    a.bias = bias;
    a.gelu = 0;
    a.dbg = 0;
    a.y = (__nv_bfloat16*)y;
    a.ldy = ldy;
    a.F = F;
    a.ldf = ldf;
    a.gain = gain;
    a.beta = beta;
    a.pec = pe_coords;
    a.lo_ext = lo_ext;
    a.pl2 = (float)log2(pe_base);
    a.eps = (float)eps;
    using Kern = void (*)(const gm::Args, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                          const CUtensorMap);
    static const Kern kerns[6] = {
        gm::gemm_kernel<32, false, true, 1>, gm::gemm_kernel<32, false, true, 2>,
        gm::gemm_kernel<32, false, true, 3>, gm::gemm_kernel<64, false, true, 1>,
        gm::gemm_kernel<64, false, true, 2>, gm::gemm_kernel<64, false, true, 3>};
    const int ki = 3 * (p.BK == 64) + (ln - 1);
    const Kern kern = kerns[ki];
    static int attr[6] = {0, 0, 0, 0, 0, 0};
    int& at = attr[ki];
    if ((int)p.smem > at) {
        F3D_CUDA_TRY(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)p.smem));
        at = (int)p.smem;
    }
    const int64_t tiles = (n + gm::kBM - 1) / gm::kBM;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, f3d_num_sms()));
    F3D_CUDA_TRY(f3d_launch(kern, dim3(grid), dim3(gm::kThreads), p.smem, st, a, amap, bmap, ymap,
                            fmap));
    return F3D_OK;
}
