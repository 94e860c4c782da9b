// Fused bucket-swin attention backward (training): the
// gradient of the per-scope softmax attention of bw/attention.py:188-268
// (differentiated; the reference itself has no backward) without ever
// materialising an m x m score tile.  Given the forward's bf16 Q/K/V, the
// upstream gradient dO (bf16) and the forward's log2-domain row logsumexp L:
//     P  = exp2(S * log2e/sqrt(dh) - L),   S = Q K^T
//     dP = dO V^T,   D = sum_j P dP / sum_j P,   dS = P * (dP - D)
//     dV = P^T dO,   dK = dS^T Q / sqrt(dh),   dQ = dS K / sqrt(dh)
// Two kernels (FlashAttention-2 backward split, no atomics):
//   * key kernel: CTA = (scope, 64-key block, head), 4 warps x 16 keys; it
//     streams the scope's query blocks (Q, dO, L, D double-buffered with
//     cp.async) and accumulates dK, dV in registers;
//   * query kernel (first): CTA = (scope, 64-query block, head); streams
//     the key blocks (K, V) twice: D of its rows (written for the key
//     kernel), then dQ.
// bf16 mma.sync m16n8k16 with fp32 accumulation; P and dS are rounded to bf16
// as MMA operands (as the forward rounds P).  Head dims 8..32 (multiples of 8,
// padded to 16 / 32 columns in shared memory).  Rows of a scope are gathered
// in place from the scattered layout (segments, as in the forward); every row
// belongs to exactly one scope per round, so outputs are plain stores.
#include <cuda_bf16.h>

#include "f3d_common.cuh"

namespace f3d {
namespace attn_bwd {

constexpr int kBR = 64;            // rows per block (keys or queries)
constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
#ifndef F3D_BWD_MINB
#define F3D_BWD_MINB 4     // resident CTAs per SM (register cap 128): 25.7 vs 29.5 ms per
                           // 4-scene training step at 1 (5: 26.2, spills)
#endif

struct Args {
    const __nv_bfloat16 *q, *k, *v, *dout;   // (rows, H*dh) head h at column h*dh
    int64_t ld_q, ld_k, ld_v, ld_do;
    const float* lse;          // (rows, ld_lse): log2-domain logsumexp of the scaled scores
    const float* delta;        // (rows, ld_delta): D per (row, head), written by the q kernel
    float* delta_out;          // the same buffer, written
    int64_t ld_lse, ld_delta;
    float *dq, *dk, *dv;       // fp32 outputs (nullable per kernel), head h at column h*dh
    int64_t ld_dq, ld_dk, ld_dv;
    int H, dh;
    float sl2;                 // log2(e) / sqrt(dh)
    float inv_sqrt;            // 1 / sqrt(dh)
    const int32_t *scope_seg, *scope_nseg, *seg_start, *seg_vstart, *scope_len;
    int nscopes, nblk;         // grid.x = nscopes * nblk (nblk = ceil(max_len / 64))
};

__device__ __forceinline__ uint32_t su32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp16(void* dst, const void* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(su32(dst)), "l"(src),
                 "r"(ok ? 16 : 0));
}
__device__ __forceinline__ void cp4(void* dst, const void* src, bool ok) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(su32(dst)), "l"(src),
                 "r"(ok ? 4 : 0));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait_group() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void ldsm4(const void* p, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(su32(p)));
}
__device__ __forceinline__ void ldsm2(const void* p, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];\n"
                 : "=r"(r0), "=r"(r1)
                 : "r"(su32(p)));
}
__device__ __forceinline__ void ldsm2t(const void* p, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];\n"
                 : "=r"(r0), "=r"(r1)
                 : "r"(su32(p)));
}
__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct Scope {
    int s0, s1, m;
};

__device__ __forceinline__ int phys_row(const Args& A, const Scope& sc, int vr) {
    int seg = sc.s0;
    for (int s = sc.s0 + 1; s < sc.s1; ++s)
        if (__ldg(A.seg_vstart + s) <= vr) seg = s;
    return __ldg(A.seg_start + seg) + (vr - __ldg(A.seg_vstart + seg));
}

// Rows [v0, v0+64) of head h into a smem tile of kStride-byte rows (real
// 16-byte chunks only; rows >= m zero-filled); optionally the per-row
// scalars lse / delta of the same rows.
template <int DH>
__device__ __forceinline__ void load_rows(const Args& A, const Scope& sc, int v0, int h,
                                          const __nv_bfloat16* src0, int64_t ld0, char* dst0,
                                          const __nv_bfloat16* src1, int64_t ld1, char* dst1,
                                          float* sl, float* sd) {
    constexpr int kStride = DH * 2 + 16;
    const int rc = A.dh >> 3;                   // real 16-byte chunks per row
    for (int idx = threadIdx.x; idx < kBR * rc; idx += kThreads) {
        const int r = idx / rc, c = idx - r * rc;
        const int vr = v0 + r;
        const bool ok = vr < sc.m;
        const int pr = ok ? phys_row(A, sc, vr) : 0;
        const int64_t col = (int64_t)h * A.dh + c * 8;
        cp16(dst0 + r * kStride + c * 16, src0 + (ok ? (int64_t)pr * ld0 + col : 0), ok);
        cp16(dst1 + r * kStride + c * 16, src1 + (ok ? (int64_t)pr * ld1 + col : 0), ok);
        if (sl && c == 0) cp4(sl + r, A.lse + (ok ? (int64_t)pr * A.ld_lse + h : 0), ok);
        if (sd && c == 0) cp4(sd + r, A.delta + (ok ? (int64_t)pr * A.ld_delta + h : 0), ok);
    }
}

template <int DH>
__device__ __forceinline__ void zero_pad(char* tile, int dh, int rows) {
    constexpr int kStride = DH * 2 + 16;
    const int c0 = dh;                           // first pad column
    if (c0 >= DH) return;
    for (int idx = threadIdx.x; idx < rows * (DH - c0); idx += kThreads) {
        const int r = idx / (DH - c0), c = c0 + idx % (DH - c0);
        *reinterpret_cast<__nv_bfloat16*>(tile + r * kStride + c * 2) = __float2bfloat16(0.f);
    }
}

__device__ __forceinline__ bool decode(const Args& A, Scope& sc, int& blk) {
    const int s = blockIdx.x / A.nblk;
    blk = blockIdx.x - s * A.nblk;
    sc.m = __ldg(A.scope_len + s);
    if (blk * kBR >= sc.m) return false;
    sc.s0 = __ldg(A.scope_seg + s);
    sc.s1 = sc.s0 + __ldg(A.scope_nseg + s);
    return true;
}

// ------------------------------------------------------------------ dK, dV
template <int DH>
__global__ void __launch_bounds__(kThreads, F3D_BWD_MINB) attn_bwd_kv_kernel(const Args A) {
    constexpr int kStride = DH * 2 + 16;
    constexpr int kTile = kBR * kStride;
    constexpr int KS = DH / 16, NT = DH / 8;
    __shared__ __align__(16) char sK[kTile], sV[kTile];
    __shared__ __align__(16) char sQ[2][kTile], sO[2][kTile];
    __shared__ float sL[2][kBR], sD[2][kBR];
    Scope sc;
    int kb;
    if (!decode(A, sc, kb)) return;
    const int h = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    zero_pad<DH>(sK, A.dh, kBR);
    zero_pad<DH>(sV, A.dh, kBR);
    zero_pad<DH>(sQ[0], A.dh, kBR);
    zero_pad<DH>(sQ[1], A.dh, kBR);
    zero_pad<DH>(sO[0], A.dh, kBR);
    zero_pad<DH>(sO[1], A.dh, kBR);
    __syncthreads();
    load_rows<DH>(A, sc, kb * kBR, h, A.k, A.ld_k, sK, A.v, A.ld_v, sV, nullptr, nullptr);
    load_rows<DH>(A, sc, 0, h, A.q, A.ld_q, sQ[0], A.dout, A.ld_do, sO[0], sL[0], sD[0]);
    commit();
    const int nqb = (sc.m + kBR - 1) / kBR;
    uint32_t aK[KS][4], aV[KS][4];
    float dk[NT][4], dv[NT][4];
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
    for (int j = 0; j < nqb; ++j) {
        if (j + 1 < nqb) {
            const int b = (j + 1) & 1;
            load_rows<DH>(A, sc, (j + 1) * kBR, h, A.q, A.ld_q, sQ[b], A.dout, A.ld_do, sO[b], sL[b],
                          sD[b]);
        }
        commit();
        wait_group<1>();
        __syncthreads();
        if (j == 0) {
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const int r = warp * 16 + (lane & 15), c = ks * 16 + (lane >> 4) * 8;
                ldsm4(sK + r * kStride + c * 2, aK[ks]);
                ldsm4(sV + r * kStride + c * 2, aV[ks]);
            }
        }
        const int b = j & 1;
        const char* q = sQ[b];
        const char* o = sO[b];
        // S^T = K Q^T, dP^T = V dO^T: 16 keys x 64 queries per warp
        float s[8][4], dp[8][4];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
            for (int e = 0; e < 4; ++e) s[nt][e] = dp[nt][e] = 0.f;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const int r = nt * 8 + (lane & 7), c = ks * 16 + ((lane >> 3) & 1) * 8;
                uint32_t b0, b1;
                ldsm2(q + r * kStride + c * 2, b0, b1);
                mma(s[nt], aK[ks], b0, b1);
                ldsm2(o + r * kStride + c * 2, b0, b1);
                mma(dp[nt], aV[ks], b0, b1);
            }
        }
        // P^T, dS^T (query column c = nt*8 + 2t + e%2 of this block)
        const int qrem = sc.m - j * kBR;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int c = nt * 8 + 2 * t + (e & 1);
                const float p = c < qrem ? ex2(fmaf(s[nt][e], A.sl2, -sL[b][c])) : 0.f;
                s[nt][e] = p;
                dp[nt][e] = p * (dp[nt][e] - sD[b][c]);
            }
        // dV += P^T dO, dK += dS^T Q (k = the block's 64 queries)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            const uint32_t pa[4] = {pack2(s[2 * kk][0], s[2 * kk][1]), pack2(s[2 * kk][2], s[2 * kk][3]),
                                    pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                                    pack2(s[2 * kk + 1][2], s[2 * kk + 1][3])};
            const uint32_t da[4] = {pack2(dp[2 * kk][0], dp[2 * kk][1]), pack2(dp[2 * kk][2], dp[2 * kk][3]),
                                    pack2(dp[2 * kk + 1][0], dp[2 * kk + 1][1]),
                                    pack2(dp[2 * kk + 1][2], dp[2 * kk + 1][3])};
#pragma unroll
            for (int nd = 0; nd < NT; ++nd) {
                const int r = kk * 16 + (lane & 15);
                uint32_t b0, b1;
                ldsm2t(o + r * kStride + nd * 16, b0, b1);
                mma(dv[nd], pa, b0, b1);
                ldsm2t(q + r * kStride + nd * 16, b0, b1);
                mma(dk[nd], da, b0, b1);
            }
        }
        __syncthreads();                           // buffer b is reloaded next iteration
    }
    // store the warp's 16 key rows (rows g, g + 8)
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int vr = kb * kBR + warp * 16 + g + 8 * hr;
        if (vr >= sc.m) continue;
        const int pr = phys_row(A, sc, vr);
        float* pk = A.dk + (int64_t)pr * A.ld_dk + (int64_t)h * A.dh;
        float* pv = A.dv + (int64_t)pr * A.ld_dv + (int64_t)h * A.dh;
#pragma unroll
        for (int nd = 0; nd < NT; ++nd) {
            const int c = nd * 8 + 2 * t;
            if (c < A.dh) {        // dh % 8 == 0: both columns real
                *reinterpret_cast<float2*>(pk + c) =
                    make_float2(dk[nd][2 * hr] * A.inv_sqrt, dk[nd][2 * hr + 1] * A.inv_sqrt);
                *reinterpret_cast<float2*>(pv + c) = make_float2(dv[nd][2 * hr], dv[nd][2 * hr + 1]);
            }
        }
    }
}

// ---------------------------------------------------------------------- dQ
// Two passes over the scope's key blocks.  Pass 0 computes this block's
//     D_i = sum_j P_ij dP_ij / sum_j P_ij
// with exactly the P the passes compute (the consistent form: sum_j dS_ij = 0
// up to fp32 rounding, so a common offset of the keys cannot leak into dQ --
// D = rowsum(dO * O) from the forward's output differs from it by the
// forward's bf16 / polynomial-exp rounding of P, which stage-1 query / key
// gradients amplify by cancellation) and writes it for the key kernel; pass 1
// accumulates dQ.
template <int DH>
__global__ void __launch_bounds__(kThreads, F3D_BWD_MINB) attn_bwd_q_kernel(const Args A) {
    constexpr int kStride = DH * 2 + 16;
    constexpr int kTile = kBR * kStride;
    constexpr int KS = DH / 16, NT = DH / 8;
    __shared__ __align__(16) char sQ[kTile], sO[kTile];
    __shared__ __align__(16) char sK[2][kTile], sV[2][kTile];
    __shared__ float sL[kBR];
    Scope sc;
    int qb;
    if (!decode(A, sc, qb)) return;
    const int h = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    zero_pad<DH>(sQ, A.dh, kBR);
    zero_pad<DH>(sO, A.dh, kBR);
    zero_pad<DH>(sK[0], A.dh, kBR);
    zero_pad<DH>(sK[1], A.dh, kBR);
    zero_pad<DH>(sV[0], A.dh, kBR);
    zero_pad<DH>(sV[1], A.dh, kBR);
    __syncthreads();
    load_rows<DH>(A, sc, qb * kBR, h, A.q, A.ld_q, sQ, A.dout, A.ld_do, sO, sL, nullptr);
    load_rows<DH>(A, sc, 0, h, A.k, A.ld_k, sK[0], A.v, A.ld_v, sV[0], nullptr, nullptr);
    commit();
    const int nkb = (sc.m + kBR - 1) / kBR;
    uint32_t aQ[KS][4], aO[KS][4];
    float lr[2] = {0.f, 0.f}, dr[2] = {0.f, 0.f};
    float spp[2] = {0.f, 0.f}, sp[2] = {0.f, 0.f};   // pass 0: sum P dP, sum P
    float dq[NT][4];
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) dq[i][e] = 0.f;
    for (int it = 0; it < 2 * nkb; ++it) {
        const int pass = it >= nkb ? 1 : 0, j = it - pass * nkb;
        if (it + 1 < 2 * nkb) {
            const int jn = (it + 1) % nkb, bn = (it + 1) & 1;
            load_rows<DH>(A, sc, jn * kBR, h, A.k, A.ld_k, sK[bn], A.v, A.ld_v, sV[bn], nullptr,
                          nullptr);
        }
        commit();
        wait_group<1>();
        __syncthreads();
        if (it == 0) {
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const int r = warp * 16 + (lane & 15), c = ks * 16 + (lane >> 4) * 8;
                ldsm4(sQ + r * kStride + c * 2, aQ[ks]);
                ldsm4(sO + r * kStride + c * 2, aO[ks]);
            }
#pragma unroll
            for (int hr = 0; hr < 2; ++hr) lr[hr] = sL[warp * 16 + g + 8 * hr];
        }
        if (it == nkb) {
            // end of pass 0: the quad's partial sums -> D of rows g, g + 8
#pragma unroll
            for (int hr = 0; hr < 2; ++hr) {
                float a = spp[hr], b = sp[hr];
                a += __shfl_xor_sync(0xffffffffu, a, 1);
                a += __shfl_xor_sync(0xffffffffu, a, 2);
                b += __shfl_xor_sync(0xffffffffu, b, 1);
                b += __shfl_xor_sync(0xffffffffu, b, 2);
                dr[hr] = b > 0.f ? a / b : 0.f;
                const int vr = qb * kBR + warp * 16 + g + 8 * hr;
                if (t == 0 && vr < sc.m)
                    A.delta_out[(int64_t)phys_row(A, sc, vr) * A.ld_delta + h] = dr[hr];
            }
        }
        const int b = it & 1;
        const char* kt = sK[b];
        const char* vt = sV[b];
        float s[8][4], dp[8][4];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
            for (int e = 0; e < 4; ++e) s[nt][e] = dp[nt][e] = 0.f;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const int r = nt * 8 + (lane & 7), c = ks * 16 + ((lane >> 3) & 1) * 8;
                uint32_t b0, b1;
                ldsm2(kt + r * kStride + c * 2, b0, b1);
                mma(s[nt], aQ[ks], b0, b1);
                ldsm2(vt + r * kStride + c * 2, b0, b1);
                mma(dp[nt], aO[ks], b0, b1);
            }
        }
        const int krem = sc.m - j * kBR;
        if (pass == 0) {
#pragma unroll
            for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int c = nt * 8 + 2 * t + (e & 1);
                    const int hr = e >> 1;
                    const float p = c < krem ? ex2(fmaf(s[nt][e], A.sl2, -lr[hr])) : 0.f;
                    sp[hr] += p;
                    spp[hr] = fmaf(p, dp[nt][e], spp[hr]);
                }
        } else {
#pragma unroll
            for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int c = nt * 8 + 2 * t + (e & 1);
                    const int hr = e >> 1;
                    const float p = c < krem ? ex2(fmaf(s[nt][e], A.sl2, -lr[hr])) : 0.f;
                    dp[nt][e] = p * (dp[nt][e] - dr[hr]);
                }
            // dQ += dS K (k = the block's 64 keys)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const uint32_t da[4] = {pack2(dp[2 * kk][0], dp[2 * kk][1]),
                                        pack2(dp[2 * kk][2], dp[2 * kk][3]),
                                        pack2(dp[2 * kk + 1][0], dp[2 * kk + 1][1]),
                                        pack2(dp[2 * kk + 1][2], dp[2 * kk + 1][3])};
#pragma unroll
                for (int nd = 0; nd < NT; ++nd) {
                    const int r = kk * 16 + (lane & 15);
                    uint32_t b0, b1;
                    ldsm2t(kt + r * kStride + nd * 16, b0, b1);
                    mma(dq[nd], da, b0, b1);
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int vr = qb * kBR + warp * 16 + g + 8 * hr;
        if (vr >= sc.m) continue;
        const int pr = phys_row(A, sc, vr);
        float* pq = A.dq + (int64_t)pr * A.ld_dq + (int64_t)h * A.dh;
#pragma unroll
        for (int nd = 0; nd < NT; ++nd) {
            const int c = nd * 8 + 2 * t;
            if (c < A.dh)
                *reinterpret_cast<float2*>(pq + c) =
                    make_float2(dq[nd][2 * hr] * A.inv_sqrt, dq[nd][2 * hr + 1] * A.inv_sqrt);
        }
    }
}

}  // namespace attn_bwd
}  // namespace f3d

using namespace f3d;

extern "C" int f3d_attn_bwd(const void* q, const void* k, const void* v, const void* dout,
                            int64_t ld_q, int64_t ld_k, int64_t ld_v, int64_t ld_do,
                            const float* lse, int64_t ld_lse, float* delta, int64_t ld_delta,
                            float* dq, int64_t ld_dq, float* dk, int64_t ld_dk, float* dv,
                            int64_t ld_dv, int H, int dh, const int32_t* scope_seg,
                            const int32_t* scope_nseg, const int32_t* seg_start,
                            const int32_t* seg_vstart, const int32_t* scope_len, int nscopes,
                            int max_len, void* stream) {
    if (H < 1 || dh < 8 || dh > 32 || (dh & 7) || nscopes < 0 || max_len < 0) return F3D_ERR_CONFIG;
    if (((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)dout) & 15) return F3D_ERR_CONFIG;
    if ((ld_q | ld_k | ld_v | ld_do) & 7) return F3D_ERR_CONFIG;
    if ((((uintptr_t)dq | (uintptr_t)dk | (uintptr_t)dv) & 7) || ((ld_dq | ld_dk | ld_dv) & 1))
        return F3D_ERR_CONFIG;
    if (nscopes == 0 || max_len == 0) return F3D_OK;
    attn_bwd::Args A;
    A.q = (const __nv_bfloat16*)q;
    A.k = (const __nv_bfloat16*)k;
    A.v = (const __nv_bfloat16*)v;
    A.dout = (const __nv_bfloat16*)dout;
    A.ld_q = ld_q;
    A.ld_k = ld_k;
    A.ld_v = ld_v;
    A.ld_do = ld_do;
    A.lse = lse;
    A.delta = delta;
    A.delta_out = delta;
    A.ld_lse = ld_lse;
    A.ld_delta = ld_delta;
    A.dq = dq;
    A.dk = dk;
    A.dv = dv;
    A.ld_dq = ld_dq;
    A.ld_dk = ld_dk;
    A.ld_dv = ld_dv;
    A.H = H;
    A.dh = dh;
    A.sl2 = (float)(1.4426950408889634 / sqrt((double)dh));
    A.inv_sqrt = (float)(1.0 / sqrt((double)dh));
    A.scope_seg = scope_seg;
    A.scope_nseg = scope_nseg;
    A.seg_start = seg_start;
    A.seg_vstart = seg_vstart;
    A.scope_len = scope_len;
    A.nscopes = nscopes;
    A.nblk = (max_len + attn_bwd::kBR - 1) / attn_bwd::kBR;
    cudaStream_t st = (cudaStream_t)stream;
    const dim3 grid((unsigned)(nscopes * A.nblk), (unsigned)H);
    // the query kernel first: it writes D for the key kernel
    if (dh <= 16) {
        attn_bwd::attn_bwd_q_kernel<16><<<grid, attn_bwd::kThreads, 0, st>>>(A);
        F3D_LAUNCH_CHECK();
        attn_bwd::attn_bwd_kv_kernel<16><<<grid, attn_bwd::kThreads, 0, st>>>(A);
    } else {
        attn_bwd::attn_bwd_q_kernel<32><<<grid, attn_bwd::kThreads, 0, st>>>(A);
        F3D_LAUNCH_CHECK();
        attn_bwd::attn_bwd_kv_kernel<32><<<grid, attn_bwd::kThreads, 0, st>>>(A);
    }
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}
