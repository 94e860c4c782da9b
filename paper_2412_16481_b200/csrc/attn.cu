// Bucket-swin attention forward (bw/attention.py:188-268 tiled_attention,
// driven per round by bw/stage.py:134-156).
//
// Each work item is (scope, 64-row query tile, head).  A scope is the
// concatenation of up to kMaxSeg physical row segments of the scattered
// layout (its buckets; bw/attention.py:120-139), tiled as ONE virtual
// sequence of m_s rows ("scope-packed"), so only the final
// key tile is ragged.  Rows are gathered straight from the fixed layout with
// cp.async (zero-fill beyond m_s), so no feature row ever moves between
// rounds.  Math: bf16 mma.sync m16n8k16 with fp32 accumulation, online
// softmax in exp2 domain (FlashAttention-2 structure, 4 warps x 16 rows).
#include <cuda_bf16.h>

#include <algorithm>
#include <cfloat>

#include "f3d_common.cuh"

namespace f3d {
namespace attn {

constexpr int kBM = 128;      // query rows per CTA (8 warps x 16 rows)
constexpr int kBN = 64;       // keys per tile
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

struct Args {
    const __nv_bfloat16* q;   // element (row, h*dh + c) at q[row*ld + h*dh + c]
    const __nv_bfloat16* k;
    const __nv_bfloat16* v;
    int64_t ld_q, ld_k, ld_v;  // row strides in elements
    void* o;                   // output rows (bf16 or f32), ld_o
    int64_t ld_o;
    int dh;                    // real head dim
    float scale_log2;          // log2(e) / sqrt(dh)
    // scopes
    const int32_t* scope_seg;  // first segment of each scope
    const int32_t* scope_nseg; // segments per scope
    const int32_t* seg_start;  // physical start
    const int32_t* seg_vstart; // virtual start within the scope
    const int32_t* scope_len;  // m_s
    const int32_t* work;       // [nwork][2] = (scope, q_start)
    int nwork;
    const uint8_t* mask;       // optional per-row validity: 1 = present (key and query);
                               // 2 = query only (its key/value row is excluded)
    int32_t* starved;          // optional counter of query rows with no valid key
    const int32_t* scope_order;  // non-empty scopes, longest first (resident kernel)
    int nlive;                 // number of non-empty scopes
    int qsplit;                // CTAs per (scope, head) in the resident kernel
    const int32_t* live;       // optional device [nwork, nlive, max_len] (device planner)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];\n"
                 : "=r"(r0), "=r"(r1)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2_t(uint32_t addr, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];\n"
                 : "=r"(r0), "=r"(r1)
                 : "r"(addr));
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

// Physical row of virtual row vr of a scope (segments are few: linear scan).
__device__ __forceinline__ int phys_row(const Args& A, int s0, int s1, int vr) {
    int seg = s0;
    for (int s = s0 + 1; s < s1; ++s)
        if (A.seg_vstart[s] <= vr) seg = s;
    return A.seg_start[seg] + (vr - A.seg_vstart[seg]);
}

// Load kRows virtual rows [v0, v0+kRows) of one head into smem rows of
// kStride bytes; rows >= m and columns >= dh are zero-filled.
template <int DH, bool kVec>
__device__ __forceinline__ void load_tile(const Args& A, const __nv_bfloat16* base, int64_t ld,
                                          int hcol, int s0, int s1, int m, int v0,
                                          __nv_bfloat16* sm, int kRows, bool ones = false) {
    constexpr int kRowB = DH * 2;
    constexpr int kStride = kRowB + 16;
    constexpr int kChunks = kRowB / 16;
    if (kVec) {
        // pad chunks (c >= real) are never written here: they are set once per
        // CTA (zeros, plus the ones column of V) by init_pad
        const int real_chunks = (A.dh * 2) / 16;
        for (int idx = threadIdx.x; idx < kRows * real_chunks; idx += kThreads) {
            const int r = idx / real_chunks;
            const int c = idx - r * real_chunks;
            const int vr = v0 + r;
            const bool ok = vr < m;
            const __nv_bfloat16* src = base;
            if (ok) src = base + (int64_t)phys_row(A, s0, s1, vr) * ld + hcol + c * 8;
            cp_async16(reinterpret_cast<char*>(sm) + r * kStride + c * 16, src, ok);
        }
    } else {
        for (int idx = threadIdx.x; idx < kRows * DH; idx += kThreads) {
            const int r = idx / DH;
            const int c = idx - r * DH;
            const int vr = v0 + r;
            __nv_bfloat16 val = __float2bfloat16(ones && c == A.dh ? 1.f : 0.f);
            if (vr < m && c < A.dh) val = base[(int64_t)phys_row(A, s0, s1, vr) * ld + hcol + c];
            *reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<char*>(sm) + r * kStride + c * 2) =
                val;
        }
    }
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Zero the pad columns [dh, DH) of every smem tile once per CTA and put 1.0 in
// column dh of the V tiles: O[:, dh] then accumulates the softmax row sum in
// the same MMA as P V (no per-score FADD).
template <int DH>
__device__ __forceinline__ void init_pad(unsigned char* smem, int dh, int rows_total,
                                         int v_row0, int v_rows) {
    constexpr int kStride = DH * 2 + 16;
    const int c0 = (dh * 2) / 16 * 8;   // first pad column (chunk aligned)
    if (c0 >= DH) return;
    for (int idx = threadIdx.x; idx < rows_total * (DH - c0); idx += kThreads) {
        const int r = idx / (DH - c0);
        const int c = c0 + (idx - r * (DH - c0));
        const bool one = (r >= v_row0 && r < v_row0 + v_rows && c == dh);
        *reinterpret_cast<__nv_bfloat16*>(smem + r * kStride + c * 2) =
            __float2bfloat16(one ? 1.f : 0.f);
    }
}

// One warp, one 64-key tile: S = Q K^T (raw), mask (tail / user mask), online
// softmax in the exp2 domain (FFMA-folded scale), O += P V with P taken from
// the S registers.  kb/vb point at the tile's 64 K / V rows in smem.
template <int DH, bool kMask>
__device__ __forceinline__ void warp_tile(const Args& A, const char* kb, const char* vb, int kbase,
                                          int m, bool tail, int s0, int s1,
                                          const uint32_t (&qf)[DH / 16][4],
                                          float (&o_acc)[DH / 8][4], float (&m_run)[2],
                                          float (&l_run)[2], bool ones, float sl2) {
    constexpr int kStride = DH * 2 + 16;
    constexpr int kNd = DH / 8;
    constexpr int kKd = DH / 16;
    const int lane = threadIdx.x & 31;
    const int t = lane & 3;
    float s[8][4];
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
        s[nb][0] = s[nb][1] = s[nb][2] = s[nb][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < kKd; ++kk) {
            uint32_t b0, b1;
            const int r = nb * 8 + (lane & 7);
            const int c = kk * 16 + ((lane >> 3) & 1) * 8;
            ldsm_x2(smem_u32(kb + r * kStride + c * 2), b0, b1);
            mma16816(s[nb], qf[kk], b0, b1);
        }
    }
    if (kMask || tail) {
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int key = kbase + nb * 8 + 2 * t + (e & 1);
                bool ok = key < m;
                if (kMask && ok) ok = (A.mask[phys_row(A, s0, s1, key)] & 1) != 0;   // bit 0: key present
                if (!ok) s[nb][e] = -INFINITY;
            }
        }
    }
    float p_scale[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        float mx = -INFINITY;
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) mx = fmaxf(mx, fmaxf(s[nb][2 * hr], s[nb][2 * hr + 1]));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float m_new = fmaxf(m_run[hr], mx);
        p_scale[hr] = ex2((m_run[hr] - m_new) * sl2);
        m_run[hr] = m_new;
        const float nms = -m_new * sl2;
        float ls = 0.f;
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
            const float p0 = ex2(fmaf(s[nb][2 * hr], sl2, nms));
            const float p1 = ex2(fmaf(s[nb][2 * hr + 1], sl2, nms));
            s[nb][2 * hr] = p0;
            s[nb][2 * hr + 1] = p1;
            if (!ones) ls += p0 + p1;
        }
        if (!ones) l_run[hr] = l_run[hr] * p_scale[hr] + ls;
    }
#pragma unroll
    for (int i = 0; i < kNd; ++i) {
        o_acc[i][0] *= p_scale[0];
        o_acc[i][1] *= p_scale[0];
        o_acc[i][2] *= p_scale[1];
        o_acc[i][3] *= p_scale[1];
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        uint32_t pa[4];
        pa[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
        pa[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
        pa[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
        pa[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
        for (int nd = 0; nd < kNd; ++nd) {
            uint32_t b0, b1;
            const int r = kk * 16 + (lane & 15);
            ldsm_x2_t(smem_u32(vb + r * kStride + nd * 16), b0, b1);
            mma16816(o_acc[nd], pa, b0, b1);
        }
    }
}

// Normalise and write this warp's 16 query rows (virtual rows q0w..q0w+15).
template <int DH, bool kMask, typename OutT>
__device__ __forceinline__ void warp_epilogue(const Args& A, int q0w, int m, int s0, int s1,
                                              int hcol, float (&o_acc)[DH / 8][4],
                                              const float (&l_run)[2], bool ones) {
    constexpr int kNd = DH / 8;
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    float l_tot[2];
    if (ones) {
        // column dh of O holds the row sum: owned by quad lane (dh % 8) / 2
        const int nd = A.dh >> 3, tq = (A.dh & 7) >> 1, e = A.dh & 1;
        float v0 = 0.f, v1 = 0.f;
#pragma unroll
        for (int i = 0; i < kNd; ++i)
            if (i == nd) {
                v0 = e ? o_acc[i][1] : o_acc[i][0];
                v1 = e ? o_acc[i][3] : o_acc[i][2];
            }
        l_tot[0] = __shfl_sync(0xffffffffu, v0, (lane & ~3) | tq);
        l_tot[1] = __shfl_sync(0xffffffffu, v1, (lane & ~3) | tq);
    } else {
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            float l = l_run[hr];
            l += __shfl_xor_sync(0xffffffffu, l, 1);
            l += __shfl_xor_sync(0xffffffffu, l, 2);
            l_tot[hr] = l;
        }
    }
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int vr = q0w + g + 8 * hr;
        if (vr >= m) continue;
        const int pr = phys_row(A, s0, s1, vr);
        bool qok = true;
        if (kMask) qok = A.mask[pr] != 0;
        const bool starved = !(l_tot[hr] > 0.f);
        if (kMask && starved && t == 0 && A.starved) atomicAdd(A.starved, 1);
        const float inv = (starved || !qok) ? 0.f : 1.f / l_tot[hr];
#pragma unroll
        for (int nd = 0; nd < kNd; ++nd) {
            const int c = nd * 8 + 2 * t;
            const float a0 = o_acc[nd][2 * hr] * inv, a1 = o_acc[nd][2 * hr + 1] * inv;
            if (sizeof(OutT) == 2) {
                __nv_bfloat16* o =
                    reinterpret_cast<__nv_bfloat16*>(A.o) + (int64_t)pr * A.ld_o + hcol;
                if (c + 1 < A.dh) {
                    *reinterpret_cast<__nv_bfloat162*>(o + c) = __floats2bfloat162_rn(a0, a1);
                } else if (c < A.dh) {
                    o[c] = __float2bfloat16(a0);
                }
            } else {
                float* o = reinterpret_cast<float*>(A.o) + (int64_t)pr * A.ld_o + hcol;
                if (c < A.dh) o[c] = a0;
                if (c + 1 < A.dh) o[c + 1] = a1;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Streaming kernel: work item = (scope, 128-row query tile, head); K/V tiles of
// 64 rows double-buffered through smem with cp.async.  Any scope length.
template <int DH, bool kVec, bool kMask, typename OutT>
__global__ void __launch_bounds__(kThreads) bswin_attn_kernel(const Args A) {
    constexpr int kStride = DH * 2 + 16;   // odd number of 16 B chunks: conflict-free ldmatrix
    constexpr int kNd = DH / 8;
    constexpr int kKd = DH / 16;
    extern __shared__ __align__(16) unsigned char smem[];
    __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem);
    __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(smem + kBM * kStride);
    __nv_bfloat16* sV = reinterpret_cast<__nv_bfloat16*>(smem + (kBM + 2 * kBN) * kStride);

    const int wi = blockIdx.x;
    if (wi >= (A.live ? __ldg(A.live) : A.nwork)) return;
    const int h = blockIdx.y;
    const int scope = A.work[2 * wi];
    const int q0 = A.work[2 * wi + 1];
    const int s0 = A.scope_seg[scope], s1 = s0 + A.scope_nseg[scope];
    const int m = A.scope_len[scope];
    const int hcol = h * A.dh;
    const bool ones = A.dh < DH;          // row sums ride in V's pad column

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const bool warp_live = q0 + warp * 16 < m;

    if (kVec) init_pad<DH>(smem, A.dh, kBM + 4 * kBN, kBM + 2 * kBN, 2 * kBN);
    load_tile<DH, kVec>(A, A.q, A.ld_q, hcol, s0, s1, m, q0, sQ, kBM);
    const int ntiles = (m + kBN - 1) / kBN;
    load_tile<DH, kVec>(A, A.k, A.ld_k, hcol, s0, s1, m, 0, sK, kBN);
    load_tile<DH, kVec>(A, A.v, A.ld_v, hcol, s0, s1, m, 0, sV, kBN, ones);
    cp_async_commit();

    float o_acc[kNd][4];
#pragma unroll
    for (int i = 0; i < kNd; ++i) o_acc[i][0] = o_acc[i][1] = o_acc[i][2] = o_acc[i][3] = 0.f;
    float m_run[2] = {-FLT_MAX, -FLT_MAX};
    float l_run[2] = {0.f, 0.f};
    uint32_t qf[kKd][4];

    for (int kt = 0; kt < ntiles; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < ntiles) {
            const int nb = buf ^ 1;
            load_tile<DH, kVec>(A, A.k, A.ld_k, hcol, s0, s1, m, (kt + 1) * kBN,
                                reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<char*>(sK) +
                                                                 nb * kBN * kStride),
                                kBN);
            load_tile<DH, kVec>(A, A.v, A.ld_v, hcol, s0, s1, m, (kt + 1) * kBN,
                                reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<char*>(sV) +
                                                                 nb * kBN * kStride),
                                kBN, ones);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        if (warp_live) {
            if (kt == 0) {
                const char* qb = reinterpret_cast<const char*>(sQ) + (warp * 16) * kStride;
#pragma unroll
                for (int kk = 0; kk < kKd; ++kk) {
                    const int r = lane & 15;
                    const int c = kk * 16 + (lane >> 4) * 8;
                    ldsm_x4(smem_u32(qb + r * kStride + c * 2), qf[kk][0], qf[kk][1], qf[kk][2],
                            qf[kk][3]);
                }
            }
            warp_tile<DH, kMask>(A, reinterpret_cast<const char*>(sK) + buf * kBN * kStride,
                                 reinterpret_cast<const char*>(sV) + buf * kBN * kStride,
                                 kt * kBN, m, kt == ntiles - 1, s0, s1, qf, o_acc, m_run, l_run,
                                 ones, A.scale_log2);
        }
        __syncthreads();
    }
    if (!warp_live) return;
    warp_epilogue<DH, kMask, OutT>(A, q0 + warp * 16, m, s0, s1, hcol, o_acc, l_run, ones);
}

// ---------------------------------------------------------------------------
// Resident kernel (small head dims, scopes <= max rows): one CTA per (scope,
// head, q-part) loads the scope's whole K and V once into smem, then every
// warp walks its own 16-row query blocks over all keys with no block barrier
// in the loop — warps run independently, so latency hides across warps.
constexpr int kResWarps = 16;
constexpr int kResThreads = kResWarps * 32;

template <int DH, typename OutT>
__global__ void __launch_bounds__(kResThreads, 1) bswin_attn_resident_kernel(const Args A) {
    constexpr int kStride = DH * 2 + 16;
    constexpr int kNd = DH / 8;
    constexpr int kKd = DH / 16;
    extern __shared__ __align__(16) unsigned char smem[];
    const int item = blockIdx.x / A.qsplit;
    const int qpart = blockIdx.x - item * A.qsplit;
    if (item >= (A.live ? __ldg(A.live + 1) : A.nlive)) return;
    const int h = blockIdx.y;
    const int scope = A.scope_order[item];
    const int s0 = A.scope_seg[scope], s1 = s0 + A.scope_nseg[scope];
    const int m = A.scope_len[scope];
    const int mpad = (m + kBN - 1) / kBN * kBN;
    const int hcol = h * A.dh;
    const bool ones = A.dh < DH;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    unsigned char* sK = smem;
    unsigned char* sV = smem + (size_t)mpad * kStride;
    unsigned char* sQ = smem + (size_t)2 * mpad * kStride + warp * 16 * kStride;

    // pad columns: zeros (K, V, Q) and the ones column of V
    {
        const int c0 = (A.dh * 2) / 16 * 8;
        if (c0 < DH) {
            const int rows = 2 * mpad;
            for (int idx = threadIdx.x; idx < rows * (DH - c0); idx += kResThreads) {
                const int r = idx / (DH - c0);
                const int c = c0 + (idx - r * (DH - c0));
                *reinterpret_cast<__nv_bfloat16*>(smem + (size_t)r * kStride + c * 2) =
                    __float2bfloat16((r >= mpad && c == A.dh) ? 1.f : 0.f);
            }
            for (int idx = lane; idx < 16 * (DH - c0); idx += 32) {
                const int r = idx / (DH - c0);
                const int c = c0 + (idx - r * (DH - c0));
                *reinterpret_cast<__nv_bfloat16*>(sQ + r * kStride + c * 2) = __float2bfloat16(0.f);
            }
        }
    }
    // K and V of the whole scope, once
    const int real_chunks = (A.dh * 2) / 16;
    for (int idx = threadIdx.x; idx < mpad * real_chunks; idx += kResThreads) {
        const int r = idx / real_chunks;
        const int c = idx - r * real_chunks;
        const bool ok = r < m;
        int64_t off = 0;
        if (ok) off = (int64_t)phys_row(A, s0, s1, r);
        cp_async16(sK + (size_t)r * kStride + c * 16, ok ? A.k + off * A.ld_k + hcol + c * 8 : A.k, ok);
        cp_async16(sV + (size_t)r * kStride + c * 16, ok ? A.v + off * A.ld_v + hcol + c * 8 : A.v, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();

    const int nqb = (m + 15) / 16;
    const int ntiles = mpad / kBN;
    for (int qb = warp * A.qsplit + qpart; qb < nqb; qb += kResWarps * A.qsplit) {
        const int q0w = qb * 16;
        // stage this warp's 16 query rows, then ldmatrix into registers
        for (int idx = lane; idx < 16 * real_chunks; idx += 32) {
            const int r = idx / real_chunks;
            const int c = idx - r * real_chunks;
            const bool ok = q0w + r < m;
            const __nv_bfloat16* src = A.q;
            if (ok) src = A.q + (int64_t)phys_row(A, s0, s1, q0w + r) * A.ld_q + hcol + c * 8;
            cp_async16(sQ + r * kStride + c * 16, src, ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        uint32_t qf[kKd][4];
#pragma unroll
        for (int kk = 0; kk < kKd; ++kk) {
            const int r = lane & 15;
            const int c = kk * 16 + (lane >> 4) * 8;
            ldsm_x4(smem_u32(sQ + r * kStride + c * 2), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
        }
        __syncwarp();
        float o_acc[kNd][4];
#pragma unroll
        for (int i = 0; i < kNd; ++i) o_acc[i][0] = o_acc[i][1] = o_acc[i][2] = o_acc[i][3] = 0.f;
        float m_run[2] = {-FLT_MAX, -FLT_MAX};
        float l_run[2] = {0.f, 0.f};
        for (int kt = 0; kt < ntiles; ++kt)
            warp_tile<DH, false>(A, reinterpret_cast<const char*>(sK) + (size_t)kt * kBN * kStride,
                                 reinterpret_cast<const char*>(sV) + (size_t)kt * kBN * kStride,
                                 kt * kBN, m, kt == ntiles - 1, s0, s1, qf, o_acc, m_run, l_run,
                                 ones, A.scale_log2);
        warp_epilogue<DH, false, OutT>(A, q0w, m, s0, s1, hcol, o_acc, l_run, ones);
    }
}

template <int DH, bool kVec, bool kMask, typename OutT>
int launch_t(const Args& A, int H, cudaStream_t st) {
    constexpr int kStride = DH * 2 + 16;
    const size_t smem = (size_t)(kBM + 4 * kBN) * kStride;
    auto kern = bswin_attn_kernel<DH, kVec, kMask, OutT>;
    if (smem > 48 * 1024) {
        static bool done = false;
        if (!done) {
            F3D_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)smem));
            done = true;
        }
    }
    kern<<<dim3(A.nwork, H), kThreads, smem, st>>>(A);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

template <int DH, typename OutT>
int launch_resident(Args A, int H, int max_len, cudaStream_t st) {
    constexpr int kStride = DH * 2 + 16;
    const int mpad = (max_len + kBN - 1) / kBN * kBN;
    const size_t smem = ((size_t)2 * mpad + 16 * kResWarps) * kStride;
    auto kern = bswin_attn_resident_kernel<DH, OutT>;
    static size_t done = 0;
    if (smem > 48 * 1024 && smem > done) {
        F3D_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        done = smem;
    }
    // enough CTAs for ~4 waves of one CTA per SM
    const int want = 4 * f3d_num_sms();
    int qs = (want + A.nlive * H - 1) / (A.nlive * H);
    const int nqb = (max_len + 15) / 16;
    qs = std::max(1, std::min(qs, std::max(1, nqb / kResWarps)));
    A.qsplit = qs;
    kern<<<dim3(A.nlive * qs, H), kResThreads, smem, st>>>(A);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

template <int DH>
int launch_dh(const Args& A, int H, bool vec, bool mask, bool out_f32, cudaStream_t st) {
    if (mask) {
        if (out_f32) return vec ? launch_t<DH, true, true, float>(A, H, st)
                                : launch_t<DH, false, true, float>(A, H, st);
        return vec ? launch_t<DH, true, true, __nv_bfloat16>(A, H, st)
                   : launch_t<DH, false, true, __nv_bfloat16>(A, H, st);
    }
    if (out_f32) return vec ? launch_t<DH, true, false, float>(A, H, st)
                            : launch_t<DH, false, false, float>(A, H, st);
    return vec ? launch_t<DH, true, false, __nv_bfloat16>(A, H, st)
               : launch_t<DH, false, false, __nv_bfloat16>(A, H, st);
}

}  // namespace attn
}  // namespace f3d

using namespace f3d;

extern "C" int f3d_bswin_attention(const void* q, const void* k, const void* v, int64_t ld_q,
                                   int64_t ld_k, int64_t ld_v, void* o, int64_t ld_o,
                                   int out_f32, int H, int dh, const int32_t* scope_seg,
                                   const int32_t* scope_nseg, const int32_t* seg_start,
                                   const int32_t* seg_vstart, const int32_t* scope_len,
                                   const int32_t* work, int nwork, const int32_t* scope_order,
                                   int nlive, int max_len, const int32_t* live,
                                   const uint8_t* mask, int32_t* starved, void* stream) {
    if (H < 1 || dh < 1 || dh > 128 || nwork < 0) return F3D_ERR_CONFIG;
    if (nwork == 0) return F3D_OK;
    attn::Args A;
    A.q = (const __nv_bfloat16*)q;
    A.k = (const __nv_bfloat16*)k;
    A.v = (const __nv_bfloat16*)v;
    A.ld_q = ld_q;
    A.ld_k = ld_k;
    A.ld_v = ld_v;
    A.o = o;
    A.ld_o = ld_o;
    A.dh = dh;
    A.scale_log2 = (float)(1.4426950408889634 / sqrt((double)dh));
    A.scope_seg = scope_seg;
    A.scope_nseg = scope_nseg;
    A.live = live;
    A.seg_start = seg_start;
    A.seg_vstart = seg_vstart;
    A.scope_len = scope_len;
    A.work = work;
    A.nwork = nwork;
    A.mask = mask;
    A.starved = starved;
    A.scope_order = scope_order;
    A.nlive = nlive;
    A.qsplit = 1;
    const bool vec = ((dh * 2) % 16 == 0) && (ld_q % 8 == 0) && (ld_k % 8 == 0) &&
                     (ld_v % 8 == 0) && (((uintptr_t)q | (uintptr_t)k | (uintptr_t)v) % 16 == 0);
    const bool msk = mask != nullptr;
    cudaStream_t st = (cudaStream_t)stream;
    const int dp = (dh + 15) / 16 * 16;
    // resident path: whole-scope K/V in smem (<= ~200 KB), small head dims
    const size_t res_smem = ((size_t)2 * ((max_len + 63) / 64 * 64) + 16 * attn::kResWarps) *
                            (dp * 2 + 16);
    if (vec && !msk && scope_order && nlive > 0 && dp <= 64 && res_smem <= 200 * 1024) {
        switch (dp) {
            case 16: return out_f32 ? attn::launch_resident<16, float>(A, H, max_len, st)
                                    : attn::launch_resident<16, __nv_bfloat16>(A, H, max_len, st);
            case 32: return out_f32 ? attn::launch_resident<32, float>(A, H, max_len, st)
                                    : attn::launch_resident<32, __nv_bfloat16>(A, H, max_len, st);
            case 48: return out_f32 ? attn::launch_resident<48, float>(A, H, max_len, st)
                                    : attn::launch_resident<48, __nv_bfloat16>(A, H, max_len, st);
            case 64: return out_f32 ? attn::launch_resident<64, float>(A, H, max_len, st)
                                    : attn::launch_resident<64, __nv_bfloat16>(A, H, max_len, st);
            default: break;
        }
    }
    switch (dp) {
        case 16: return attn::launch_dh<16>(A, H, vec, msk, out_f32, st);
        case 32: return attn::launch_dh<32>(A, H, vec, msk, out_f32, st);
        case 48: return attn::launch_dh<48>(A, H, vec, msk, out_f32, st);
        case 64: return attn::launch_dh<64>(A, H, vec, msk, out_f32, st);
        case 80: return attn::launch_dh<80>(A, H, vec, msk, out_f32, st);
        case 96: return attn::launch_dh<96>(A, H, vec, msk, out_f32, st);
        case 112: return attn::launch_dh<112>(A, H, vec, msk, out_f32, st);
        case 128: return attn::launch_dh<128>(A, H, vec, msk, out_f32, st);
        default: return F3D_ERR_CONFIG;
    }
}
