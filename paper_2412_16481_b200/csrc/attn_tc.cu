// Bucket-swin attention on 5th-generation tensor cores (tcgen05 / TMEM).
//
// Same contract as csrc/attn.cu (bw/attention.py:188-268 per scope, one launch
// per round), FlashAttention-style with the Blackwell execution model:
//   * persistent CTAs (one per SM) walk the (query group, head) work list; a
//     group is NQ 128-row Q tiles (NQ = 3/2/1 for dh <= 32/64/128) that
//     share every 64-key K/V tile;
//   * warps 0-2 gather Q / K / V rows of the scope straight from the fixed
//     scattered layout with cp.async into UMMA core-matrix smem tiles (a
//     scope is up to W physical segments, so rows are gathered, not boxed);
//     completion is signalled on mbarriers (cp.async.mbarrier.arrive);
//   * warp 3 (one elected thread) issues tcgen05.mma: S_g = Q_g K^T and
//     O_g = P_g V into TMEM per Q tile g, tcgen05.commit -> mbarriers;
//   * NQ softmax warpgroups (one thread per query row = TMEM lane) copy their
//     S row out of TMEM (freeing it for the next tile's MMA at once), run the
//     online softmax in the exp2 domain, write P (bf16) to smem for the PV
//     MMA, and fold O_j into register accumulators.
// Shared-memory tiles use the SWIZZLE_NONE canonical layout: element (r, c)
// of an R x C bf16 tile lives at (r/8)*16*C + (c/8)*128 + (r%8)*16 + (c%8)*2.
#include <cuda_bf16.h>

#include <algorithm>
#include <cfloat>

#include "f3d_common.cuh"
#include "tc_common.cuh"

namespace f3d {
namespace attn_tc {

using namespace f3d::tc;

constexpr int kBM = 128;          // rows per Q tile (TMEM lanes)
constexpr int kBN = 64;           // keys per K/V tile
constexpr int kLoadWarps = 3;     // warps 0-2
constexpr int kMmaWarp = 3;       // completes warpgroup 0
constexpr int kNst = 3;           // K/V stages

// Q tiles per work item (one softmax warpgroup each): as many as registers
// allow (the softmax thread keeps its 64-key S row and DH-wide O row live).
template <int DH>
__host__ __device__ constexpr int nq_for() {
    return DH <= 32 ? 3 : (DH <= 64 ? 2 : 1);
}
template <int DH>
__host__ __device__ constexpr int threads_for() {
    return (4 + 4 * nq_for<DH>()) * 32;
}

struct Args {
    const __nv_bfloat16 *q, *k, *v;
    int64_t ld_q, ld_k, ld_v;
    void* o;
    int64_t ld_o;
    int out_f32;
    int H, dh;
    float scale_log2;
    const int32_t *scope_seg, *scope_nseg, *seg_start, *seg_vstart, *scope_len, *work;
    int nwork;
    const int32_t* live;   // optional device [nwork, ...]
};

template <int DH>
struct Cfg {
    static constexpr int NQ = nq_for<DH>();
    static constexpr int kQBytes = kBM * DH * 2;        // one Q tile
    static constexpr int kKVBytes = kBN * DH * 2;       // one of K or V
    static constexpr int kPBytes = kBM * kBN * 2;       // one P tile
    static constexpr int kOffQ = 0;                     // 2 buffers x NQ Q tiles
    static constexpr int kOffKV = kOffQ + 2 * NQ * kQBytes;
    static constexpr int kOffP = kOffKV + kNst * 2 * kKVBytes;
    static constexpr int kOffBar = kOffP + NQ * kPBytes;
    static constexpr int kNumBars = 4 + 2 * kNst + 4 * NQ;
    static constexpr int kSmem = kOffBar + kNumBars * 8 + 16;
    static constexpr int kTmemS = 0;                    // S of tile g, buffer b: (2g+b)*kBN
    static constexpr int kTmemPV = 2 * NQ * kBN;        // PV of tile g: kTmemPV + g*DH
    static constexpr int kTmemCols = NQ * (2 * kBN + DH) <= 256 ? 256 : 512;
    static_assert(NQ * (2 * kBN + DH) <= 512, "TMEM budget");
    static_assert(kSmem <= 227 * 1024, "smem budget");
};

__device__ __forceinline__ int phys_row(const Args& A, int s0, int s1, int vr) {
    int seg = s0;
    for (int s = s0 + 1; s < s1; ++s)
        if (__ldg(A.seg_vstart + s) <= vr) seg = s;
    return __ldg(A.seg_start + seg) + (vr - __ldg(A.seg_vstart + seg));
}

// byte offset of 16-byte chunk (row r, chunk c) in an R x C core-matrix tile
template <int C>
__device__ __forceinline__ uint32_t core_off(int r, int c) {
    return (uint32_t)((r >> 3) * (16 * C) + c * 128 + (r & 7) * 16);
}

struct Item {
    int scope, q0, h, m, s0, s1, nt, nq;   // nq: Q tiles of this item holding real rows
};

template <int NQ>
__device__ __forceinline__ Item decode(const Args& A, int item) {
    Item it;
    const int wi = item / A.H;
    it.h = item - wi * A.H;
    it.scope = __ldg(A.work + 2 * wi);
    it.q0 = __ldg(A.work + 2 * wi + 1);
    it.s0 = __ldg(A.scope_seg + it.scope);
    it.s1 = it.s0 + __ldg(A.scope_nseg + it.scope);
    it.m = __ldg(A.scope_len + it.scope);
    it.nt = (it.m + kBN - 1) / kBN;
    it.nq = min(NQ, (it.m - it.q0 + kBM - 1) / kBM);
    return it;
}

// Gather rows [v0, v0+R) of head h (real chunks only; zero-fill past m).
template <int DH, int R>
__device__ __forceinline__ void gather(const Args& A, const __nv_bfloat16* base, int64_t ld,
                                       const Item& it, int v0, uint32_t dst, int tid) {
    const int rc = A.dh >> 3;   // real 16-byte chunks per row
    const int hcol = it.h * A.dh;
    for (int idx = tid; idx < R * rc; idx += kLoadWarps * 32) {
        const int r = idx / rc;
        const int c = idx - r * rc;
        const int vr = v0 + r;
        const bool ok = vr < it.m;
        const __nv_bfloat16* src = base;
        if (ok) src = base + (int64_t)phys_row(A, it.s0, it.s1, vr) * ld + hcol + c * 8;
        cp_async16z(dst + core_off<DH>(r, c), src, ok);
    }
}

template <int DH, typename OutT>
__global__ void __launch_bounds__(threads_for<DH>(), 1) bswin_attn_tc_kernel(const Args A) {
    using C = Cfg<DH>;
    constexpr int NQ = C::NQ;
    constexpr int kThreads = threads_for<DH>();
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    // every barrier below completes at most one phase ahead of its waiter
    uint64_t* q_full = bars + 0;                 // [2] loaders -> MMA (Q buffer filled)
    uint64_t* q_empty = bars + 2;                // [2] MMA -> loaders (Q buffer consumed)
    uint64_t* kv_full = bars + 4;                // [kNst]
    uint64_t* kv_empty = bars + 4 + kNst;        // [kNst]
    uint64_t* s_full = bars + 4 + 2 * kNst;      // [NQ][2] MMA -> softmax (S_g in buffer b)
    uint64_t* p_full = s_full + 2 * NQ;          // [NQ] softmax -> MMA (P_g written, S read,
                                                 //      previous P_g V folded)
    uint64_t* pv_full = s_full + 3 * NQ;         // [NQ] MMA -> softmax (P_g V ready)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::kNumBars);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int total = (A.live ? __ldg(A.live) : A.nwork) * A.H;

    // zero the operand tiles once: pad chunks (dh < DH) are never written again
    for (int i = tid; i < C::kOffBar / 16; i += kThreads)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(q_full + b, kLoadWarps * 32);
            mbar_init(q_empty + b, 1);
        }
        for (int s = 0; s < kNst; ++s) {
            mbar_init(kv_full + s, kLoadWarps * 32);
            mbar_init(kv_empty + s, 1);
        }
        for (int g = 0; g < NQ; ++g) {
            mbar_init(s_full + 2 * g, 1);
            mbar_init(s_full + 2 * g + 1, 1);
            mbar_init(p_full + g, 128);
            mbar_init(pv_full + g, 1);
        }
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(tmem_slot, C::kTmemCols);
        tmem_relinquish();
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sm_base = saddr(smem);

    if (warp < kLoadWarps) {
        // ------------------------------------------------ loader warps
        uint32_t q_use = 0, kv_it = 0;
        for (int item = blockIdx.x; item < total; item += gridDim.x) {
            const Item it = decode<NQ>(A, item);
            const int qb = q_use & 1;
            mbar_wait(q_empty + qb, ((q_use >> 1) & 1) ^ 1);
            for (int g = 0; g < it.nq; ++g)
                gather<DH, kBM>(A, A.q, A.ld_q, it, it.q0 + g * kBM,
                                sm_base + C::kOffQ + (qb * NQ + g) * C::kQBytes, tid);
            cp_async_arrive(q_full + qb);
            ++q_use;
            for (int j = 0; j < it.nt; ++j, ++kv_it) {
                const int s = kv_it % kNst;
                const uint32_t u = kv_it / kNst;
                mbar_wait(kv_empty + s, (u & 1) ^ 1);
                const uint32_t kb = sm_base + C::kOffKV + s * 2 * C::kKVBytes;
                gather<DH, kBN>(A, A.k, A.ld_k, it, j * kBN, kb, tid);
                gather<DH, kBN>(A, A.v, A.ld_v, it, j * kBN, kb + C::kKVBytes, tid);
                cp_async_arrive(kv_full + s);
            }
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------ MMA warp (one thread)
        if (lane == 0) {
            constexpr uint32_t idS = idesc_bf16(kBM, kBN, 0, 0);
            constexpr uint32_t idPV = idesc_bf16(kBM, DH, 0, 1);
            uint32_t q_use = 0, kv_it = 0;
            uint32_t tg[NQ];                     // tiles processed by group g so far
#pragma unroll
            for (int g = 0; g < NQ; ++g) tg[g] = 0;
            for (int item = blockIdx.x; item < total; item += gridDim.x) {
                const Item it = decode<NQ>(A, item);
                const int qb = q_use & 1;
                mbar_wait(q_full + qb, (q_use >> 1) & 1);
                // S_g,j -> TMEM buffer (tg[g]+j)&1.  Reusing that buffer needs
                // softmax g done with S_g,j-2: implied by p_full_g,j-2, waited
                // before PV_g,j-2 was issued.
                auto issue_S = [&](int g, int j) {
                    const int s = (kv_it + j) % kNst;
                    const int b = (tg[g] + j) & 1;
                    const uint32_t kb = sm_base + C::kOffKV + s * 2 * C::kKVBytes;
                    const uint32_t qa = sm_base + C::kOffQ + (qb * NQ + g) * C::kQBytes;
#pragma unroll
                    for (int k = 0; k < DH / 16; ++k)
                        umma_f16(tmem + C::kTmemS + (2 * g + b) * kBN,
                                 smem_desc(qa + k * 256, 128, 16 * DH),
                                 smem_desc(kb + k * 256, 128, 16 * DH), idS, k > 0);
                    umma_commit(s_full + 2 * g + b);
                };
                auto wait_kv = [&](int j) {
                    const uint32_t kvi = kv_it + j;
                    mbar_wait(kv_full + kvi % kNst, (kvi / kNst) & 1);
                    tc_fence_after();
                };
                wait_kv(0);
                for (int g = 0; g < it.nq; ++g) issue_S(g, 0);
                for (int j = 0; j < it.nt; ++j) {
                    const int s = (kv_it + j) % kNst;
                    const uint32_t vb = sm_base + C::kOffKV + s * 2 * C::kKVBytes + C::kKVBytes;
                    if (j + 1 < it.nt) {
                        wait_kv(j + 1);
                        for (int g = 0; g < it.nq; ++g) issue_S(g, j + 1);
                    }
                    for (int g = 0; g < it.nq; ++g) {
                        mbar_wait(p_full + g, (tg[g] + j) & 1);           // P_g,j in smem
                        tc_fence_after();
                        const uint32_t pb = sm_base + C::kOffP + g * C::kPBytes;
#pragma unroll
                        for (int k = 0; k < kBN / 16; ++k)
                            umma_f16(tmem + C::kTmemPV + g * DH,
                                     smem_desc(pb + k * 256, 128, 16 * kBN),
                                     smem_desc(vb + k * 32 * DH, 16 * DH, 128), idPV, k > 0);
                        umma_commit(pv_full + g);
                    }
                    umma_commit(kv_empty + s);
                }
                umma_commit(q_empty + qb);
                ++q_use;
                kv_it += it.nt;
                for (int g = 0; g < it.nq; ++g) tg[g] += it.nt;
            }
        }
    } else {
        // ------------------------------------------------ softmax warpgroups
        const int sw = warp - (kMmaWarp + 1);             // 0 .. 4*NQ-1
        const int g = sw >> 2;                            // Q tile of this warpgroup
        const int r = (sw & 3) * 32 + lane;               // row in the tile = TMEM lane
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const float sl2 = A.scale_log2;
        const uint32_t vbase = tmem + lane_base + C::kTmemPV + g * DH;
        const uint32_t pb = sm_base + C::kOffP + g * C::kPBytes;
        uint32_t tg = 0;
        for (int item = blockIdx.x; item < total; item += gridDim.x) {
            const Item it = decode<NQ>(A, item);
            if (g >= it.nq) continue;                     // this Q tile is past the scope
            float o[DH];
#pragma unroll
            for (int i = 0; i < DH; ++i) o[i] = 0.f;
            float m_run = -INFINITY, l_run = 0.f, alpha_prev = 0.f;
            for (int j = 0; j < it.nt; ++j) {
                const uint32_t t = tg + j;
                const int b = t & 1;
                mbar_wait(s_full + 2 * g + b, (t >> 1) & 1);
                tc_fence_after();
                uint32_t x[kBN];
                {
                    const uint32_t sb = tmem + lane_base + C::kTmemS + (2 * g + b) * kBN;
                    uint32_t (&x0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&x[0]);
                    uint32_t (&x1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&x[32]);
                    tmem_ld32(sb, x0);
                    tmem_ld32(sb + 32, x1);
                    tmem_wait_ld();
                }
                const int kvalid = it.m - j * kBN;        // keys < kvalid are real
                if (kvalid < kBN) {
#pragma unroll
                    for (int e = 0; e < kBN; ++e)
                        if (e >= kvalid) x[e] = __float_as_uint(-INFINITY);
                }
                float mx = -INFINITY;
#pragma unroll
                for (int e = 0; e < kBN; ++e) mx = fmaxf(mx, __uint_as_float(x[e]));
                const float m_new = fmaxf(m_run, mx);
                const float alpha = (m_run == -INFINITY) ? 0.f : ex2f((m_run - m_new) * sl2);
                const float nms = -m_new * sl2;
                // fold the previous tile's P V (this also frees P_g for overwrite)
                if (j > 0) {
                    mbar_wait(pv_full + g, (t - 1) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int c = 0; c < DH / 16; ++c) {
                        uint32_t y[16];
                        tmem_ld16(vbase + c * 16, y);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 16; ++e)
                            o[c * 16 + e] = fmaf(o[c * 16 + e], alpha_prev, __uint_as_float(y[e]));
                    }
                }
                // P = exp2(s*sl2 - m*sl2) -> bf16 smem (core-matrix rows)
                float sum = 0.f;
#pragma unroll
                for (int c = 0; c < kBN / 8; ++c) {
                    uint32_t pk[4];
#pragma unroll
                    for (int e = 0; e < 8; e += 2) {
                        const float p0 = ex2f(fmaf(__uint_as_float(x[c * 8 + e]), sl2, nms));
                        const float p1 = ex2f(fmaf(__uint_as_float(x[c * 8 + e + 1]), sl2, nms));
                        sum += p0 + p1;
                        __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
                        pk[e >> 1] = *reinterpret_cast<uint32_t*>(&h2);
                    }
                    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(pb + core_off<kBN>(r, c)),
                                 "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3])
                                 : "memory");
                }
                fence_proxy_async();
                tc_fence_before();
                mbar_arrive(p_full + g);
                l_run = l_run * alpha + sum;
                m_run = m_new;
                alpha_prev = alpha;
            }
            // last tile's P V, then normalise and write the row
            {
                mbar_wait(pv_full + g, (tg + it.nt - 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < DH / 16; ++c) {
                    uint32_t y[16];
                    tmem_ld16(vbase + c * 16, y);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        o[c * 16 + e] = fmaf(o[c * 16 + e], alpha_prev, __uint_as_float(y[e]));
                }
            }
            const int vr = it.q0 + g * kBM + r;
            if (vr < it.m) {
                const int pr = phys_row(A, it.s0, it.s1, vr);
                const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
                const int hcol = it.h * A.dh;
                if (sizeof(OutT) == 2) {
                    __nv_bfloat16* out =
                        reinterpret_cast<__nv_bfloat16*>(A.o) + (int64_t)pr * A.ld_o + hcol;
#pragma unroll
                    for (int c = 0; c < DH; c += 2)
                        if (c < A.dh)
                            *reinterpret_cast<__nv_bfloat162*>(out + c) =
                                __floats2bfloat162_rn(o[c] * inv, o[c + 1] * inv);
                } else {
                    float* out = reinterpret_cast<float*>(A.o) + (int64_t)pr * A.ld_o + hcol;
#pragma unroll
                    for (int c = 0; c < DH; ++c)
                        if (c < A.dh) out[c] = o[c] * inv;
                }
            }
            tg += it.nt;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, C::kTmemCols);
}

template <int DH, typename OutT>
int launch(const Args& A, cudaStream_t st) {
    using C = Cfg<DH>;
    auto kern = bswin_attn_tc_kernel<DH, OutT>;
    static bool attr = false;
    if (!attr) {
        F3D_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          C::kSmem));
        attr = true;
    }
    const int total = A.nwork * A.H;
    const int grid = std::max(1, std::min(total, f3d_num_sms()));
    kern<<<grid, threads_for<DH>(), C::kSmem, st>>>(A);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

template <int DH>
int launch_dh(const Args& A, cudaStream_t st) {
    return A.out_f32 ? launch<DH, float>(A, st) : launch<DH, __nv_bfloat16>(A, st);
}

}  // namespace attn_tc
}  // namespace f3d

using namespace f3d;

extern "C" int f3d_attention_tc_qstep(int dh) {
    const int dp = (dh + 15) / 16 * 16;
    const int nq = dp <= 32 ? 3 : (dp <= 64 ? 2 : 1);
    return nq * f3d::attn_tc::kBM;
}

extern "C" int f3d_bswin_attention_tc(const void* q, const void* k, const void* v, int64_t ld_q,
                                      int64_t ld_k, int64_t ld_v, void* o, int64_t ld_o,
                                      int out_f32, int H, int dh, const int32_t* scope_seg,
                                      const int32_t* scope_nseg, const int32_t* seg_start,
                                      const int32_t* seg_vstart, const int32_t* scope_len,
                                      const int32_t* work, int nwork, const int32_t* live,
                                      void* stream) {
    if (H < 1 || dh < 8 || dh > 128 || (dh & 7) || nwork < 0) return F3D_ERR_CONFIG;
    if (((uintptr_t)q | (uintptr_t)k | (uintptr_t)v) & 15) return F3D_ERR_CONFIG;
    if ((ld_q | ld_k | ld_v) & 7) return F3D_ERR_CONFIG;
    if (nwork == 0) return F3D_OK;
    attn_tc::Args A;
    A.q = (const __nv_bfloat16*)q;
    A.k = (const __nv_bfloat16*)k;
    A.v = (const __nv_bfloat16*)v;
    A.ld_q = ld_q;
    A.ld_k = ld_k;
    A.ld_v = ld_v;
    A.o = o;
    A.ld_o = ld_o;
    A.out_f32 = out_f32;
    A.H = H;
    A.dh = dh;
    A.scale_log2 = (float)(1.4426950408889634 / sqrt((double)dh));
    A.scope_seg = scope_seg;
    A.scope_nseg = scope_nseg;
    A.seg_start = seg_start;
    A.seg_vstart = seg_vstart;
    A.scope_len = scope_len;
    A.work = work;
    A.nwork = nwork;
    A.live = live;
    cudaStream_t st = (cudaStream_t)stream;
    switch ((dh + 15) / 16 * 16) {
        case 16: return attn_tc::launch_dh<16>(A, st);
        case 32: return attn_tc::launch_dh<32>(A, st);
        case 48: return attn_tc::launch_dh<48>(A, st);
        case 64: return attn_tc::launch_dh<64>(A, st);
        case 80: return attn_tc::launch_dh<80>(A, st);
        case 96: return attn_tc::launch_dh<96>(A, st);
        case 112: return attn_tc::launch_dh<112>(A, st);
        case 128: return attn_tc::launch_dh<128>(A, st);
        default: return F3D_ERR_CONFIG;
    }
}
