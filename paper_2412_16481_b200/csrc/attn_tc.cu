// Bucket-swin attention on 5th-generation tensor cores (tcgen05 / TMEM / TMA).
//
// Same contract as csrc/attn.cu (bw/attention.py:188-268 per scope, one launch
// per round), FlashAttention-style with the Blackwell execution model:
//   * persistent CTAs (one per SM) walk the (query group, head) work list; a
//     group is NQ = 2 128-row Q tiles that share every 64-key K/V tile;
//   * loads: a scope is the concatenation of up to W physical row segments of
//     the fixed scattered layout (adjacent buckets are merged, so most scopes
//     are one segment).  A tile whose rows lie inside one segment is fetched
//     by TMA (one elected thread, 2-D boxes of the head's columns, swizzled
//     straight into the UMMA operand layout); a tile that straddles two
//     segments or runs past the scope end is gathered row by row with
//     cp.async (zero-filled past m) by warps 0-2.  Both complete on the
//     same mbarrier (96 cp.async arrivals + one elected arrive[.expect_tx]);
//   * warp 3 walks the schedule and one elected lane issues tcgen05.mma:
//     S_g = Q_g K^T into one of NSB TMEM S buffers per Q tile, then
//     O_g += P_g V with P_g read from TMEM (the softmax writes it over S_g) and
//     O_g accumulated in TMEM across all key tiles; tcgen05.commit ->
//     mbarriers;
//   * NQ softmax warpgroups (thread = query row = TMEM lane) read S with
//     tcgen05.ld, run the online softmax in the exp2 domain, and store P as
//     bf16 back into TMEM.  The running max only moves (and O is rescaled in
//     TMEM) when a row's max grows by more than 2^8.  When the head dim is
//     padded (dh < DH) a ones column in V makes the PV MMA produce the row
//     sums, so the softmax does no per-score add.
// Operand tiles use the UMMA swizzled layouts (SW = 2*min(DH,64) bytes per
// row): Q and K K-major, V MN-major; a 128-wide head is two 64-column blocks.
// Element (r, c) of an R-row tile: block b = c / BW, byte o = r*SW + (c%BW)*2,
// o ^= ((o >> 7) & (SW/16 - 1)) << 4, at b*R*SW + o (Swizzle<log2(SW/16),4,3>).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cfloat>
#include <cstring>

#include "f3d_common.cuh"
#include "tc_common.cuh"

#ifndef F3D_EXPERIMENT
#define F3D_EXPERIMENT 0   // developer A/B knob (tools/): 1 no loads, 2 no exp,
#endif                     // 3 per-role wait-cycle counters (f3d_attn_prof)
#if F3D_EXPERIMENT == 4
// per softmax warp of CTA 0: clock at S ready, exp start, exp end of its first 96 tiles
__device__ long long g_attn_trace[16][96][3];
// per softmax warp of CTA 0 and item: next_item returned, final pv wait start, epilogue start, end
__device__ long long g_attn_trace2[16][16][8];
#endif
#if F3D_EXPERIMENT == 3
__device__ unsigned long long g_attn_prof[24];
#define PROF_MARK(var) const long long var = clock64()
#define PROF_ADD(slot, a, b) if ((threadIdx.x & 31) == 0) prof[slot] += (b) - (a)
#define PROF_WAIT(slot, call)                                            \
    do {                                                                 \
        const long long _t0 = clock64();                                 \
        call;                                                            \
        if ((threadIdx.x & 31) == 0) prof[slot] += clock64() - _t0;      \
    } while (0)
#else
#define PROF_WAIT(slot, call) call
#define PROF_MARK(var)
#define PROF_ADD(slot, a, b)
#endif

namespace f3d {
namespace attn_tc {

using namespace f3d::tc;

constexpr int kBM = 128;          // rows per Q tile (TMEM lanes)
#ifndef F3D_BN_SMALL
#define F3D_BN_SMALL 64    // keys per K/V tile for head dims <= 32
#endif
// keys per K/V tile (S tile columns)
template <int DH>
__host__ __device__ constexpr int bn_for() { return DH <= 32 ? F3D_BN_SMALL : 64; }
#ifndef F3D_NQ_SMALL
#define F3D_NQ_SMALL 3     // Q tiles per work item for head dims <= 32 (measured: 3 > 2 by 1-4 %)
#endif
// Q tiles per work item (one softmax warpgroup each)
__host__ __device__ constexpr int nq_for_dh(int DH) { return DH <= 32 ? F3D_NQ_SMALL : 2; }
constexpr int kLoadWarps = 1;     // warp 0
constexpr int kLoadThreads = kLoadWarps * 32;
// Warps 1..NQ issue the MMAs of Q tile g = warp - 1 (one issuing thread each):
// measured (tools/ubench/mma_ts.cu) one thread issues at most one M128 N<=64
// tcgen05.mma per ~45 clk, two threads reach the tensor pipe's own rate --
// one issuer for all Q tiles was the co-bottleneck at small head dims.
// warps before the softmax warpgroups: the loader and the NQ issuers, at least
// one whole warpgroup (the softmax warps' TMEM lane quarter is warp % 4)
__host__ __device__ constexpr int pre_warps(int nq) { return nq + 1 > 4 ? nq + 1 : 4; }
// Softmax column split: CS warps share each 32-row lane quarter of a Q tile
// and take kBN/CS key columns each (row max / sum exchanged through shared
// memory) -- more warps per SM sub-partition to hide the per-tile latencies
// of the exp-bound small-head softmax.
template <int DH>
__host__ __device__ constexpr int cs_for() {
    return DH == 64 ? 2 : 1;   // measured: DH 64 451 -> 492 TFLOP/s; DH 32 (0.165 -> 0.185 ms) and DH 128 (948 -> 919) slower
}
// Resident CTAs per SM for head dims <= 32 (A/B knob): with several small
// CTAs (NQ = 1 each) the softmax warps of an SM sub-partition belong to
// different, independently progressing CTAs instead of three Q tiles of one
// item that advance in lock step.
#ifndef F3D_CTAS_SMALL
#define F3D_CTAS_SMALL 1
#endif
template <int DH>
__host__ __device__ constexpr int ctas_per_sm() { return DH <= 32 ? F3D_CTAS_SMALL : 1; }
template <int DH>
__host__ __device__ constexpr int threads_for() {
    return (pre_warps(nq_for_dh(DH)) + 4 * nq_for_dh(DH) * cs_for<DH>()) * 32;
}
constexpr float kRescale = 8.f;   // move the running max only when it grows by > 2^8
constexpr int kMaps = 6;          // TMA maps: {q, k, v} x {first block, second block}
// 1 pair in poly_every<DH>() uses ex2_poly (0: none).  Measured (config B
// dh=24, one round: 1 in 3 0.138 ms, 1 in 4 0.140, 1 in 2 0.146, none 0.154;
// config D dh=128: 7 % slower): the softmax is issue-bound, not MUFU-bound,
// once dh >= 64.
#ifndef F3D_POLY_SMALL
#define F3D_POLY_SMALL 3
#endif
#ifndef F3D_POLY_MID
#define F3D_POLY_MID 0
#endif
#ifndef F3D_POLY_LARGE
#define F3D_POLY_LARGE 0
#endif
template <int DH>
__host__ __device__ constexpr int poly_every() {
    return DH <= 32 ? F3D_POLY_SMALL : DH <= 64 ? F3D_POLY_MID : F3D_POLY_LARGE;
}


// 2^x of a packed pair on the FMA/ALU pipes for x <= 2^8 (softmax arguments): round x to
// j = rint(x) with the 1.5*2^23 trick, 2^f for f in [-0.5, 0.5] by a cubic
// (relative error <= 8e-4, below the bf16 rounding of P), exponent added
// as an integer.  Arguments below -127 flush to 0 like ex2.approx.ftz.
// The rounding trick and the cubic run as f32x2.
__device__ __forceinline__ void ex2_poly2(uint64_t a, float& p0, float& p1) {
    float x0, x1;
    f2_split(a, x0, x1);
    const uint64_t x = f2(fmaxf(x0, -127.f), fmaxf(x1, -127.f));
    const uint64_t C = f2(12582912.f, 12582912.f);
    const uint64_t t = fadd2(x, C);
    const uint64_t f = fsub2(x, fsub2(t, C));
    uint64_t p = ffma2(f2(0.0555041086648216f, 0.0555041086648216f), f,
                       f2(0.2402264923172690f, 0.2402264923172690f));
    p = ffma2(p, f, f2(0.6931471805599453f, 0.6931471805599453f));
    p = ffma2(p, f, f2(1.f, 1.f));
    float q0, q1, t0, t1;
    f2_split(p, q0, q1);
    f2_split(t, t0, t1);
    p0 = __int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23));
    p1 = __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23));
}

__host__ __device__ constexpr int dh_tile(int dh) {   // padded head dim of the kernel
    return dh <= 16 ? 16 : dh <= 32 ? 32 : dh <= 64 ? 64 : 128;
}

// Swizzled operand layout of a DH-wide head.
template <int DH>
struct Lay {
    static constexpr int SW = DH >= 64 ? 128 : 2 * DH;  // bytes per block row (= swizzle span)
    static constexpr int BW = SW / 2;                   // elements per block row
    static constexpr int NBLK = DH / BW;
    static constexpr int XM = SW / 16 - 1;              // swizzle xor mask (16-byte chunks)
    static constexpr uint32_t LT = SW == 128 ? 2u : (SW == 64 ? 4u : 6u);   // UMMA layout type
    // byte offset of 16-byte chunk c of row r in an R-row tile
    template <int R>
    static __device__ __forceinline__ uint32_t off(int r, int c) {
        const int b = c / (BW / 8), cc = c - b * (BW / 8);
        uint32_t o = (uint32_t)(r * SW + cc * 16);
        o ^= ((o >> 7) & XM) << 4;
        return (uint32_t)(b * R * SW) + o;
    }
};


// Dynamic work distribution (when the plan's live words are given): warp 0
// takes items from a global counter (live[4]) as it is about to load them and
// hands them to the MMA / softmax warps through a ring of shared-memory slots.
// The last CTA to finish resets the counters (live[4], live[5]) for the next
// launch on the plan.  Measured without it (static item += gridDim.x): the
// softmax warps of the busiest CTAs ran 15 % longer than the average.
constexpr int kItemRing = 4;
// Item records in shared memory, written by warp 0 when it takes an item:
// the decoded item and its segment table, so the MMA / softmax warps never
// chase the work list / scope / segment arrays through global memory (two to
// four dependent L2 round trips at every item start and in the epilogue's
// row mapping).  A slot is held until its consumers finished the item.
constexpr int kMaxSeg = 8;                    // scopes with more segments map rows from global
constexpr int kRecInts = 32;                  // 9 fields + 2 * kMaxSeg, padded
enum { R_ITEM = 0, R_SCOPE, R_Q0, R_H, R_M, R_S0, R_S1, R_NT, R_NQ, R_VST, R_ST = R_VST + kMaxSeg };

template <int DH>
__host__ __device__ constexpr int nsb_for() {
    return nq_for_dh(DH) * (3 * bn_for<DH>() + DH) <= 512 ? 3 : 2;
}

struct Maps {
    CUtensorMap m[kMaps];
};

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
    int use_tma;
    int o_vec;             // output rows allow 16-byte stores
    float* lse;            // optional: per (row, head) log2-domain logsumexp (training)
    int64_t ld_lse;
};

template <int DH>
struct Cfg {
    static constexpr int kBN = bn_for<DH>();
    static constexpr int NQ = nq_for_dh(DH);
    static constexpr int NSB = nsb_for<DH>();
    static constexpr int kQBytes = kBM * DH * 2;        // one Q tile
    static constexpr int kKVBytes = kBN * DH * 2;       // one of K or V
    static constexpr int CS = cs_for<DH>();
    static constexpr int kXchg = CS > 1 ? NQ * 4 * 3 * CS * 32 * 4 : 0;   // pair exchange
    static constexpr int kRecBytes = kItemRing * kRecInts * 4;
    static constexpr int kBudget = 227 * 1024 / ctas_per_sm<DH>() - 1024 - 512 - kXchg - kRecBytes;
    // K/V depth first (>= 4 stages), then a second Q buffer if it still fits
    static constexpr int NQB = (2 * NQ * kQBytes + 4 * 2 * kKVBytes <= kBudget) ? 2 : 1;
    static constexpr int kNstFit = (kBudget - NQB * NQ * kQBytes) / (2 * kKVBytes);
    static constexpr int kNst = kNstFit > 6 ? 6 : kNstFit;
    static constexpr int kOffQ = 0;
    static constexpr int kOffKV = kOffQ + NQB * NQ * kQBytes;
    static constexpr int kOffBar = kOffKV + kNst * 2 * kKVBytes;
    static constexpr int kNumBars = 2 * NQB + 2 * kNst + (3 * NSB + 1) * NQ + 2 * kItemRing;
    // after the barriers: TMEM address word, kItemRing item slots
    // pair exchange: [NQ][4 quarters][2 parities][CS][32] row maxima, + row sums
    static constexpr int kOffX = kOffBar + kNumBars * 8 + 4 + 4 * kItemRing + 12;
    static constexpr int kOffRec = kOffX + kXchg;
    static constexpr int kSmem = kOffRec + kRecBytes + 1024;   // + 1 KB alignment slack
    static constexpr int kTmemS = 0;                    // S/P of tile g, buffer b: (NSB*g+b)*kBN
    static constexpr int kTmemO = NSB * NQ * kBN;       // O of tile g: kTmemO + g*DH
    static constexpr int kTmemNeed = NQ * (NSB * kBN + DH);
    static constexpr int kTmemCols = kTmemNeed <= 32 ? 32 : kTmemNeed <= 64 ? 64
                                     : kTmemNeed <= 128 ? 128 : kTmemNeed <= 256 ? 256 : 512;
    static_assert(kTmemCols * ctas_per_sm<DH>() <= 512, "TMEM for the resident CTAs");
    static_assert(NQ * (NSB * kBN + DH) <= 512, "TMEM budget");
    static_assert(kNst >= 2, "K/V pipeline depth");
    static_assert(kSmem <= 227 * 1024, "smem budget");
};

__device__ __forceinline__ int phys_row(const Args& A, int s0, int s1, int vr) {
    int seg = s0;
    for (int s = s0 + 1; s < s1; ++s)
        if (__ldg(A.seg_vstart + s) <= vr) seg = s;
    return __ldg(A.seg_start + seg) + (vr - __ldg(A.seg_vstart + seg));
}

struct Item {
    int scope, q0, h, m, s0, s1, nt, nq;   // nq: Q tiles of this item holding real rows
};

template <int NQ, int kBN>
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

__device__ __forceinline__ Item rec_item(const volatile int* R) {
    Item it;
    it.scope = R[R_SCOPE];
    it.q0 = R[R_Q0];
    it.h = R[R_H];
    it.m = R[R_M];
    it.s0 = R[R_S0];
    it.s1 = R[R_S1];
    it.nt = R[R_NT];
    it.nq = R[R_NQ];
    return it;
}

// phys_row from the item record's segment table
__device__ __forceinline__ int phys_row_rec(const Args& A, const volatile int* R, const Item& it, int vr) {
    const int nseg = it.s1 - it.s0;
    if (nseg > kMaxSeg) return phys_row(A, it.s0, it.s1, vr);
    int k = 0;
    for (int i = 1; i < nseg; ++i)
        if (R[R_VST + i] <= vr) k = i;
    return R[R_ST + k] + (vr - R[R_VST + k]);
}

// First physical row of [v0, v0 + R) if those virtual rows lie inside one
// segment (so inside the scope, all real): the tile can be one TMA box.
__device__ __forceinline__ int tile_run(const Args& A, const Item& it, int v0, int R) {
    int seg = it.s0;
    for (int s = it.s0 + 1; s < it.s1; ++s)
        if (__ldg(A.seg_vstart + s) <= v0) seg = s;
    const int vs = __ldg(A.seg_vstart + seg);
    const int ve = seg + 1 < it.s1 ? __ldg(A.seg_vstart + seg + 1) : it.m;
    return v0 + R <= ve ? __ldg(A.seg_start + seg) + (v0 - vs) : -1;
}

// cp.async fallback: rows [v0, v0+R) of head h, one row per loader thread,
// real 16-byte chunks only, zero-filled past m.
template <int DH, int R>
__device__ __forceinline__ void gather_rows(const Args& A, const __nv_bfloat16* base, int64_t ld,
                                            const Item& it, int v0, uint32_t dst, int tid) {
#if F3D_EXPERIMENT == 1
    return;
#endif
    const int rc = A.dh >> 3;
    for (int r = tid; r < R; r += kLoadThreads) {
        const int vr = v0 + r;
        const bool ok = vr < it.m;
        const __nv_bfloat16* src = base;
        if (ok) src = base + (int64_t)phys_row(A, it.s0, it.s1, vr) * ld + it.h * A.dh;
        for (int c = 0; c < rc; ++c)
            cp_async16z(dst + Lay<DH>::template off<R>(r, c), src + c * 8, ok);
    }
}


// TMA of rows [p0, p0 + R) of head h (map pair mp: q=0, k=2, v=4) into a
// tile of R rows: one box of 64 rows per column block and 64-row slab.
template <int DH, int R, int BOX>
__device__ __forceinline__ void tma_rows(const Maps& M, int mp, const Args& A, int h, int p0,
                                         uint32_t dst, uint64_t* bar) {
    using L = Lay<DH>;
    static_assert(R % BOX == 0, "tile rows in whole boxes");
    const int c0 = h * A.dh;
#pragma unroll
    for (int b = 0; b < L::NBLK; ++b) {
        if (b * L::BW >= A.dh) break;
#pragma unroll
        for (int s = 0; s < R / BOX; ++s)
            tma_2d(dst + b * R * L::SW + s * BOX * L::SW, &M.m[mp + b], bar, c0 + b * L::BW,
                   p0 + s * BOX);
    }
}

// ONES: dh < DH, the row sums come from the ones column of V (a compile-time
// flag: with a runtime one the compiler kept the per-score sum adds in the exp
// loop and selected the result afterwards -- 2 dead FADDs per pair).
template <int DH, typename OutT, bool ONES>
__global__ void __launch_bounds__(threads_for<DH>(), ctas_per_sm<DH>())
    bswin_attn_tc_kernel(const Args A, const __grid_constant__ Maps M) {
    using C = Cfg<DH>;
    using L = Lay<DH>;
    constexpr int NQ = C::NQ;
    constexpr int NQB = C::NQB;
    constexpr int NSB = C::NSB;
    constexpr int kNst = C::kNst;
    constexpr int CS = C::CS;
    constexpr int kBN = C::kBN;
    constexpr int kThreads = threads_for<DH>();
    extern __shared__ unsigned char smem_raw[];
    // swizzled tiles need 1024-byte aligned bases
    unsigned char* smem = smem_raw + ((1024 - (saddr(smem_raw) & 1023)) & 1023);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    // every barrier below completes at most one phase ahead of its waiter
    uint64_t* q_full = bars;                     // [NQB] loaders -> MMA
    uint64_t* q_empty = q_full + NQB;            // [NQB] MMA -> loaders
    uint64_t* kv_full = q_empty + NQB;           // [kNst]
    uint64_t* kv_empty = kv_full + kNst;         // [kNst]
    uint64_t* s_full = kv_empty + kNst;          // [NQ][NSB] MMA -> softmax (S_g in buffer b)
    // [NQ][NSB] softmax -> MMA: P_g,t in TMEM buffer t%NSB (O rescaled).  Per
    // buffer, because the softmax may finish tiles t+1.. before the MMA
    // thread has consumed tile t (S_g,t .. S_g,t+NSB-1 are all in flight).
    uint64_t* p_full = s_full + NSB * NQ;
    // [NQ][NSB] MMA -> softmax: O_g += P_g,t V done, on buffer t%NSB.  A
    // waiter for PV_g,t has already seen S_g,t+1 complete, which was issued
    // after PV_g,t+1-NSB: so the barrier is never a phase behind either.
    uint64_t* pv_done = p_full + NSB * NQ;
    uint64_t* o_free = pv_done + NSB * NQ;       // [NQ] softmax -> MMA (O_g read out)
    uint64_t* item_full = o_free + NQ;           // [kItemRing] warp 0 -> consumers
    uint64_t* item_empty = item_full + kItemRing;   // [kItemRing] consumers -> warp 0
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::kNumBars);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    int total = 0;                               // work items (read after pdl_wait)
    const bool dyn = A.live != nullptr;
    int32_t* sched = dyn ? const_cast<int32_t*>(A.live) + 4 : nullptr;   // [next item, CTAs done]
    // consumers of each item: the NQ MMA issuers and every softmax warp
    constexpr int kConsumers = NQ + 4 * NQ * CS;
    // the CTA's item sequence (static round robin, or the global counter) is
    // taken by warp 0 and handed to the MMA / softmax warps through a ring of
    // shared-memory item records
    uint32_t item_k = 0;
    int item_static = blockIdx.x;
    int* recs = reinterpret_cast<int*>(smem + C::kOffRec);
    // next record slot (-1: no more items); a consumer releases its slot with
    // release_slot once done with the item
    auto next_slot = [&]() -> int {
        const int slot = item_k % kItemRing;
        const uint32_t ph = (item_k / kItemRing) & 1;
        ++item_k;
        volatile int* R = recs + slot * kRecInts;
        if (warp == 0) {                       // producer
            if (item_k > kItemRing) mbar_wait(item_empty + slot, ph ^ 1);
            int r = 0;
            if (lane == 0) {
                if (dyn) {
                    r = atomicAdd(sched, 1);
                } else {
                    r = item_static;
                    item_static += gridDim.x;
                }
                if (r >= total) r = -1;
                R[R_ITEM] = r;
                if (r >= 0) {
                    const Item it = decode<NQ, kBN>(A, r);
                    R[R_SCOPE] = it.scope;
                    R[R_Q0] = it.q0;
                    R[R_H] = it.h;
                    R[R_M] = it.m;
                    R[R_S0] = it.s0;
                    R[R_S1] = it.s1;
                    R[R_NT] = it.nt;
                    R[R_NQ] = it.nq;
                    const int nseg = min(it.s1 - it.s0, kMaxSeg);
                    for (int i = 0; i < nseg; ++i) {
                        R[R_VST + i] = __ldg(A.seg_vstart + it.s0 + i);
                        R[R_ST + i] = __ldg(A.seg_start + it.s0 + i);
                    }
                }
                mbar_arrive(item_full + slot);
            }
            r = __shfl_sync(0xffffffffu, r, 0);
            return r < 0 ? -1 : slot;
        }
        mbar_wait(item_full + slot, ph);
        const int r = R[R_ITEM];
        __syncwarp();
        return r < 0 ? -1 : slot;
    };
    auto release_slot = [&](int slot) {
        __syncwarp();
        if (lane == 0) mbar_arrive(item_empty + slot);
    };
    constexpr bool ones = ONES;                  // V column dh = 1 -> O column dh = row sum
#if F3D_EXPERIMENT == 3
    unsigned long long prof[24] = {0};
    const long long t_start = clock64();
#endif

    // zero the operand tiles once: pad chunks (dh < DH) are never written again
    for (int i = tid; i < C::kOffBar / 16; i += kThreads)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    if (ones) {
        const __nv_bfloat16 one = __float2bfloat16(1.f);
        for (int i = tid; i < kNst * kBN; i += kThreads) {
            const int s = i / kBN, r = i - s * kBN;
            *reinterpret_cast<__nv_bfloat16*>(smem + C::kOffKV + s * 2 * C::kKVBytes + C::kKVBytes +
                                              L::template off<kBN>(r, A.dh >> 3) + (A.dh & 7) * 2) =
                one;
        }
    }
    if (tid == 0) {
        for (int b = 0; b < NQB; ++b) {
            mbar_init(q_full + b, kLoadThreads + 1);
            mbar_init(q_empty + b, NQ);                  // one commit / arrive per issuer
        }
        for (int s = 0; s < kNst; ++s) {
            mbar_init(kv_full + s, kLoadThreads + 1);
            mbar_init(kv_empty + s, NQ);
        }
        for (int g = 0; g < NQ; ++g) {
            for (int b = 0; b < NSB; ++b) {
                mbar_init(s_full + NSB * g + b, 1);
                mbar_init(p_full + NSB * g + b, 128 * CS);
                mbar_init(pv_done + NSB * g + b, 1);
            }
            mbar_init(o_free + g, 128 * CS);
        }
        for (int i = 0; i < kItemRing; ++i) {
            mbar_init(item_full + i, 1);
            mbar_init(item_empty + i, kConsumers);
        }
        fence_mbar_init();
        if (A.use_tma)
            for (int i = 0; i < kMaps; ++i)
                asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&M.m[i]))
                             : "memory");
    }
    if (warp == 0) {
        tmem_alloc(tmem_slot, C::kTmemCols);
        tmem_relinquish();
    }
    fence_proxy_async();
    // local set-up above overlaps the previous kernel's tail under
    // programmatic dependent launch; inputs are read from here on
    pdl_wait();
    total = (A.live ? __ldg(A.live) : A.nwork) * A.H;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sm_base = saddr(smem);

    if (warp < kLoadWarps) {
        // ------------------------------------------------ loader warps
        uint32_t q_use = 0, kv_it = 0;
        for (int slot = next_slot(); slot >= 0; slot = next_slot()) {
            const Item it = rec_item(recs + slot * kRecInts);
            const int qb = q_use % NQB;
            PROF_WAIT(10, mbar_wait(q_empty + qb, ((q_use / NQB) & 1) ^ 1));
            const uint32_t qdst = sm_base + C::kOffQ + qb * NQ * C::kQBytes;
            {
                int run[NQ];
                uint32_t bytes = 0;
#pragma unroll
                for (int g = 0; g < NQ; ++g) {
                    run[g] = -1;
                    if (g < it.nq) {
                        run[g] = A.use_tma ? tile_run(A, it, it.q0 + g * kBM, kBM) : -1;
                        if (run[g] < 0)
                            gather_rows<DH, kBM>(A, A.q, A.ld_q, it, it.q0 + g * kBM,
                                                 qdst + g * C::kQBytes, tid);
                        else
                            bytes += kBM * A.dh * 2;
                    }
                }
                cp_async_arrive(q_full + qb);
                if (tid == 0) {
                    if (bytes) {
                        mbar_arrive_expect(q_full + qb, bytes);
#pragma unroll
                        for (int g = 0; g < NQ; ++g)
                            if (run[g] >= 0)
                                tma_rows<DH, kBM, 64>(M, 0, A, it.h, run[g], qdst + g * C::kQBytes,
                                                  q_full + qb);
                    } else {
                        mbar_arrive(q_full + qb);
                    }
                }
            }
            ++q_use;
            for (int j = 0; j < it.nt; ++j, ++kv_it) {
                const int s = kv_it % kNst;
                const uint32_t u = kv_it / kNst;
                PROF_WAIT(9, mbar_wait(kv_empty + s, (u & 1) ^ 1));
                const uint32_t kb = sm_base + C::kOffKV + s * 2 * C::kKVBytes;
                const int run = A.use_tma ? tile_run(A, it, j * kBN, kBN) : -1;
                if (run < 0) {
                    gather_rows<DH, kBN>(A, A.k, A.ld_k, it, j * kBN, kb, tid);
                    gather_rows<DH, kBN>(A, A.v, A.ld_v, it, j * kBN, kb + C::kKVBytes, tid);
                }
                cp_async_arrive(kv_full + s);
                if (tid == 0) {
                    if (run >= 0) {
                        mbar_arrive_expect(kv_full + s, 2 * kBN * A.dh * 2);
                        tma_rows<DH, kBN, kBN>(M, 2, A, it.h, run, kb, kv_full + s);
                        tma_rows<DH, kBN, kBN>(M, 4, A, it.h, run, kb + C::kKVBytes, kv_full + s);
                    } else {
                        mbar_arrive(kv_full + s);
                    }
                }
            }
        }
    } else if (warp < pre_warps(NQ)) {
        // ------------------------------------------------ MMA issuers
        // Warp 1 + g issues every MMA of Q tile g (warp-uniform control flow
        // and waits; one elected lane issues every tcgen05.mma / commit).
        // A K/V stage is released (kv_empty) once every issuer's MMAs on it
        // completed; an issuer with no Q tile g in an item still takes part:
        // it waits for each of the item's K/V stages to be full before
        // arriving (so its arrival can never count toward an earlier phase).
        // Descriptors are built once: per tile only the 14-bit start-address
        // field moves (addresses < 2^18, so adding (bytes >> 4) never carries).
        const int g = warp - 1;
        constexpr uint32_t idS = idesc_bf16(kBM, kBN, 0, 0);
        constexpr uint32_t idPV = idesc_bf16(kBM, DH, 0, 1);
        // K-major Q / K: rows of SW bytes, 8-row groups SBO = 8*SW apart
        const uint64_t dQ = sw_desc(sm_base + C::kOffQ, 16, 8 * L::SW, L::LT);
        const uint64_t dK = sw_desc(sm_base + C::kOffKV, 16, 8 * L::SW, L::LT);
        // MN-major V: LBO = column-block stride, SBO = 8-key group stride
        const uint64_t dV = sw_desc(sm_base + C::kOffKV + C::kKVBytes, kBN * L::SW, 8 * L::SW, L::LT);
        constexpr uint32_t kStageD = (2 * C::kKVBytes) >> 4;   // descriptor step per K/V stage
        constexpr uint32_t kQD = C::kQBytes >> 4;              // per Q tile
        uint32_t q_use = 0, kv_it = 0;
        uint32_t tg = 0, ig = 0;             // tiles / items of Q tile g processed so far
        if (g < NQ) {
        for (int slot = next_slot(); slot >= 0; release_slot(slot), slot = next_slot()) {
            const Item it = rec_item(recs + slot * kRecInts);
            const int qb = q_use % NQB;
            PROF_WAIT(4, mbar_wait(q_full + qb, (q_use / NQB) & 1));
            tc_fence_after();
            auto wait_kv = [&](int j) {
                const uint32_t kvi = kv_it + j;
                PROF_WAIT(5, mbar_wait(kv_full + kvi % kNst, (kvi / kNst) & 1));
                tc_fence_after();
            };
            if (g >= it.nq) {
                // no Q tile g here: release the Q buffer and each K/V stage
                if (lane == 0) mbar_arrive(q_empty + qb);
                for (int j = 0; j < it.nt; ++j) {
                    wait_kv(j);
                    if (lane == 0) mbar_arrive(kv_empty + (kv_it + j) % kNst);
                }
                __syncwarp();
                ++q_use;
                kv_it += it.nt;
                continue;
            }
            const uint64_t dqg = dQ + (uint64_t)(qb * NQ * kQD + g * kQD);
            // S_g,j -> TMEM buffer (tg+j)%NSB, which last held P_g,j-NSB:
            // PV_g,j-NSB was issued before by this thread (in-order execution).
            auto issue_S = [&](int j) {
                const uint32_t s = (kv_it + j) % kNst;
                const uint32_t b = (tg + j) % NSB;
                const uint64_t dk = dK + (uint64_t)(s * kStageD);
                const uint32_t d = tmem + C::kTmemS + (NSB * g + b) * kBN;
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < DH / 16; ++k) {
                        // K-step k: column block k*16/BW, 32-byte step inside the swizzled row
                        constexpr int kPerBlk = L::BW / 16;
                        const uint32_t oq = (uint32_t)(((k / kPerBlk) * kBM * L::SW + (k % kPerBlk) * 32) >> 4);
                        const uint32_t ok = (uint32_t)(((k / kPerBlk) * kBN * L::SW + (k % kPerBlk) * 32) >> 4);
                        umma_f16(d, dqg + oq, dk + ok, idS, k > 0);
                    }
                    umma_commit(s_full + NSB * g + b);
                }
                __syncwarp();
            };
            for (int j = 0; j < NSB && j < it.nt; ++j) {
                wait_kv(j);
                issue_S(j);
            }
            if (it.nt <= NSB) {
                if (elect_one()) umma_commit(q_empty + qb);
                __syncwarp();
            }
            for (int j = 0; j < it.nt; ++j) {
                const uint32_t s = (kv_it + j) % kNst;
                const uint64_t dv = dV + (uint64_t)(s * kStageD);
                if (j == 0 && ig > 0) PROF_WAIT(7, mbar_wait(o_free + g, (ig - 1) & 1));
                const uint32_t t = tg + j;     // P_g,j in TMEM buffer t % NSB
                PROF_WAIT(6, mbar_wait(p_full + NSB * g + t % NSB, (t / NSB) & 1));
                tc_fence_after();
                const uint32_t pa = tmem + C::kTmemS + (NSB * g + t % NSB) * kBN;
                const uint32_t od = tmem + C::kTmemO + g * DH;
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < kBN / 16; ++k)   // 16 keys = two 8-key groups
                        umma_f16_ts(od, pa + k * 8, dv + (uint64_t)((16 * L::SW * k) >> 4), idPV,
                                    (j > 0 || k > 0) ? 1u : 0u);
                    umma_commit(pv_done + NSB * g + t % NSB);
                    umma_commit(kv_empty + s);         // S_g,j and PV_g,j read stage s
                }
                __syncwarp();
                if (j + NSB < it.nt) {
                    wait_kv(j + NSB);
                    issue_S(j + NSB);
                    if (j + NSB + 1 == it.nt) {          // last S of the item issued
                        if (elect_one()) umma_commit(q_empty + qb);
                        __syncwarp();
                    }
                }
            }
            ++q_use;
            kv_it += it.nt;
            tg += it.nt;
            ++ig;
        }
        }
    } else {
        // ------------------------------------------------ softmax warpgroups
        const int sw = warp - pre_warps(NQ);               // 0 .. 4*NQ*CS-1
        const int wgi = sw >> 2;
        const int g = wgi / CS;                           // Q tile of this warpgroup
        const int hh = wgi - g * CS;                      // column share of this warp
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;                // row in the tile = TMEM lane
        const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
        const float sl2 = A.scale_log2;
        constexpr int KC = kBN / CS;                      // S columns per warp
        constexpr int OC = DH / CS;                       // O columns per warp
        const uint32_t obase = tmem + lane_base + C::kTmemO + g * DH;
        const uint32_t ocols = obase + hh * OC;
        // pair exchange slots (CS == 2): [g][quarter][slot 0..2][share][lane]
        float* xg = reinterpret_cast<float*>(smem + C::kOffX) + ((g * 4 + quarter) * 3) * CS * 32;
        const int bar_id = 1 + g * 4 + quarter;           // named barrier of the pair
        auto pair_max = [&](float v, int slot) -> float {
            if (CS == 1) return v;
            xg[(slot * CS + hh) * 32 + lane] = v;
            asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(32 * CS) : "memory");
            return fmaxf(v, xg[(slot * CS + (hh ^ 1)) * 32 + lane]);
        };
        uint32_t tg = 0;
#if F3D_EXPERIMENT == 4
        int titem = 0;
#endif
        for (int slot = next_slot(); slot >= 0; release_slot(slot), slot = next_slot()) {
            PROF_MARK(td0);
#if F3D_EXPERIMENT == 4
            if (blockIdx.x == 0 && lane == 0 && titem < 16) g_attn_trace2[warp][titem][0] = clock64();
#endif
            const volatile int* rec = recs + slot * kRecInts;
            const Item it = rec_item(rec);
            if (g >= it.nq) continue;                     // this Q tile is past the scope
            PROF_MARK(td1);
            PROF_ADD(20, td0, td1);
            float ms = -INFINITY, l = 0.f;                // running max (scaled, log2), sum
            // every row of this warp is past the scope end (the scope's last
            // Q tile): nothing to compute or store -- the warp only keeps the
            // barrier protocol (its P / O rows are never read for output)
            const bool dead = it.q0 + g * kBM + quarter * 32 >= it.m;
            for (int j = 0; j < it.nt; ++j) {
                const uint32_t t = tg + j;
                const int b = t % NSB;
                const uint32_t sb = tmem + lane_base + C::kTmemS + (NSB * g + b) * kBN;
                PROF_WAIT(1, mbar_wait(s_full + NSB * g + b, (t / NSB) & 1));
#if F3D_EXPERIMENT == 4
                if (blockIdx.x == 0 && lane == 0 && t < 96) g_attn_trace[warp][t][0] = clock64();
#endif
                tc_fence_after();
                if (dead) {
                    tc_fence_before();
                    mbar_arrive(p_full + NSB * g + b);
                    continue;
                }
                uint32_t x[KC];
                {
                    PROF_MARK(tl0);
#pragma unroll
                    for (int c = 0; c + 32 <= KC; c += 32)
                        tmem_ld32(sb + hh * KC + c, *reinterpret_cast<uint32_t(*)[32]>(&x[c]));
                    if (KC % 32 == 16)
                        tmem_ld16(sb + hh * KC + (KC & ~31),
                                  *reinterpret_cast<uint32_t(*)[16]>(&x[KC & ~31]));
                    tmem_wait_ld();
                    PROF_MARK(tl1);
                    PROF_ADD(16, tl0, tl1);
                }
#if F3D_EXPERIMENT == 3
                if (lane == 0) ++prof[12];
#endif
                PROF_MARK(tm0);
                const int kvalid = it.m - j * kBN - hh * KC;     // my keys < kvalid are real
                if (kvalid < KC) {
#pragma unroll
                    for (int e = 0; e < KC; ++e)
                        if (e >= kvalid) x[e] = __float_as_uint(-INFINITY);
                }
                // row max with 8 independent chains (short dependency depth)
                float mx[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) mx[q] = __uint_as_float(x[q]);
#pragma unroll
                for (int e = 8; e < KC; e += 8)
#pragma unroll
                    for (int q = 0; q < 8; ++q) mx[q] = fmaxf(mx[q], __uint_as_float(x[e + q]));
                const float mxs = pair_max(fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                                 fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))),
                                           t & 1) * sl2;
                PROF_MARK(tm1);
                PROF_ADD(17, tm0, tm1);
                if (j == 0) {
                    ms = mxs;
                } else {
                    // the pair computed the same row maxima: both warps take
                    // the same branch and rescale their own O columns
                    const bool need = mxs > ms + kRescale;
                    if (__any_sync(0xffffffffu, need)) {
                        // O_g must hold P_g,j-1 V before it is rescaled in place
                        PROF_WAIT(2, mbar_wait(pv_done + NSB * g + (t - 1) % NSB, ((t - 1) / NSB) & 1));
                        tc_fence_after();
                        const float alpha = need ? ex2f(ms - mxs) : 1.f;
                        if (need) {
                            ms = mxs;
                            l *= alpha;
                        }
#pragma unroll
                        for (int c = 0; c < OC; c += 16) {
                            uint32_t y[16];
                            tmem_ld16(ocols + c, y);
                            tmem_wait_ld();
                            const uint64_t al2 = f2(alpha, alpha);
#pragma unroll
                            for (int e = 0; e < 16; e += 2) {
                                float u0, u1;
                                f2_split(fmul2(f2(__uint_as_float(y[e]), __uint_as_float(y[e + 1])), al2),
                                         u0, u1);
                                y[e] = __float_as_uint(u0);
                                y[e + 1] = __float_as_uint(u1);
                            }
                            tmem_st16(ocols + c, y);
                        }
#if F3D_EXPERIMENT == 3
                        if (lane == 0) ++prof[13];
#endif
                    }
                }
                // P = exp2(s*sl2 - ms) (<= 2^8) -> bf16 pairs over the S columns
                const float nms = -ms;
                const uint64_t sl2x2 = f2(sl2, sl2), nms2 = f2(nms, nms);
                PROF_MARK(te0);
#if F3D_EXPERIMENT == 4
                if (blockIdx.x == 0 && lane == 0 && t < 96) g_attn_trace[warp][t][1] = clock64();
#endif
                float sum = 0.f;
#pragma unroll
                for (int e = 0; e < KC; e += 2) {
#if F3D_EXPERIMENT == 2
                    const float p0 = fmaf(__uint_as_float(x[e]), sl2, nms);
                    const float p1 = fmaf(__uint_as_float(x[e + 1]), sl2, nms);
#else
                    // every kPolyEvery-th pair on the FMA pipe: the MUFU unit
                    // (16 ex2/clk/SM) is the softmax roof at small head dims
                    const uint64_t a2 =
                        ffma2(f2(__uint_as_float(x[e]), __uint_as_float(x[e + 1])), sl2x2, nms2);
                    constexpr int kPE = poly_every<DH>();
                    const bool poly = kPE > 0 && ((e >> 1) % (kPE > 0 ? kPE : 1)) == kPE - 1;
                    float p0, p1;
                    if (poly) {
                        ex2_poly2(a2, p0, p1);
                    } else {
                        float a0, a1;
                        f2_split(a2, a0, a1);
                        p0 = ex2f(a0);
                        p1 = ex2f(a1);
                    }
#endif
                    if (!ones) sum += p0 + p1;
                    __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
                    x[e >> 1] = *reinterpret_cast<uint32_t*>(&h2);   // in place: x[e/2] consumed
                }
                l += sum;
                PROF_MARK(te1);
#if F3D_EXPERIMENT == 4
                if (blockIdx.x == 0 && lane == 0 && t < 96) g_attn_trace[warp][t][2] = clock64();
#endif
                PROF_ADD(18, te0, te1);
                if (KC == 64)
                    tmem_st32(sb, *reinterpret_cast<uint32_t(*)[32]>(&x[0]));
                else if (KC == 48) {
                    tmem_st16(sb, *reinterpret_cast<uint32_t(*)[16]>(&x[0]));
                    tmem_st8(sb + 16, *reinterpret_cast<uint32_t(*)[8]>(&x[16]));
                } else
                    tmem_st16(sb + hh * (KC / 2), *reinterpret_cast<uint32_t(*)[16]>(&x[0]));
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(p_full + NSB * g + b);
                PROF_MARK(te2);
                PROF_ADD(19, te1, te2);
            }
            // O_g complete: normalise and write the row
            {
                const uint32_t tl = tg + it.nt - 1;
#if F3D_EXPERIMENT == 4
                if (blockIdx.x == 0 && lane == 0 && titem < 16) g_attn_trace2[warp][titem][1] = clock64();
#endif
                PROF_WAIT(3, mbar_wait(pv_done + NSB * g + tl % NSB, (tl / NSB) & 1));
#if F3D_EXPERIMENT == 4
                if (blockIdx.x == 0 && lane == 0 && titem < 16) g_attn_trace2[warp][titem][2] = clock64();
#endif
            }
            PROF_MARK(tq0);
            tc_fence_after();
            if (dead) {
                tc_fence_before();
                mbar_arrive(o_free + g);
                tg += it.nt;
                continue;
            }
            float lsum = l;
            // one TMEM round trip for a 32-column O row (sum column included)
            constexpr bool kO32 = OC == 32 && CS == 1;
            uint32_t yo[kO32 ? 32 : 1];
            if (kO32) {
                tmem_ld32(ocols, *reinterpret_cast<uint32_t(*)[32]>(&yo[0]));
                tmem_wait_ld();
                if (ones)   // dh is a multiple of 8 below 32 (selects: no indexed local copy)
                    lsum = __uint_as_float(A.dh == 8 ? yo[8 % (kO32 ? 32 : 1)]
                                           : A.dh == 16 ? yo[16 % (kO32 ? 32 : 1)]
                                                        : yo[24 % (kO32 ? 32 : 1)]);
            } else if (ones) {
                uint32_t y[16];
                tmem_ld16(obase + (A.dh & ~15), y);
                tmem_wait_ld();
                lsum = __uint_as_float(y[A.dh & 15]);
            } else if (CS > 1) {
                xg[(2 * CS + hh) * 32 + lane] = l;       // slot 2: partial row sums
                asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(32 * CS) : "memory");
                lsum = l + xg[(2 * CS + (hh ^ 1)) * 32 + lane];
            }
#if F3D_EXPERIMENT == 4
            if (blockIdx.x == 0 && lane == 0 && titem < 16) g_attn_trace2[warp][titem][4] = clock64();
#endif
            float inv = 0.f;                              // MUFU reciprocal (<= 1 ulp)
            if (lsum > 0.f) asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(lsum));
            const int vr = it.q0 + g * kBM + r;
            const bool live_row = vr < it.m;
            const int pr = live_row ? phys_row_rec(A, rec, it, vr) : 0;
#if F3D_EXPERIMENT == 4
            if (blockIdx.x == 0 && lane == 0 && titem < 16) g_attn_trace2[warp][titem][5] = clock64();
#endif
            // P = exp2(s * scale_log2 - lse) recomputes this row's softmax
            if (A.lse && live_row && hh == 0)
                A.lse[(int64_t)pr * A.ld_lse + it.h] = lsum > 0.f ? ms + __log2f(lsum) : -INFINITY;
            const int hcol = it.h * A.dh + hh * OC;     // this warp's output columns
#pragma unroll
            for (int c = 0; c < OC / 16; ++c) {
                uint32_t y[16];
                if (kO32) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) y[e] = yo[(c * 16 + e) % (kO32 ? 32 : 1)];
                } else {
                    tmem_ld16(ocols + c * 16, y);
                    tmem_wait_ld();
                }
                if (!live_row) continue;
                if (sizeof(OutT) == 2) {
                    __nv_bfloat16* out =
                        reinterpret_cast<__nv_bfloat16*>(A.o) + (int64_t)pr * A.ld_o + hcol;
#pragma unroll
                    for (int e = 0; e < 16; e += 8) {
                        if (hh * OC + c * 16 + e >= A.dh) break;
                        uint32_t w[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            __nv_bfloat162 h2 = __floats2bfloat162_rn(
                                __uint_as_float(y[e + 2 * q]) * inv, __uint_as_float(y[e + 2 * q + 1]) * inv);
                            w[q] = *reinterpret_cast<uint32_t*>(&h2);
                        }
                        if (A.o_vec)   // 16-byte stores: 8 columns at a time
                            *reinterpret_cast<uint4*>(out + c * 16 + e) = make_uint4(w[0], w[1], w[2], w[3]);
                        else
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                *reinterpret_cast<uint32_t*>(out + c * 16 + e + 2 * q) = w[q];
                    }
                } else {
                    float* out = reinterpret_cast<float*>(A.o) + (int64_t)pr * A.ld_o + hcol;
#pragma unroll
                    for (int e = 0; e < 16; e += 4) {
                        if (hh * OC + c * 16 + e >= A.dh) break;
                        const float4 v = make_float4(__uint_as_float(y[e]) * inv, __uint_as_float(y[e + 1]) * inv,
                                                     __uint_as_float(y[e + 2]) * inv, __uint_as_float(y[e + 3]) * inv);
                        if (A.o_vec)
                            *reinterpret_cast<float4*>(out + c * 16 + e) = v;
                        else {
                            out[c * 16 + e] = v.x;
                            out[c * 16 + e + 1] = v.y;
                            out[c * 16 + e + 2] = v.z;
                            out[c * 16 + e + 3] = v.w;
                        }
                    }
                }
            }
#if F3D_EXPERIMENT == 4
            if (blockIdx.x == 0 && lane == 0 && titem < 16) g_attn_trace2[warp][titem][6] = clock64();
#endif
            tc_fence_before();
            mbar_arrive(o_free + g);
            tg += it.nt;
            PROF_MARK(tq1);
#if F3D_EXPERIMENT == 4
            if (blockIdx.x == 0 && lane == 0 && titem < 16) g_attn_trace2[warp][titem][3] = clock64();
            ++titem;
#endif
            PROF_ADD(21, tq0, tq1);
        }
        PROF_MARK(tend);
        PROF_ADD(22, t_start, tend);
    }
#if F3D_EXPERIMENT == 3
    if (lane == 0) {
        const int role = warp < kLoadWarps ? 11 : (warp < pre_warps(NQ) ? 8 : 0);
        prof[role] += clock64() - t_start;
        for (int i = 0; i < 24; ++i)
            if (prof[i]) atomicAdd(&g_attn_prof[i], prof[i]);
    }
#endif
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, C::kTmemCols);
    if (dyn && tid == 0) {
        // this CTA took its last item (the counter is past total): the last
        // CTA to get here resets the scheduler words for the next launch
        __threadfence();
        if (atomicAdd(sched + 1, 1) == (int)gridDim.x - 1) {
            sched[0] = 0;
            sched[1] = 0;
            __threadfence();
        }
    }
}

// ------------------------------------------------------------- host side

template <int DH, typename OutT, bool ONES>
int launch(Args A, int64_t n_rows, cudaStream_t st) {
    using C = Cfg<DH>;
    using LY = Lay<DH>;
    auto kern = bswin_attn_tc_kernel<DH, OutT, ONES>;
    static bool attr = false;
    if (!attr) {
        F3D_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          C::kSmem));
        attr = true;
    }
    Maps M;
    memset(&M, 0, sizeof(M));
    // TMA boxes cover the head's own columns: blocks of BW, the last one
    // possibly narrower (dh < DH); pad columns of the tiles stay zero
    const int64_t ncols = (int64_t)A.H * A.dh;
    A.use_tma = n_rows > 0 ? 1 : 0;
    const void* bases[3] = {A.q, A.k, A.v};
    const int64_t lds[3] = {A.ld_q, A.ld_k, A.ld_v};
    for (int t = 0; t < 3 && A.use_tma; ++t)
        for (int b = 0; b < 2; ++b) {
            const int w = std::min(LY::BW, A.dh - b * LY::BW);
            if (w <= 0) continue;
            if (!make_map(&M.m[2 * t + b], bases[t], lds[t], ncols, n_rows, w, LY::SW,
                          t == 0 ? 64 : C::kBN))
                A.use_tma = 0;
        }

    const int total = A.nwork * A.H;
    const int grid = std::max(1, std::min(total, f3d_num_sms() * ctas_per_sm<DH>()));
    F3D_CUDA_TRY(f3d_launch(kern, dim3(grid), dim3(threads_for<DH>()), C::kSmem, st, A, M));
    return F3D_OK;
}

template <int DH>
int launch_dh(const Args& A, int64_t n_rows, cudaStream_t st) {
    if (A.dh < DH)
        return A.out_f32 ? launch<DH, float, true>(A, n_rows, st)
                         : launch<DH, __nv_bfloat16, true>(A, n_rows, st);
    return A.out_f32 ? launch<DH, float, false>(A, n_rows, st)
                     : launch<DH, __nv_bfloat16, false>(A, n_rows, st);
}

}  // namespace attn_tc
}  // namespace f3d

using namespace f3d;

#if F3D_EXPERIMENT == 4
extern "C" int f3d_attn_trace(long long* out_host) {
    int e = (int)cudaMemcpyFromSymbol(out_host, g_attn_trace, sizeof(g_attn_trace));
    return e ? e : (int)cudaMemcpyFromSymbol(out_host + 16 * 96 * 3, g_attn_trace2, sizeof(g_attn_trace2));
}
#endif
#if F3D_EXPERIMENT == 3
extern "C" int f3d_attn_prof(unsigned long long* out24_host, int reset) {
    cudaMemcpyFromSymbol(out24_host, g_attn_prof, sizeof(g_attn_prof));
    if (reset) {
        unsigned long long z[24] = {0};
        cudaMemcpyToSymbol(g_attn_prof, z, sizeof(z));
    }
    return 0;
}
#endif

extern "C" int f3d_attention_tc_qstep(int dh) {
    return f3d::attn_tc::nq_for_dh(f3d::attn_tc::dh_tile(dh)) * f3d::attn_tc::kBM;
}

extern "C" int f3d_bswin_attention_tc(const void* q, const void* k, const void* v, int64_t ld_q,
                                      int64_t ld_k, int64_t ld_v, void* o, int64_t ld_o,
                                      int out_f32, int H, int dh, const int32_t* scope_seg,
                                      const int32_t* scope_nseg, const int32_t* seg_start,
                                      const int32_t* seg_vstart, const int32_t* scope_len,
                                      const int32_t* work, int nwork, const int32_t* live,
                                      int64_t n_rows, float* lse, int64_t ld_lse, void* stream) {
    if (H < 1 || dh < 8 || dh > 128 || (dh & 7) || nwork < 0 || n_rows < 0) return F3D_ERR_CONFIG;
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
    A.use_tma = 0;
    A.lse = lse;
    A.ld_lse = ld_lse;
    {
        const int esz = out_f32 ? 4 : 2;
        A.o_vec = (((uintptr_t)o & 15) == 0 && (ld_o * esz) % 16 == 0 && (dh * esz) % 16 == 0) ? 1 : 0;
    }
    cudaStream_t st = (cudaStream_t)stream;
    switch (attn_tc::dh_tile(dh)) {
        case 16: return attn_tc::launch_dh<16>(A, n_rows, st);
        case 32: return attn_tc::launch_dh<32>(A, n_rows, st);
        case 64: return attn_tc::launch_dh<64>(A, n_rows, st);
        case 128: return attn_tc::launch_dh<128>(A, n_rows, st);
        default: return F3D_ERR_CONFIG;
    }
}
