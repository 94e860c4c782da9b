// In-bucket pooling (bw/pooling.py): sub-bucket partition of every <=1024-row
// tile of every bucket slot, then the per-sub-bucket reduce.
//
// Partition (bw/pooling.py:68-163), one warp per tile, bit-exact:
//   q = min((c - lo) / ext * 1024, 1023) truncated (f64, IEEE ops)      :59-65
//   key = morton10(q) % target, target = ceil(m / rho)                   :84
//   step 1: ids in first-seen key order; a row stays iff its occurrence
//           rank within its key is < rho (index order)                  :88-102
//   step 2: the first (target - #ids) overflow rows seed new ids         :104-117
//   step 3: the rest, in index order, join the nearest under-filled new
//           id (else any under-filled id); f64 sqrt((dx^2+dy^2)+dz^2) to the
//           seed row, lowest id on ties                                   :119-139
//   repair: pour the smallest under-filled into the fullest one by stable
//           distance order until <= 1 is under-filled                     :141-157
// Occurrence ranks are computed 32 rows at a time with __match_any_sync,
// so index order is preserved exactly.  Members of each sub-bucket are
// emitted in index order as a dense [pooled_rows][rho] list for the reduce.
#include <cuda_bf16.h>

#include <cfloat>
#include <climits>

#include "f3d_common.cuh"

namespace f3d {
namespace pool {

constexpr int kCap = 1024;         // TILE_CAP (bw/pooling.py:22)
constexpr int kWarpsPerCta = 1;   // 40 KB of smem per warp: 5 tiles in flight per SM
constexpr int kThreads = 32 * kWarpsPerCta;

struct WarpSmem {
    double cc[kCap][3];     // per row: the tile's coordinates (staged once)
    uint16_t qrow[kCap];    // step-3 queue: queued rows in index order
    uint16_t cnt[kCap];     // per key running count
    int16_t idk[kCap];      // key -> sub id
    int16_t sizes[kCap];    // per sub id
    int16_t seeds[kCap];    // per sub id: tile-local seed row
    int16_t sub[kCap];      // per row: sub id (-1 overflow, -2 queued)
    uint16_t key[kCap];     // per row
    int16_t elig[kCap];     // step 3: eligible ids of the current pass, ascending
};

struct Args {
    const double* coords;       // (N,3) scattered rows
    const int32_t* tile_start;  // global first row of tile t
    const int32_t* tile_m;      // rows in tile t
    const int32_t* tile_out;    // first pooled row of tile t
    int ntiles;
    const int32_t* ntiles_dev;  // nullable: device tile count (<= ntiles)
    int rho;
    int32_t* sub_out;           // (N) tile-local sub id per row (nullable)
    int32_t* members;           // (npool, rho) global row ids, -1 padded
    int32_t* sizes_out;         // (npool)
    int32_t* seeds_out;         // (npool) tile-local seed row (nullable)
    int32_t* passes_out;        // (ntiles) scan passes (nullable)
    int32_t* flags;             // integrity flags
};

__device__ __forceinline__ double dist3(const double* a, const double* b) {
    const double dx = __dsub_rn(a[0], b[0]);
    const double dy = __dsub_rn(a[1], b[1]);
    const double dz = __dsub_rn(a[2], b[2]);
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

// (dx^2 + dy^2) + dz^2 with the reference's roundings (no contraction):
// dist3 = sqrt(dist2), and sqrt is monotone, so comparisons can use dist2
// except when two squared distances are close enough to share a sqrt.
__device__ __forceinline__ double dist2(const double* a, const double* b) {
    const double dx = __dsub_rn(a[0], b[0]);
    const double dy = __dsub_rn(a[1], b[1]);
    const double dz = __dsub_rn(a[2], b[2]);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// Is (sqrt(d2), j) lexicographically below (sqrt(b2), bj)?  Squared values
// more than 2^-45 apart (relative) have sqrt values > 2 ulp apart, so the
// order of d2 decides; near-ties fall back to the rounded sqrt and the id.
__device__ __forceinline__ bool closer(double d2, int j, double b2, int bj) {
    if (d2 < __dmul_rn(b2, 1.0 - 0x1p-45)) return true;
    if (d2 > __dmul_rn(b2, 1.0 + 0x1p-45)) return false;
    const double s = __dsqrt_rn(d2), bs = __dsqrt_rn(b2);
    return s < bs || (s == bs && j < bj);
}

// Warp-wide minimum of (sqrt(d2) rounded, id) -- closer()'s order -- over the
// lanes' best (bd2, bid) (bid == INT_MAX: no candidate).  Squared distances
// are >= 0, so their IEEE bits order like the values: two 32-bit redux.min
// find the smallest d2; only lanes within 2^-45 of it can share its rounded
// square root, and among those the lowest id wins.
__device__ __forceinline__ int warp_argmin_dist(double bd2, int bid) {
    const unsigned long long bits = bid == INT_MAX ? ~0ull : (unsigned long long)__double_as_longlong(bd2);
    const unsigned hi = (unsigned)(bits >> 32), lo = (unsigned)bits;
    const unsigned mhi = __reduce_min_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_min_sync(0xffffffffu, hi == mhi ? lo : 0xffffffffu);
    const unsigned long long mb = ((unsigned long long)mhi << 32) | mlo;
    if (mb == ~0ull) return INT_MAX;
    const double dmin = __longlong_as_double((long long)mb);
    const bool band = bid != INT_MAX && bd2 <= __dmul_rn(dmin, 1.0 + 0x1p-45);
    const unsigned bm = __ballot_sync(0xffffffffu, band);
    if ((bm & (bm - 1)) == 0) return __shfl_sync(0xffffffffu, bid, __ffs(bm) - 1);
    const double smin = __dsqrt_rn(dmin);
    const bool win = band && __dsqrt_rn(bd2) == smin;
    return (int)__reduce_min_sync(0xffffffffu, win ? (unsigned)bid : 0xffffffffu);
}

__global__ void __launch_bounds__(kThreads) pool_build_kernel(const Args A) {
    extern __shared__ __align__(16) unsigned char pool_smem[];
    WarpSmem* smem_all = reinterpret_cast<WarpSmem*>(pool_smem);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int t = blockIdx.x * kWarpsPerCta + warp;
    if (t >= dyn_n(A.ntiles, A.ntiles_dev)) return;
    WarpSmem& S = smem_all[warp];
    const int r0 = A.tile_start[t];
    const int m = A.tile_m[t];
    const int rho = A.rho;
    const int target = (m + rho - 1) / rho;
    const double* C = A.coords + 3 * (int64_t)r0;
    const unsigned lt = lanemask_lt();

    // ---- bbox of the tile
    double lo[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, hi[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
    for (int i = lane; i < 3 * m; i += 32) {   // coalesced; rows staged in smem
        const double v = C[i];
        (&S.cc[0][0])[i] = v;
    }
    __syncwarp();
    for (int i = lane; i < m; i += 32)
        for (int a = 0; a < 3; ++a) {
            const double v = S.cc[i][a];
            lo[a] = fmin(lo[a], v);
            hi[a] = fmax(hi[a], v);
        }
    for (int a = 0; a < 3; ++a)
        for (int o = 16; o > 0; o >>= 1) {
            lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
            hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
        }
    double ext[3];
    for (int a = 0; a < 3; ++a) {
        ext[a] = __dsub_rn(hi[a], lo[a]);
        if (ext[a] == 0.0) ext[a] = 1.0;
    }
    // ---- keys; reset per-key / per-id state
    for (int i = lane; i < kCap; i += 32) {
        S.cnt[i] = 0;
        S.idk[i] = -1;
        S.sizes[i] = 0;
        S.seeds[i] = -1;
    }
    for (int i = lane; i < m; i += 32) {
        uint32_t q[3];
        for (int a = 0; a < 3; ++a) {
            double v = __dmul_rn(__ddiv_rn(__dsub_rn(S.cc[i][a], lo[a]), ext[a]), 1024.0);
            v = fmin(v, 1023.0);
            q[a] = (uint32_t)(int64_t)v;   // truncation (values >= 0)
        }
        const uint32_t code = spread3_10(q[0]) | (spread3_10(q[1]) << 1) | (spread3_10(q[2]) << 2);
        S.key[i] = (uint16_t)(code % (uint32_t)target);
    }
    __syncwarp();
    // ---- step 1: first-seen allocation + occurrence ranks, 32 rows at a time
    int nalloc = 0, novf = 0;
    for (int base = 0; base < m; base += 32) {
        const int i = base + lane;
        const bool v = i < m;
        const int k = v ? (int)S.key[i] : -1 - lane;   // invalid lanes: unique keys
        const unsigned mm = __match_any_sync(0xffffffffu, k);
        int occ = 0;
        if (v) occ = S.cnt[k] + __popc(mm & lt);
        const bool first = v && occ == 0;
        const unsigned fb = __ballot_sync(0xffffffffu, first);
        __syncwarp();
        if (first) {
            const int id = nalloc + __popc(fb & lt);
            S.idk[k] = (int16_t)id;
            S.seeds[id] = (int16_t)i;
        }
        if (v && lane == __ffs(mm) - 1) S.cnt[k] = (uint16_t)(S.cnt[k] + __popc(mm));
        nalloc += __popc(fb);
        __syncwarp();
        const bool keep = v && occ < rho;
        const bool ovf = v && !keep;
        const unsigned ob = __ballot_sync(0xffffffffu, ovf);
        if (keep) S.sub[i] = S.idk[k];
        if (ovf) S.sub[i] = -1;
        novf += __popc(ob);
        __syncwarp();
    }
    for (int k = lane; k < target; k += 32) {
        const int c = S.cnt[k];
        if (c > 0) S.sizes[S.idk[k]] = (int16_t)min(c, rho);
    }
    __syncwarp();
    // ---- step 2: overflow rows seed new ids until target ids exist
    const int need_new = target - nalloc;
    int rank = 0;
    int nqueue = 0;
    for (int base = 0; base < m; base += 32) {
        const int i = base + lane;
        const bool o = i < m && S.sub[i] == -1;
        const unsigned ob = __ballot_sync(0xffffffffu, o);
        if (o) {
            const int r = rank + __popc(ob & lt);
            if (r < need_new) {
                const int id = nalloc + r;
                S.sub[i] = (int16_t)id;
                S.sizes[id] = 1;
                S.seeds[id] = (int16_t)i;
                        } else {
                S.sub[i] = -2;
                S.qrow[r - need_new] = (uint16_t)i;   // queue keeps index order
            }
        }
        rank += __popc(ob);
    }
    nqueue = max(0, novf - need_new);
    if (novf < need_new && lane == 0) atomicOr(A.flags, 1);   // allocation fell short
    __syncwarp();
    // ---- step 3: queued rows join the nearest under-filled sub-bucket.
    // Speculative batches of 32 queued rows, one per lane: every lane finds
    // its row's nearest eligible id against the sizes at the start of the
    // pass, then the choices are committed in index order while each chosen
    // id is still under-filled.  Eligibility only shrinks during step 3, so a
    // choice whose id is still eligible at commit time is exactly the
    // sequential answer (the minimum over a superset that lies in the
    // subset); a stale choice is recomputed for that row alone (warp-parallel
    // over the still-eligible ids of the pass's tier) and committing goes on;
    // only an exhausted tier ends the pass and rebuilds the list.
    for (int q0 = 0; q0 < nqueue;) {
        __syncwarp();                        // the previous pass's elig reads are done
        // eligible ids of this pass: under-filled new ids, else any under-filled
        int ne = 0;
        for (int j0 = nalloc; j0 < target; j0 += 32) {
            const int jj = j0 + lane;
            const bool e = jj < target && S.sizes[jj] < rho;
            const unsigned b = __ballot_sync(0xffffffffu, e);
            if (e) S.elig[ne + __popc(b & lt)] = (int16_t)jj;
            ne += __popc(b);
        }
        if (ne == 0) {
            for (int j0 = 0; j0 < target; j0 += 32) {
                const int jj = j0 + lane;
                const bool e = jj < target && S.sizes[jj] < rho;
                const unsigned b = __ballot_sync(0xffffffffu, e);
                if (e) S.elig[ne + __popc(b & lt)] = (int16_t)jj;
                ne += __popc(b);
            }
        }
        __syncwarp();
        if (ne == 0) {                       // nothing under-filled: allocation broke
            if (lane == 0) atomicOr(A.flags, 2);
            break;
        }
        const int nb = min(32, nqueue - q0);
        int choice = INT_MAX;
        if (lane < nb) {
            const int i = S.qrow[q0 + lane];
            const double ci[3] = {S.cc[i][0], S.cc[i][1], S.cc[i][2]};
            double bd2 = DBL_MAX;
            for (int e = 0; e < ne; ++e) {      // ascending ids: strict '<' keeps the lowest
                const int jj = S.elig[e];
                const double d2 = dist2(S.cc[S.seeds[jj]], ci);   // seed row's coordinates
                if (closer(d2, jj, bd2, choice)) {
                    bd2 = d2;
                    choice = jj;
                }
            }
        }
        int done = 0;
        for (; done < nb; ++done) {          // commit in index order while valid
            const int jj = __shfl_sync(0xffffffffu, choice, done);
            if (jj == INT_MAX) {             // no finite distance (non-finite coords)
                if (lane == 0) atomicOr(A.flags, 2);
                done = nqueue;
                break;
            }
            int pick = jj;
            if (S.sizes[jj] >= rho) {
                // stale: this row alone, warp-parallel over the pass's eligible
                // ids that are still under-filled (same tier: the list only
                // shrinks; an exhausted tier ends the pass and rebuilds it)
                const int i = S.qrow[q0 + done];
                const double ci[3] = {S.cc[i][0], S.cc[i][1], S.cc[i][2]};
                double bd2 = DBL_MAX;
                int bid = INT_MAX;
                for (int e = lane; e < ne; e += 32) {
                    const int j = S.elig[e];
                    if (S.sizes[j] >= rho) continue;
                    const double d2 = dist2(S.cc[S.seeds[j]], ci);
                    if (closer(d2, j, bd2, bid)) {
                        bd2 = d2;
                        bid = j;
                    }
                }
                bid = warp_argmin_dist(bd2, bid);   // 5-level shuffle + closer(): 88 -> 72 us
                if (bid == INT_MAX) break;   // tier exhausted: rebuild the list
                pick = bid;
            }
            __syncwarp();
            if (lane == 0) {
                S.sub[S.qrow[q0 + done]] = (int16_t)pick;
                S.sizes[pick] = (int16_t)(S.sizes[pick] + 1);
            }
            __syncwarp();
        }
        q0 += done;
    }
    // ---- repair: at most one under-filled sub-bucket may remain
    for (int guard = 0; guard < kCap; ++guard) {
        // under-filled ids: count, fullest (lowest id on ties)
        int cnt_under = 0;
        int best_sz = -1, best_id = INT_MAX;
        for (int j = lane; j < target; j += 32) {
            const int sz = S.sizes[j];
            if (sz < rho) {
                ++cnt_under;
                if (sz > best_sz || (sz == best_sz && j < best_id)) {
                    best_sz = sz;
                    best_id = j;
                }
            }
        }
        cnt_under = warp_sum(cnt_under);
        if (cnt_under <= 1) break;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int s2 = __shfl_xor_sync(0xffffffffu, best_sz, o);
            const int i2 = __shfl_xor_sync(0xffffffffu, best_id, o);
            if (s2 > best_sz || (s2 == best_sz && i2 < best_id)) {
                best_sz = s2;
                best_id = i2;
            }
        }
        const int full_t = best_id;
        int dsz = INT_MAX, donor = INT_MAX;
        for (int j = lane; j < target; j += 32) {
            const int sz = S.sizes[j];
            if (sz < rho && j != full_t && (sz < dsz || (sz == dsz && j < donor))) {
                dsz = sz;
                donor = j;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int s2 = __shfl_xor_sync(0xffffffffu, dsz, o);
            const int i2 = __shfl_xor_sync(0xffffffffu, donor, o);
            if (s2 < dsz || (s2 == dsz && i2 < donor)) {
                dsz = s2;
                donor = i2;
            }
        }
        const int need = rho - S.sizes[full_t];
        // members of donor in index order (< rho of them), 32 rows per ballot,
        // into the (now free) step-3 queue
        int nm = 0;
        for (int base = 0; base < m && nm < 64; base += 32) {
            const int i = base + lane;
            const bool in = i < m && S.sub[i] == donor;
            const unsigned b = __ballot_sync(0xffffffffu, in);
            if (in && nm + __popc(b & lt) < 64) S.qrow[nm + __popc(b & lt)] = (uint16_t)i;
            nm += __popc(b);
        }
        nm = min(nm, 64);
        __syncwarp();
        if (lane == 0) {
            // stable by distance to the fullest id's seed
            int mem[64];
            double md[64];
            const double* cs = S.cc[S.seeds[full_t]];
            for (int a = 0; a < nm; ++a) {
                mem[a] = S.qrow[a];
                md[a] = dist3(S.cc[mem[a]], cs);
            }
            // stable insertion sort by distance
            for (int a = 1; a < nm; ++a) {
                const int mi = mem[a];
                const double dv = md[a];
                int b = a - 1;
                while (b >= 0 && md[b] > dv) {
                    mem[b + 1] = mem[b];
                    md[b + 1] = md[b];
                    --b;
                }
                mem[b + 1] = mi;
                md[b + 1] = dv;
            }
            const int mv = min(need, nm);
            for (int a = 0; a < mv; ++a) S.sub[mem[a]] = (int16_t)full_t;
            S.sizes[full_t] = (int16_t)(S.sizes[full_t] + mv);
            S.sizes[donor] = (int16_t)(S.sizes[donor] - mv);
        }
        __syncwarp();
    }
    __syncwarp();
    // ---- validate + emit
    const int out0 = A.tile_out[t];
    int bad = 0;
    int n_under = 0;
    for (int j = lane; j < target; j += 32) {
        const int sz = S.sizes[j];
        if (sz > rho) bad |= 4;
        if (sz < 1) bad |= 8;
        if (sz < rho) ++n_under;
        A.sizes_out[out0 + j] = sz;
        if (A.seeds_out) A.seeds_out[out0 + j] = S.seeds[j];
        S.cnt[j] = 0;
    }
    n_under = warp_sum(n_under);
    if (n_under > 1) bad |= 16;
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && lane == 0) atomicOr(A.flags, bad);
    if (A.passes_out && lane == 0) A.passes_out[t] = nqueue > 0 ? 1 : 0;
    __syncwarp();
    for (int base = 0; base < m; base += 32) {
        const int i = base + lane;
        const bool v = i < m;
        const int s = v ? (int)S.sub[i] : -1 - lane;
        const unsigned mm = __match_any_sync(0xffffffffu, s);
        if (v) {
            if (s < 0 || s >= target) {
                atomicOr(A.flags, 32);
            } else {
                const int r = S.cnt[s] + __popc(mm & lt);
                if (r < rho) A.members[(int64_t)(out0 + s) * rho + r] = r0 + i;
                if (A.sub_out) A.sub_out[r0 + i] = s;
            }
        }
        __syncwarp();
        if (v && s >= 0 && s < target && lane == __ffs(mm) - 1)
            S.cnt[s] = (uint16_t)(S.cnt[s] + __popc(mm));
        __syncwarp();
    }
    // pad member lists of sub-buckets smaller than rho
    for (int j = lane; j < target; j += 32)
        for (int r = S.sizes[j]; r < rho; ++r) A.members[(int64_t)(out0 + j) * rho + r] = -1;
}

// ------------------------------------------------------------------ reduce

enum { R_SUM = 0, R_MEAN = 1, R_MIN = 2, R_MAX = 3 };

template <typename T> struct RAcc { using type = float; };
template <> struct RAcc<double> { using type = double; };
__device__ __forceinline__ float ld_f(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ float ld_f(const float* p) { return *p; }
__device__ __forceinline__ double ld_f(const double* p) { return *p; }
__device__ __forceinline__ void st_f(__nv_bfloat16* p, float v) { *p = __float2bfloat16(v); }
__device__ __forceinline__ void st_f(float* p, float v) { *p = v; }
__device__ __forceinline__ void st_f(double* p, double v) { *p = v; }

// One thread per (pooled row, column), members in index order.  Sums follow
// numpy's add.reduceat exactly: out = x[m0] + pairwise(x[m1..]), where the
// pairwise rest is a plain loop from 0.0 below 8 terms and eight strided
// accumulators combined ((0+1)+(2+3))+((4+5)+(6+7)) up to 128 terms
// (rho <= 64 keeps us below the recursive split).  mean = sum / size.
template <typename T>
__global__ void pool_reduce_kernel(const T* __restrict__ x, int64_t ldx, int d,
                                   const int32_t* __restrict__ members,
                                   const int32_t* __restrict__ sizes, int64_t npool,
                                   const int32_t* npool_dev, int rho, int op,
                                   T* __restrict__ out, int64_t ldo) {
    using A = typename RAcc<T>::type;
    const int64_t tot = dyn_n(npool, npool_dev) * d;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / d;
        const int c = (int)(t - j * d);
        const int32_t* mem = members + j * rho;
        const int sz = sizes[j];
        auto X = [&](int r) -> A { return (A)ld_f(x + (int64_t)mem[r] * ldx + c); };
        A acc = X(0);
        if (op == R_MIN || op == R_MAX) {
            for (int r = 1; r < sz; ++r) {
                const A v = X(r);
                if (op == R_MIN) acc = v < acc ? v : acc;
                else acc = v > acc ? v : acc;
            }
        } else if (sz > 1) {
            const int nr = sz - 1;
            A res;
            if (nr < 8) {
                res = (A)0;
                for (int r = 1; r <= nr; ++r) res = res + X(r);
            } else {
                A a8[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) a8[q] = X(1 + q);
                const int full = nr - nr % 8;
                for (int i = 8; i < full; i += 8)
#pragma unroll
                    for (int q = 0; q < 8; ++q) a8[q] = a8[q] + X(1 + i + q);
                res = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
                for (int i = full; i < nr; ++i) res = res + X(1 + i);
            }
            acc = acc + res;
        }
        if (op == R_MEAN) acc = acc / (A)sz;
        st_f(out + j * ldo + c, acc);
    }
}

// fp32 rows with d % 4 == 0: one thread per (pooled row, 4 columns), float4
// loads/stores, 32-bit index math; per column the same operations in the same
// order as pool_reduce_kernel (so the same bits).
__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 f4_min(float4 a, float4 b) {
    return make_float4(b.x < a.x ? b.x : a.x, b.y < a.y ? b.y : a.y, b.z < a.z ? b.z : a.z,
                       b.w < a.w ? b.w : a.w);
}
__device__ __forceinline__ float4 f4_max(float4 a, float4 b) {
    return make_float4(b.x > a.x ? b.x : a.x, b.y > a.y ? b.y : a.y, b.z > a.z ? b.z : a.z,
                       b.w > a.w ? b.w : a.w);
}

// SMALL (rho <= 8: at most 7 terms after the first, the plain-loop branch of
// the pairwise sum) drops the eight-accumulator branch: 72 -> <= 40 registers,
// occupancy 37.5 -> 75 %, for a pass that waits on its gathered row loads.
template <bool SMALL>
__global__ void __launch_bounds__(256, SMALL ? 6 : 3) pool_reduce4_kernel(
                                    const float* __restrict__ x, int64_t ldx, int d4,
                                    const int32_t* __restrict__ members,
                                    const int32_t* __restrict__ sizes, int npool,
                                    const int32_t* npool_dev, int rho, int op,
                                    float* __restrict__ out, int64_t ldo,
                                    const __nv_bfloat16* __restrict__ y = nullptr,
                                    int64_t ldy = 0, const float* __restrict__ yb = nullptr) {
    pdl_wait();
    const int np = (int)dyn_n(npool, npool_dev);
    const uint32_t tot = (uint32_t)np * (uint32_t)d4;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += gridDim.x * blockDim.x) {
        const uint32_t j = t / (uint32_t)d4;
        const int c = 4 * (int)(t - j * (uint32_t)d4);
        const int32_t* mem = members + (int64_t)j * rho;
        const int sz = sizes[j];
        const float4 b4 = (y && yb) ? __ldg(reinterpret_cast<const float4*>(yb + c))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
        // y: the stage's pending residual, x + (y + b) with f3d_row_ln's ops
        auto X = [&](int r) -> float4 {
            float4 v = __ldg(reinterpret_cast<const float4*>(x + (int64_t)mem[r] * ldx + c));
            if (y) {
                const uint2 w = *reinterpret_cast<const uint2*>(y + (int64_t)mem[r] * ldy + c);
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
                const float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
                v.x += a.x + b4.x;
                v.y += a.y + b4.y;
                v.z += b.x + b4.z;
                v.w += b.y + b4.w;
            }
            return v;
        };
        float4 acc = X(0);
        if (op == R_MIN || op == R_MAX) {
            for (int r = 1; r < sz; ++r) acc = op == R_MIN ? f4_min(acc, X(r)) : f4_max(acc, X(r));
        } else if (sz > 1) {
            const int nr = sz - 1;
            float4 res;
            if (SMALL || nr < 8) {
                res = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int r = 1; r <= nr; ++r) res = f4_add(res, X(r));
            } else {
                float4 a8[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) a8[q] = X(1 + q);
                const int full = nr - nr % 8;
                for (int i = 8; i < full; i += 8)
#pragma unroll
                    for (int q = 0; q < 8; ++q) a8[q] = f4_add(a8[q], X(1 + i + q));
                res = f4_add(f4_add(f4_add(a8[0], a8[1]), f4_add(a8[2], a8[3])),
                             f4_add(f4_add(a8[4], a8[5]), f4_add(a8[6], a8[7])));
                for (int i = full; i < nr; ++i) res = f4_add(res, X(1 + i));
            }
            acc = f4_add(acc, res);
        }
        if (op == R_MEAN) {
            const float fs = (float)sz;
            acc = make_float4(acc.x / fs, acc.y / fs, acc.z / fs, acc.w / fs);
        }
        *reinterpret_cast<float4*>(out + (int64_t)j * ldo + c) = acc;
    }
}

}  // namespace pool
}  // namespace f3d

using namespace f3d;

extern "C" int f3d_pool_build(const double* coords, const int32_t* tile_start,
                              const int32_t* tile_m, const int32_t* tile_out, int ntiles, int rho,
                              int32_t* sub_out, int32_t* members, int32_t* sizes_out,
                              int32_t* seeds_out, int32_t* passes_out, int32_t* flags,
                              const int32_t* ntiles_dev, void* stream) {
    if (rho < 1 || rho > 64 || ntiles < 0) return F3D_ERR_CONFIG;
    cudaStream_t st = (cudaStream_t)stream;
    F3D_CUDA_TRY(f3d_zero_i32(flags, 1, st));
    if (ntiles == 0) return F3D_OK;
    pool::Args A{coords, tile_start, tile_m, tile_out, ntiles, ntiles_dev, rho, sub_out, members, sizes_out,
                 seeds_out, passes_out, flags};
    const int grid = (ntiles + pool::kWarpsPerCta - 1) / pool::kWarpsPerCta;
    const size_t smem = sizeof(pool::WarpSmem) * pool::kWarpsPerCta;
    static bool attr = false;
    if (!attr) {
        F3D_CUDA_TRY(cudaFuncSetAttribute(pool::pool_build_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    pool::pool_build_kernel<<<grid, pool::kThreads, smem, st>>>(A);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

extern "C" int f3d_pool_reduce(const void* x, int dtype, int64_t ldx, int d,
                               const int32_t* members, const int32_t* sizes, int64_t npool,
                               int rho, int op, void* out, int64_t ldo, const int32_t* npool_dev,
                               void* stream) {
    if (d < 1 || rho < 1 || op < 0 || op > 3 || npool < 0) return F3D_ERR_CONFIG;
    if (npool == 0) return F3D_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t tot = npool * d;
    int64_t g = (tot + 255) / 256;
    if (g > (int64_t)f3d_num_sms() * 32) g = (int64_t)f3d_num_sms() * 32;
    if (dtype == 2)
        pool::pool_reduce_kernel<double><<<(unsigned)g, 256, 0, st>>>(
            (const double*)x, ldx, d, members, sizes, npool, npool_dev, rho, op, (double*)out, ldo);
    else if (dtype == 1 && d % 4 == 0 && ldx % 4 == 0 && ldo % 4 == 0 &&
             (((uintptr_t)x | (uintptr_t)out) & 15) == 0 && npool * (d / 4) < ((int64_t)1 << 31)) {
        int64_t g4 = (npool * (d / 4) + 255) / 256;
        if (g4 > (int64_t)f3d_num_sms() * 32) g4 = (int64_t)f3d_num_sms() * 32;
        if (rho <= 8)
            pool::pool_reduce4_kernel<true><<<(unsigned)g4, 256, 0, st>>>(
                (const float*)x, ldx, d / 4, members, sizes, (int)npool, npool_dev, rho, op,
                (float*)out, ldo);
        else
            pool::pool_reduce4_kernel<false><<<(unsigned)g4, 256, 0, st>>>(
                (const float*)x, ldx, d / 4, members, sizes, (int)npool, npool_dev, rho, op,
                (float*)out, ldo);
    } else if (dtype == 1)
        pool::pool_reduce_kernel<float><<<(unsigned)g, 256, 0, st>>>(
            (const float*)x, ldx, d, members, sizes, npool, npool_dev, rho, op, (float*)out, ldo);
    else if (dtype == 0)
        pool::pool_reduce_kernel<__nv_bfloat16><<<(unsigned)g, 256, 0, st>>>(
            (const __nv_bfloat16*)x, ldx, d, members, sizes, npool, npool_dev, rho, op,
            (__nv_bfloat16*)out, ldo);
    else
        return F3D_ERR_CONFIG;
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

// parent[members[j*rho + r]] = j for r < sizes[j]: the pooled row of every
// scattered row, the map unpooling gathers by.
__global__ void pool_parent_kernel(const int32_t* __restrict__ members,
                                   const int32_t* __restrict__ sizes, int64_t npool,
                                   const int32_t* npool_dev, int rho, int32_t* __restrict__ parent) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t j = t / rho;
    const int r = (int)(t - j * rho);
    if (j >= dyn_n(npool, npool_dev) || r >= sizes[j]) return;
    const int32_t row = members[j * rho + r];
    if (row >= 0) parent[row] = (int32_t)j;
}

extern "C" int f3d_pool_parent(const int32_t* members, const int32_t* sizes, int64_t npool,
                               int rho, int32_t* parent, const int32_t* npool_dev, void* stream) {
    if (npool < 0 || rho < 1 || rho > 64) return F3D_ERR_CONFIG;
    if (npool == 0) return F3D_OK;
    const int64_t tot = npool * rho;
    pool_parent_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        members, sizes, npool, npool_dev, rho, parent);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

extern "C" int f3d_pool_reduce_res(const float* x, int64_t ldx, const void* y_bf16, int64_t ldy,
                                   const float* ybias, int d, const int32_t* members,
                                   const int32_t* sizes, int64_t npool, int rho, int op,
                                   float* out, int64_t ldo, const int32_t* npool_dev,
                                   void* stream) {
    if (d < 4 || d % 4 || rho < 1 || op < 0 || op > 3 || npool < 0 || ldx % 4 || ldo % 4 ||
        ldy % 4 || (((uintptr_t)x | (uintptr_t)out | (uintptr_t)ybias) & 15) ||
        ((uintptr_t)y_bf16 & 7) || npool * (d / 4) >= ((int64_t)1 << 31))
        return F3D_ERR_CONFIG;
    if (npool == 0) return F3D_OK;
    int64_t g4 = (npool * (d / 4) + 255) / 256;
    if (g4 > (int64_t)f3d_num_sms() * 32) g4 = (int64_t)f3d_num_sms() * 32;
    if (rho <= 8)
        F3D_CUDA_TRY(f3d_launch(pool::pool_reduce4_kernel<true>, dim3((unsigned)g4), dim3(256), 0,
                                (cudaStream_t)stream, x, ldx, d / 4, members, sizes, (int)npool,
                                npool_dev, rho, op, out, ldo, (const __nv_bfloat16*)y_bf16, ldy,
                                ybias));
    else
        F3D_CUDA_TRY(f3d_launch(pool::pool_reduce4_kernel<false>, dim3((unsigned)g4), dim3(256), 0,
                                (cudaStream_t)stream, x, ldx, d / 4, members, sizes, (int)npool,
                                npool_dev, rho, op, out, ldo, (const __nv_bfloat16*)y_bf16, ldy,
                                ybias));
    return F3D_OK;
}
