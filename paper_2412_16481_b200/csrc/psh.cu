// PSH bucket assignment: exact parallel fill-time fixed point.
//
// Reference semantics (bw/_kernels.py:41-90, bw/bucketing.py:275-320): per
// batch, points are visited in index order; a point takes its home bucket if
// fewer than S earlier points hold it, else the first of P clamped probe
// buckets with room (strict-div probes that hash to -1 are skipped), else the
// unbounded recycle bucket K; its offset is its pre-increment count.
//
// Parallel restatement: let T[c] be the (sorted-domain) position of the point
// holding slot S-1 of bucket c (INT_MAX if c never fills).  Point p has room in
// c  <=>  fewer than S earlier takers  <=>  T[c] >= p.  Iterate
//     D <- home;  repeat { T <- S-th taker of each bucket under D;
//                          D' <- first candidate c with T[c] >= p, else K }
// until D' == D.  By induction on p every fixed point equals the sequential
// result, and prefix p is correct after p+1 sweeps, so it terminates.
//
// One cooperative launch runs everything: an optional stable batch sort, the
// sweeps (decide + per-tile histograms, column scans over tiles, in-tile
// stable ranks via __match_any_sync), and the final base/dest pass.  Points
// live in tiles of 2048 (8 warps x 8 rounds x 32 lanes); per-warp u16
// histograms of the K+1 local buckets sit in shared memory.
#include <algorithm>
#include <climits>

#include "f3d_common.cuh"

namespace f3d {
namespace psh {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
// Points per lane (PL) is a kernel template parameter: tiles of kWarps*32*PL
// points.  Small scenes want small tiles (more CTAs in the latency-bound
// sweeps: config B 100K points 53 -> 43 us with PL = 2), large ones large
// tiles (config D 1M points 172 us with PL = 8 vs 269 with PL = 2).
constexpr int kPerLaneSmall = 2, kPerLaneLarge = 8;
constexpr int64_t kSmallTileMaxN = 300000;   // n below this: PL = 2
template <int PL> struct TileC {
    static constexpr int kPerLane = PL;
    static constexpr int kWarpSpan = 32 * PL;
    static constexpr int kTile = kWarps * 32 * PL;
};
constexpr int kTileMin = kWarps * 32 * kPerLaneSmall;   // workspace sizing (most tiles)
constexpr int kMaxBins = 12288;               // smem histogram limit (8 * 12288 * 2 B)
constexpr int kMaxProbes = 128;
constexpr int kScanU = 4;

enum { INFO_SWEEPS = 0, INFO_FALLBACK = 1, INFO_BATCH_ERR = 2 };

struct Params {
    const int32_t* vox;    // (n,3) original order
    const int32_t* home;   // (n)
    const int32_t* batch;  // (n) or null
    int n, nbatch, K, S, P, max_sweeps;
    const int32_t* n_dev;  // nullable: device point count (<= n), single batch only
    HashParams hp;
    int vmax;
    int8_t probe[kMaxProbes * 3];
    int32_t *bucket_id, *bucket_offset, *counts, *base, *dest, *info;
    // workspace
    int4* pk;          // sorted domain: x, y, z, home
    int32_t* D;        // sorted domain decision (local bucket id)
    int32_t* off;      // sorted domain offset
    int32_t* orig;     // sorted -> original index (multi-batch)
    int32_t* T0;       // nslots
    int32_t* T1;       // nslots
    int32_t* hist;     // max_tiles * max(K+1, nbatch)
    int32_t* tile_p0;  // sorted-domain tile start (multi), max_tiles + 1
    int32_t* tile_b;   // tile -> batch (multi)
    int32_t* btile;    // batch -> first tile (multi), nbatch + 1
    int32_t* bstart;   // batch -> first sorted position, nbatch + 1
    int32_t* flags;    // max_sweeps + 2 "changed" words
    unsigned* bar;     // grid barrier counter (zeroed before the launch)
    int max_tiles;
    int base_in_smem;    // nbatch*(K+1) ints of dynamic smem past the histograms
    // fused voxelize + remap + hash (f3d_psh_assign_coords; single batch):
    // the kernel reads the float64 coordinates itself instead of vox / home
    const double* coords;
    double org[3];
    double vs;
    int64_t* stats;      // [min x,y,z, max x,y,z, max quotient] of the remapped voxels
    long long* part;     // per-CTA partial extrema, 8 per CTA
};

// Grid-wide barrier on a per-call counter in the caller's workspace (zeroed
// by a small kernel before the launch; the launch is still cooperative, for
// co-residency):
// every call's barrier state is its own, whatever else runs concurrently
// (two Backbones on two streams, tests/test_gpu_backbone.py;
// tools/psh_concurrency.py).
struct GridBar {
    unsigned* ctr;
    unsigned target;
    __device__ __forceinline__ void sync() {
        __syncthreads();
        if (threadIdx.x == 0) {
            target += gridDim.x;                 // monotonic: barrier k ends at k * grid
            unsigned cur;
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
            do {
                asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(ctr) : "memory");
            } while (cur < target);
        }
        __syncthreads();
    }
};

// floor((c - o) / vs) with no contraction: __dsub_rn then __ddiv_rn
// (bw/geometry.py:69-72; the same arithmetic as csrc/hash.cu)
__device__ __forceinline__ long long vox_floor(double c, double o, double vs) {
    return vox_floor_inv(c, o, vs, __drcp_rn(vs));
}

// Block-wide min (kMin) / max of 64-bit values into out[] (thread 0 writes).
template <int N, int kMin>
__device__ __forceinline__ void block_extrema(long long (&v)[N], long long* sh, long long* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < N; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long b = __shfl_xor_sync(0xffffffffu, v[k], o);
            v[k] = k < kMin ? min(v[k], b) : max(v[k], b);
        }
        if (lane == 0) sh[warp * N + k] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < N) {
        const int k = threadIdx.x;
        long long a = sh[k];
        for (int w = 1; w < kWarps; ++w) a = k < kMin ? min(a, sh[w * N + k]) : max(a, sh[w * N + k]);
        out[k] = a;
    }
    __syncthreads();
}

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ void zero_hist(uint16_t* h, int words32) {
    uint32_t* w = reinterpret_cast<uint32_t*>(h);
    for (int i = threadIdx.x; i < words32; i += kThreads) w[i] = 0u;
}

// Count this warp's keys into its private u16 row (keys < 0 ignored).
template <int kPerLane>
__device__ __forceinline__ void warp_count(const int (&key)[kPerLane], uint16_t* row) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < kPerLane; ++j) {
        const int k = key[j];
        const unsigned m = __match_any_sync(0xffffffffu, k);
        if (k >= 0 && lane == __ffs(m) - 1) row[k] = (uint16_t)(row[k] + __popc(m));
        __syncwarp();
    }
}

// Stable rank of each key within the tile, given row = exclusive prefix of
// this warp's keys over earlier warps of the tile.
template <int kPerLane>
__device__ __forceinline__ void warp_rank(const int (&key)[kPerLane], uint16_t* row,
                                          int (&rank)[kPerLane]) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < kPerLane; ++j) {
        const int k = key[j];
        const unsigned m = __match_any_sync(0xffffffffu, k);
        const int b = (k >= 0) ? (int)row[k] : 0;
        rank[j] = b + __popc(m & lt);
        __syncwarp();
        if (k >= 0 && lane == __ffs(m) - 1) row[k] = (uint16_t)(b + __popc(m));
        __syncwarp();
    }
}

// Sum the per-warp rows into hist_row (global), one int per bin.
__device__ __forceinline__ void store_tile_hist(const uint16_t* h, int stride, int nbins,
                                                int32_t* hist_row) {
    for (int c = threadIdx.x; c < nbins; c += kThreads) {
        int s = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += h[w * stride + c];
        hist_row[c] = s;
    }
}

// Exclusive prefix across the warps, in place (values stay < 2048).
__device__ __forceinline__ void warp_prefix_rows(uint16_t* h, int stride, int nbins) {
    for (int c = threadIdx.x; c < nbins; c += kThreads) {
        int run = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const int t = h[w * stride + c];
            h[w * stride + c] = (uint16_t)run;
            run += t;
        }
    }
}

// One warp: exclusive scan of hist[t*stride + col] over tiles [t0, t1) in
// place; returns the column total.
__device__ int column_scan(int32_t* hist, int stride, int col, int t0, int t1) {
    const int lane = threadIdx.x & 31;
    int carry = 0;
    for (int base = t0; base < t1; base += 32 * kScanU) {
        int v[kScanU];
        int s = 0;
#pragma unroll
        for (int u = 0; u < kScanU; ++u) {
            const int t = base + lane * kScanU + u;
            v[u] = (t < t1) ? __ldcg(hist + (int64_t)t * stride + col) : 0;
            s += v[u];
        }
        const int incl = warp_incl_scan(s);
        int e = carry + incl - s;
#pragma unroll
        for (int u = 0; u < kScanU; ++u) {
            const int t = base + lane * kScanU + u;
            if (t < t1) hist[(int64_t)t * stride + col] = e;
            e += v[u];
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    return carry;
}

// First candidate bucket with room for point p (T[c] >= p), else K.
__device__ __forceinline__ int decide(const int4 q, int p, const int32_t* __restrict__ T,
                                      const Params& P_, const int8_t* probe) {
    if (__ldcg(T + q.w) >= p) return q.w;
#ifndef F3D_PSH_CHUNK
#define F3D_PSH_CHUNK 2   // measured (config D, 1M points): 2 -> 98 us, 4 -> 118, 8 -> 115
#endif
    constexpr int kChunk = F3D_PSH_CHUNK;   // candidates hashed (and their T loaded) per step
    for (int p0 = 0; p0 < P_.P; p0 += kChunk) {
        int cand[kChunk];
#pragma unroll
        for (int u = 0; u < kChunk; ++u) {
            const int pi = p0 + u;
            cand[u] = -1;
            if (pi < P_.P) {
                const int x = min(max(q.x + (int)probe[3 * pi + 0], 0), P_.vmax);
                const int y = min(max(q.y + (int)probe[3 * pi + 1], 0), P_.vmax);
                const int z = min(max(q.z + (int)probe[3 * pi + 2], 0), P_.vmax);
                cand[u] = hash_bucket1(x, y, z, P_.hp);
            }
        }
        int tv[kChunk];
#pragma unroll
        for (int u = 0; u < kChunk; ++u) tv[u] = cand[u] >= 0 ? __ldcg(T + cand[u]) : -1;
#pragma unroll
        for (int u = 0; u < kChunk; ++u)
            if (cand[u] >= 0 && tv[u] >= p) return cand[u];
    }
    return P_.K;
}

struct TileInfo {
    int p0, p1, b;
};

template <int kTile>
__device__ __forceinline__ TileInfo tile_info(const Params& P_, bool multi, int t, int n) {
    TileInfo ti;
    if (multi) {
        ti.p0 = __ldcg(P_.tile_p0 + t);
        ti.b = __ldcg(P_.tile_b + t);
        ti.p1 = min(ti.p0 + kTile, __ldcg(P_.bstart + ti.b + 1));
    } else {
        ti.p0 = t * kTile;
        ti.p1 = min(ti.p0 + kTile, n);
        ti.b = 0;
    }
    return ti;
}

// Exact sequential semantics, 32 points at a time (one warp): the App. A
// fixed point on a window.  With the counters ctr at the window start, lane i
// takes the first candidate c with ctr[c] + #{j < i : D_j = c} < S (home,
// then the clamped probes, strict -1 skipped), else the recycle bucket K.
// Iterate from D = home until no lane changes: lane i is final after i + 1
// iterations (its decision depends only on lanes j < i), so at most 33
// iterations.  Then offset = ctr[D] + rank among the earlier lanes with the
// same D, and ctr[c] += takers.  ctr may live in shared or global memory
// (only this warp touches it); sD is this warp's 32-int scratch.
// Replaces the reference's per-point loop (bw/_kernels.py:41-90) with a
// 32-wide window; the decisions are identical (same induction as App. A).
__device__ void warp_exact_window(const Params& P_, int32_t* ctr, const int4 q, bool active,
                                  int* sD, const int8_t* probe, int& d_out, int& off_out) {
    const int lane = threadIdx.x & 31;
    const int S = P_.S;
    int D = active ? q.w : -1;
    for (int iter = 0; iter < 34; ++iter) {
        sD[lane] = D;
        __syncwarp();
        int nd = -1;
        if (active) {
            // room for this lane in c given the earlier lanes' current choices
            auto room = [&](int c) -> bool {
                const int base = ctr[c];
                if (base >= S) return false;                // full at the window start
                if (base + lane < S) return true;           // < lane earlier takers fit
                int cnt = 0;
                for (int j = 0; j < lane; ++j) cnt += (sD[j] == c);
                return base + cnt < S;
            };
            if (room(q.w)) {
                nd = q.w;
            } else {
                for (int pi = 0; pi < P_.P; ++pi) {
                    const int x = min(max(q.x + (int)probe[3 * pi + 0], 0), P_.vmax);
                    const int y = min(max(q.y + (int)probe[3 * pi + 1], 0), P_.vmax);
                    const int z = min(max(q.z + (int)probe[3 * pi + 2], 0), P_.vmax);
                    const int c = hash_bucket1(x, y, z, P_.hp);
                    if (c >= 0 && room(c)) {
                        nd = c;
                        break;
                    }
                }
                if (nd < 0) nd = P_.K;
            }
        }
        const bool ch = __any_sync(0xffffffffu, nd != D);
        __syncwarp();                                       // sD reads done
        D = nd;
        if (!ch) break;
    }
    const unsigned m = __match_any_sync(0xffffffffu, D);
    off_out = active ? ctr[D] + __popc(m & lanemask_lt()) : 0;
    d_out = D;
    __syncwarp();
    if (active && lane == __ffs(m) - 1) ctr[D] += __popc(m);
    __syncwarp();
}

// One batch of the sorted domain [pb0, pb1) by one warp, counters in ctr
// (W ints; written to counts[b] at the end).
__device__ void warp_exact_batch(const Params& P_, int b, int pb0, int pb1, int32_t* ctr,
                                 int* sD, const int8_t* probe) {
    const int lane = threadIdx.x & 31;
    const int W = P_.K + 1;
    for (int c = lane; c < W; c += 32) ctr[c] = 0;
    __syncwarp();
    for (int w0 = pb0; w0 < pb1; w0 += 32) {
        const int p = w0 + lane;
        const bool active = p < pb1;
        const int4 q = active ? __ldcg(P_.pk + p) : make_int4(0, 0, 0, 0);
        int d, o;
        warp_exact_window(P_, ctr, q, active, sD, probe, d, o);
        if (active) {
            P_.D[p] = d;
            P_.off[p] = o;
        }
    }
    __syncwarp();
    for (int c = lane; c < W; c += 32) P_.counts[(int64_t)b * W + c] = ctr[c];
}

// Exclusive scan of the nslots slot counts (block-wide): block 0 writes base
// (when write_global), and s_base (nullable) receives a shared-memory copy.
__device__ void slot_base(const Params& P_, int nslots, int32_t* s_base, bool write_global) {
    const int tid = threadIdx.x, lane = tid & 31;
    __shared__ int s_part[kThreads];
    __syncthreads();
    const int per = (nslots + kThreads - 1) / kThreads;
    const int a0 = min(tid * per, nslots), a1 = min(a0 + per, nslots);
    int s = 0;
    for (int i = a0; i < a1; ++i) s += __ldcg(P_.counts + i);
    s_part[tid] = s;
    __syncthreads();
    if (tid < 32) {
        int acc = 0;
        for (int w = 0; w < kThreads / 32; ++w) {
            const int v = s_part[w * 32 + lane];
            const int incl = warp_incl_scan(v);
            s_part[w * 32 + lane] = acc + incl - v;
            acc += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    __syncthreads();
    int run = s_part[tid];
    for (int i = a0; i < a1; ++i) {
        if (write_global) P_.base[i] = run;
        if (s_base) s_base[i] = run;
        run += __ldcg(P_.counts + i);
    }
    __syncthreads();
}

// --------------------------------------------------------------- the kernel

template <int PL, bool FUSED>
__global__ void __launch_bounds__(kThreads, FUSED ? 2 : 4) psh_kernel(const Params P_) {
    constexpr int kPerLane = TileC<PL>::kPerLane;
    constexpr int kWarpSpan = TileC<PL>::kWarpSpan;
    constexpr int kTile = TileC<PL>::kTile;
    GridBar grid{P_.bar, 0u};
    extern __shared__ __align__(16) uint16_t sh[];
    __shared__ int8_t probe[kMaxProbes * 3];
    __shared__ int s_flag;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const bool multi = P_.nbatch > 1;
    const int n = (int)dyn_n(P_.n, P_.n_dev);
    const int K = P_.K;
    const int W = K + 1;
    const int nbins = multi ? max(W, P_.nbatch) : W;
    const int stride = (nbins + 1) & ~1;  // u16 row stride, even
    uint16_t* myrow = sh + warp * stride;
    const int hwords = kWarps * stride / 2;

    for (int i = tid; i < P_.P * 3; i += kThreads) probe[i] = P_.probe[i];
    if (blockIdx.x == 0)
        for (int i = tid; i < P_.max_sweeps + 2; i += kThreads) P_.flags[i] = 0;

    const int gwarp = blockIdx.x * kWarps + warp;
    const int nwarps = gridDim.x * kWarps;

    // ------------------------------- fused: voxelize + per-axis extrema
    __shared__ long long s_red[kWarps * 6];
    __shared__ long long s_gmin[3];
    long long qmax = LLONG_MIN;          // largest div quotient seen (stats[6])
    // raw voxel coordinates of this thread's points of sweep 0, kept in
    // registers across the extrema barrier when every CTA owns <= 1 tile
    long long raw[kPerLane][3];
    bool cached = false;
    if constexpr (FUSED) {
        long long v[6] = {LLONG_MAX, LLONG_MAX, LLONG_MAX, LLONG_MIN, LLONG_MIN, LLONG_MIN};
        const int nt0 = cdiv_dev(n, kTile);
        cached = nt0 <= (int)gridDim.x;
        for (int t = blockIdx.x; t < nt0; t += gridDim.x) {   // the sweeps' tile mapping
#pragma unroll
            for (int j = 0; j < kPerLane; ++j) {
                const int p = t * kTile + warp * kWarpSpan + j * 32 + lane;
                if (p >= n) continue;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const long long x = vox_floor(P_.coords[3 * (int64_t)p + a], P_.org[a], P_.vs);
                    raw[j][a] = x;
                    v[a] = min(v[a], x);
                    v[3 + a] = max(v[3 + a], x);
                }
            }
        }
        block_extrema<6, 3>(v, s_red, P_.part + 8 * blockIdx.x);
        grid.sync();
        // every CTA reduces the partials: warp a < 3 the minimum of axis a
        if (warp < 3) {
            long long m = LLONG_MAX;
            for (int b = lane; b < (int)gridDim.x; b += 32) m = min(m, __ldcg(P_.part + 8 * b + warp));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) s_gmin[warp] = m;
        }
        __syncthreads();
    }

    int ntiles;
    // ------------------------------------------------ stable batch sort
    if (multi) {
        const int B = P_.nbatch;
        const int nto = cdiv_dev(P_.n, kTile);
        for (int t = blockIdx.x; t < nto; t += gridDim.x) {
            zero_hist(sh, hwords);
            __syncthreads();
            int key[kPerLane];
#pragma unroll
            for (int j = 0; j < kPerLane; ++j) {
                const int i = t * kTile + warp * kWarpSpan + j * 32 + lane;
                int b = -1;
                if (i < P_.n) {
                    b = P_.batch[i];
                    if (b < 0 || b >= B) {
                        atomicOr(P_.info + INFO_BATCH_ERR, 1);
                        b = -1;
                    }
                }
                key[j] = b;
            }
            warp_count(key, myrow);
            __syncthreads();
            store_tile_hist(sh, stride, B, P_.hist + (int64_t)t * B);
            __syncthreads();
        }
        grid.sync();
        for (int b = gwarp; b < B; b += nwarps) {
            const int tot = column_scan(P_.hist, B, b, 0, nto);
            if (lane == 0) P_.counts[b] = tot;  // temp: batch sizes
        }
        grid.sync();
        if (blockIdx.x == 0 && tid == 0) {
            int pos = 0, tl = 0;
            for (int b = 0; b < B; ++b) {
                const int cb = __ldcg(P_.counts + b);
                if (cb == 0) P_.info[INFO_BATCH_ERR] |= 2;  // non-contiguous ids
                P_.bstart[b] = pos;
                P_.btile[b] = tl;
                for (int q = 0; q < cb; q += kTile) {
                    P_.tile_p0[tl] = pos + q;
                    P_.tile_b[tl] = b;
                    ++tl;
                }
                pos += cb;
            }
            P_.bstart[B] = pos;
            P_.btile[B] = tl;
        }
        grid.sync();
        for (int t = blockIdx.x; t < nto; t += gridDim.x) {
            zero_hist(sh, hwords);
            __syncthreads();
            int key[kPerLane];
#pragma unroll
            for (int j = 0; j < kPerLane; ++j) {
                const int i = t * kTile + warp * kWarpSpan + j * 32 + lane;
                int b = (i < P_.n) ? P_.batch[i] : -1;
                key[j] = (b >= 0 && b < B) ? b : -1;
            }
            warp_count(key, myrow);
            __syncthreads();
            warp_prefix_rows(sh, stride, B);
            __syncthreads();
            int rank[kPerLane];
            warp_rank(key, myrow, rank);
#pragma unroll
            for (int j = 0; j < kPerLane; ++j) {
                const int i = t * kTile + warp * kWarpSpan + j * 32 + lane;
                if (key[j] >= 0) {
                    const int b = key[j];
                    const int pos = __ldcg(P_.bstart + b) + __ldcg(P_.hist + (int64_t)t * B + b) + rank[j];
                    P_.orig[pos] = i;
                    P_.pk[pos] = make_int4(P_.vox[3 * (int64_t)i], P_.vox[3 * (int64_t)i + 1],
                                           P_.vox[3 * (int64_t)i + 2], P_.home[i]);
                }
            }
            __syncthreads();
        }
        grid.sync();
        ntiles = __ldcg(P_.btile + B);
    } else {
        ntiles = cdiv_dev(n, kTile);
    }

    // ------------------------------------------------------------ sweeps
    const int nslots = P_.nbatch * W;
    // the slot base scan in shared memory, past the histogram rows (host
    // decides whether it fits)
    const bool local_base = P_.base_in_smem != 0;
    int32_t* s_base = reinterpret_cast<int32_t*>(sh + kWarps * stride);
    bool converged0 = false;
    int32_t* Tc = P_.T0;
    int32_t* Tn = P_.T1;
    int sweep = 0;
    bool fallback = false;
    // Sweep 0 with at most one tile per CTA: phase A ranks its keys within
    // each warp while counting them (warp_rank instead of warp_count) and
    // keeps keys and ranks in registers, and the per-warp rows stay in shared
    // memory; when sweep 0 is final, phase C only turns the rows into
    // cross-warp prefixes -- no second read of D, count and rank pass.
    const bool one_tile = ntiles <= (int)gridDim.x;
    // key | (in-warp rank << 16), -1 for no point (keys < 2^14, ranks < 2^11)
    uint32_t kra[kPerLane];
    for (;;) {
        // Phase A: decide + per-tile histogram
        int changed = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const TileInfo ti = tile_info<kTile>(P_, multi, t, n);
            zero_hist(sh, hwords);
            __syncthreads();
            int key[kPerLane];
            const int32_t* Tb = Tc + (int64_t)ti.b * W;
#pragma unroll
            for (int j = 0; j < kPerLane; ++j) {
                const int p = ti.p0 + warp * kWarpSpan + j * 32 + lane;
                int k = -1;
                if (p < ti.p1) {
                    if (sweep == 0) {
                        int4 q;
                        if constexpr (FUSED) {
                            // remap (subtract the axis minimum), range check, home
                            // hash: the arithmetic of hash.cu hash_point
                            // (bw/hashing.py:60-149)
                            long long c3[3];
#pragma unroll
                            for (int a = 0; a < 3; ++a)
                                c3[a] = (cached ? raw[j][a]
                                                : vox_floor(P_.coords[3 * (int64_t)p + a], P_.org[a],
                                                            P_.vs)) -
                                        s_gmin[a];
                            const long long lim = 1ll << P_.hp.bits;
                            q = make_int4(0, 0, 0, 0);
                            if (c3[0] < lim && c3[1] < lim && c3[2] < lim) {
                                int64_t key = P_.hp.kind <= XOR_DIV ? (c3[0] ^ c3[1] ^ c3[2])
                                                                    : morton3(c3[0], c3[1], c3[2]);
                                if (P_.hp.kind == XOR_DIV || P_.hp.kind == ZORDER_DIV) {
                                    key = (key < 0x7FFFFFFFll && P_.hp.S_div < 0x7FFFFFFFll)
                                              ? (int64_t)P_.hp.fdiv.div((uint32_t)key)
                                              : key / P_.hp.S_div;
                                    qmax = max(qmax, (long long)key);
                                }
                                const int hk = key < 0x7FFFFFFFll ? (int)P_.hp.fk.mod((uint32_t)key)
                                                                  : (int)(key % P_.K);
                                q = make_int4((int)c3[0], (int)c3[1], (int)c3[2], hk);
                            }
                            P_.pk[p] = q;
                        } else if (multi) {
                            q = __ldcg(P_.pk + p);
                        } else {
                            q = make_int4(P_.vox[3 * (int64_t)p], P_.vox[3 * (int64_t)p + 1],
                                          P_.vox[3 * (int64_t)p + 2], P_.home[p]);
                            P_.pk[p] = q;
                        }
                        k = q.w;
                        if (k < 0 || k >= K) {  // precondition: home in [0, K)
                            atomicOr(P_.info + INFO_BATCH_ERR, 4);
                            k = K;
                        }
                    } else {
                        const int4 q = __ldcg(P_.pk + p);
                        k = decide(q, p, Tb, P_, probe);
                        changed |= (k != P_.D[p]);
                    }
                    P_.D[p] = k;
                }
                key[j] = k;
            }
            if (sweep == 0 && one_tile) {
                int rank[kPerLane];
                warp_rank(key, myrow, rank);
#pragma unroll
                for (int j = 0; j < kPerLane; ++j)
                    kra[j] = key[j] < 0 ? 0xFFFFFFFFu : (uint32_t)key[j] | ((uint32_t)rank[j] << 16);
            } else {
                warp_count(key, myrow);
            }
            __syncthreads();
            store_tile_hist(sh, stride, W, P_.hist + (int64_t)t * W);
            __syncthreads();
        }
        if (sweep > 0) {
            const int any = __syncthreads_or(changed);
            if (tid == 0 && any) atomicOr(P_.flags + sweep, 1);
        }
        if constexpr (FUSED) {
            if (sweep == 0) {
                long long qv[1] = {qmax};
                block_extrema<1, 0>(qv, s_red, P_.part + 8 * blockIdx.x + 6);
            }
        }
        grid.sync();
        if (sweep > 0) {
            if (tid == 0) s_flag = *((volatile int32_t*)(P_.flags + sweep));
            __syncthreads();
            if (s_flag == 0) break;  // D unchanged: previous offsets are final
        }
        if (sweep >= P_.max_sweeps) {
            fallback = true;
            break;
        }
        // Phase B: column scans over each batch's tiles; counts; T reset
        {
            const int ncols = P_.nbatch * W;
            for (int col = gwarp; col < ncols; col += nwarps) {
                const int b = col / W;
                const int c = col - b * W;
                const int t0 = multi ? __ldcg(P_.btile + b) : 0;
                const int t1 = multi ? __ldcg(P_.btile + b + 1) : ntiles;
                const int tot = column_scan(P_.hist, W, c, t0, t1);
                if (lane == 0) {
                    P_.counts[col] = tot;
                    if (c < K && tot < P_.S) Tn[col] = INT_MAX;
                    // sweep 0 (D = home): no bucket above S means every point
                    // is among its home's first S takers -- D = home is the
                    // fixed point and this sweep's offsets are final
                    if (sweep == 0 && c < K && tot > P_.S) atomicOr(P_.flags, 1);
                }
            }
        }
        grid.sync();
        // sweep 0 without overflow: phase C writes the final outputs itself
        // (base scanned locally from the counts), no further sweep or barrier
        bool final_c = false;
        if (sweep == 0 && local_base) {
            if (tid == 0) s_flag = *((volatile int32_t*)P_.flags);
            __syncthreads();
            final_c = s_flag == 0;
            if (final_c) slot_base(P_, nslots, s_base, blockIdx.x == 0);
        }
        // Phase C: in-tile stable ranks -> offsets; S-th taker -> T
        if (final_c && one_tile) {
            const int t = blockIdx.x;
            if (t < ntiles) {
                const TileInfo ti = tile_info<kTile>(P_, multi, t, n);
                warp_prefix_rows(sh, stride, W);       // phase A's per-warp counts
                __syncthreads();
                const int32_t* hrow = P_.hist + (int64_t)t * W;
#pragma unroll
                for (int j = 0; j < kPerLane; ++j) {
                    const int p = ti.p0 + warp * kWarpSpan + j * 32 + lane;
                    if (kra[j] != 0xFFFFFFFFu) {
                        const int k = (int)(kra[j] & 0xFFFFu);
                        const int o = __ldcg(hrow + k) + myrow[k] + (int)(kra[j] >> 16);
                        const int i = multi ? __ldcg(P_.orig + p) : p;
                        P_.bucket_id[i] = k;
                        P_.bucket_offset[i] = o;
                        P_.dest[i] = s_base[ti.b * W + k] + o;
                    }
                }
            }
            converged0 = true;
            break;
        }
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const TileInfo ti = tile_info<kTile>(P_, multi, t, n);
            zero_hist(sh, hwords);
            __syncthreads();
            int key[kPerLane];
#pragma unroll
            for (int j = 0; j < kPerLane; ++j) {
                const int p = ti.p0 + warp * kWarpSpan + j * 32 + lane;
                key[j] = (p < ti.p1) ? P_.D[p] : -1;
            }
            warp_count(key, myrow);
            __syncthreads();
            warp_prefix_rows(sh, stride, W);
            __syncthreads();
            int rank[kPerLane];
            warp_rank(key, myrow, rank);
            const int32_t* hrow = P_.hist + (int64_t)t * W;
#pragma unroll
            for (int j = 0; j < kPerLane; ++j) {
                const int p = ti.p0 + warp * kWarpSpan + j * 32 + lane;
                if (key[j] >= 0) {
                    const int o = __ldcg(hrow + key[j]) + rank[j];
                    if (final_c) {
                        const int i = multi ? __ldcg(P_.orig + p) : p;
                        P_.bucket_id[i] = key[j];
                        P_.bucket_offset[i] = o;
                        P_.dest[i] = s_base[ti.b * W + key[j]] + o;
                    } else {
                        P_.off[p] = o;
                        if (key[j] < K && o == P_.S - 1) Tn[(int64_t)ti.b * W + key[j]] = p;
                    }
                }
            }
            __syncthreads();
        }
        if (final_c) {
            converged0 = true;
            break;
        }
        grid.sync();
        int32_t* tmp = Tc;
        Tc = Tn;
        Tn = tmp;
        ++sweep;
    }

    if (fallback) {
        // Exact path past max_sweeps: one warp per batch (warp 0 of CTAs
        // b, b + grid, ...), 32-point windows, counters in shared memory.
        __shared__ int sD[32];
        if (warp == 0) {
            int32_t* ctr = reinterpret_cast<int32_t*>(sh);   // W ints <= the histogram area
            for (int b = blockIdx.x; b < P_.nbatch; b += gridDim.x) {
                const int pb0 = multi ? __ldcg(P_.bstart + b) : 0;
                const int pb1 = multi ? __ldcg(P_.bstart + b + 1) : n;
                warp_exact_batch(P_, b, pb0, pb1, ctr, sD, probe);
            }
        }
        grid.sync();
    }

    // ------------------------------------------- final: base scan, dest
    // The exclusive scan of the slot counts is small: when it fits in this
    // CTA's shared memory every CTA computes it itself (block 0 also writes
    // base) and goes straight on to its tiles' dest -- no grid barrier.
    if (!converged0 && (local_base || blockIdx.x == 0))
        slot_base(P_, nslots, local_base ? s_base : nullptr, blockIdx.x == 0);
    if (blockIdx.x == 0 && tid == 0) {
        P_.info[INFO_SWEEPS] = sweep + 1;
        P_.info[INFO_FALLBACK] = fallback ? 1 : 0;
        if constexpr (FUSED) {
            // range statistics of the remapped voxels (min is 0 by construction)
            long long mx[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN}, q = LLONG_MIN;
            for (int b = 0; b < (int)gridDim.x; ++b) {
                for (int a = 0; a < 3; ++a) mx[a] = max(mx[a], __ldcg(P_.part + 8 * b + 3 + a));
                q = max(q, __ldcg(P_.part + 8 * b + 6));
            }
            for (int a = 0; a < 3; ++a) {
                P_.stats[a] = n > 0 ? 0 : LLONG_MAX;
                P_.stats[3 + a] = n > 0 ? mx[a] - s_gmin[a] : LLONG_MIN;
            }
            P_.stats[6] = q;
            P_.info[INFO_BATCH_ERR] = 0;     // single batch, home in [0, K) by construction
            P_.info[3] = 0;
        }
    }
    if (converged0) return;
    if (!local_base) grid.sync();
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TileInfo ti = tile_info<kTile>(P_, multi, t, n);
        const int32_t* bb = local_base ? s_base + ti.b * W : P_.base + (int64_t)ti.b * W;
        for (int p = ti.p0 + tid; p < ti.p1; p += kThreads) {
            const int i = multi ? __ldcg(P_.orig + p) : p;
            const int d = __ldcg(P_.D + p);
            const int o = __ldcg(P_.off + p);
            P_.bucket_id[i] = d;
            P_.bucket_offset[i] = o;
            P_.dest[i] = (local_base ? bb[d] : __ldcg(bb + d)) + o;
        }
    }
}

struct WsLayout {
    size_t pk, D, off, orig, T0, T1, hist, tile_p0, tile_b, btile, bstart, flags, bar, total;
};

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static WsLayout layout(int64_t n, int32_t nbatch, int32_t K, int max_sweeps) {
    WsLayout L;
    const int64_t max_tiles = n / kTileMin + nbatch + 1;
    const int64_t nslots = (int64_t)nbatch * (K + 1);
    const int64_t nbins = nbatch > 1 ? std::max<int64_t>(K + 1, nbatch) : (K + 1);
    size_t o = 0;
    L.pk = o;      o = align256(o + sizeof(int4) * n);
    L.D = o;       o = align256(o + 4 * n);
    L.off = o;     o = align256(o + 4 * n);
    L.orig = o;    o = align256(o + (nbatch > 1 ? 4 * n : 4));
    L.T0 = o;      o = align256(o + 4 * nslots);
    L.T1 = o;      o = align256(o + 4 * nslots);
    L.hist = o;    o = align256(o + 4 * max_tiles * nbins);
    L.tile_p0 = o; o = align256(o + 4 * (max_tiles + 1));
    L.tile_b = o;  o = align256(o + 4 * (max_tiles + 1));
    L.btile = o;   o = align256(o + 4 * (nbatch + 1));
    L.bstart = o;  o = align256(o + 4 * (nbatch + 1));
    L.flags = o;   o = align256(o + 4 * (max_sweeps + 2));
    L.bar = o;     o = align256(o + 4);
    L.total = o;
    return L;
}

constexpr int kMaxSweepsCap = 4096;

}  // namespace psh
}  // namespace f3d

using namespace f3d;

extern "C" size_t f3d_psh_workspace_size(int64_t n, int32_t nbatch, int32_t K) {
    return psh::layout(n, nbatch, K, psh::kMaxSweepsCap).total;
}

// Bucket counts beyond the shared-memory histogram limit: one warp per batch
// over the original order (32-index windows, lanes of other batches idle),
// counters in the batch's slice of counts (global).  Then one CTA scans the
// slot counts and writes dest.
__global__ void __launch_bounds__(32) psh_warp_exact_kernel(psh::Params P_) {
    __shared__ int sD[32];
    __shared__ int8_t probe[psh::kMaxProbes * 3];
    const int lane = threadIdx.x;
    const int b = blockIdx.x;
    const int W = P_.K + 1;
    const int n = (int)dyn_n(P_.n, P_.n_dev);
    for (int i = lane; i < P_.P * 3; i += 32) probe[i] = P_.probe[i];
    int32_t* ctr = P_.counts + (int64_t)b * W;
    for (int c = lane; c < W; c += 32) ctr[c] = 0;
    __syncwarp();
    for (int w0 = 0; w0 < n; w0 += 32) {
        const int i = w0 + lane;
        bool active = i < n;
        if (active && P_.batch) {
            const int bi = P_.batch[i];
            if (b == 0 && (bi < 0 || bi >= P_.nbatch)) atomicOr(P_.info + psh::INFO_BATCH_ERR, 1);
            active = bi == b;
        }
        if (!__any_sync(0xffffffffu, active)) continue;
        int4 q = make_int4(0, 0, 0, 0);
        if (active)
            q = make_int4(P_.vox[3 * (int64_t)i], P_.vox[3 * (int64_t)i + 1],
                          P_.vox[3 * (int64_t)i + 2], P_.home[i]);
        int d, o;
        psh::warp_exact_window(P_, ctr, q, active, sD, probe, d, o);
        if (active) {
            P_.bucket_id[i] = d;
            P_.bucket_offset[i] = o;
        }
    }
}

__global__ void __launch_bounds__(1024) psh_exact_finish_kernel(psh::Params P_) {
    __shared__ int s_warp[32];
    __shared__ int s_carry;
    const int W = P_.K + 1;
    const int nslots = P_.nbatch * W;
    const int n = (int)dyn_n(P_.n, P_.n_dev);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int s0 = 0; s0 < nslots; s0 += 1024) {
        const int s = s0 + tid;
        const int v = s < nslots ? P_.counts[s] : 0;
        const int incl = warp_incl_scan(v);
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) s_warp[lane] = warp_incl_scan(s_warp[lane]);
        __syncthreads();
        const int excl = s_carry + (warp ? s_warp[warp - 1] : 0) + incl - v;
        if (s < nslots) P_.base[s] = excl;
        __syncthreads();
        if (tid == 0) s_carry += s_warp[31];
        __syncthreads();
    }
    for (int i = tid; i < n; i += 1024) {
        const int b = P_.batch ? P_.batch[i] : 0;
        if (b < 0 || b >= P_.nbatch) continue;
        P_.dest[i] = P_.base[(int64_t)b * W + P_.bucket_id[i]] + P_.bucket_offset[i];
    }
    if (tid == 0) {
        P_.info[0] = 0;
        P_.info[1] = 2;
    }
}

namespace {
constexpr int kMaxGrid = 4096;    // per-CTA partials reserved in the fused workspace

// Launch the cooperative kernel for prepared params (p.n, p.nbatch, p.K set).
// info4 (nullable): the caller's 4 status words, zeroed with the barrier word
int launch_psh(psh::Params& p, bool fused, cudaStream_t st, int32_t* info4 = nullptr) {
    const int K = p.K, nbatch = p.nbatch;
    const int nbins = nbatch > 1 ? std::max(K + 1, nbatch) : K + 1;
    const bool small = p.n < psh::kSmallTileMaxN;
    const int stride = (nbins + 1) & ~1;
    const size_t hist_bytes = (size_t)psh::kWarps * stride * sizeof(uint16_t);
    const size_t base_bytes = (size_t)4 * nbatch * (K + 1);
    p.base_in_smem = hist_bytes + base_bytes <= 200 * 1024 ? 1 : 0;
    const size_t smem = hist_bytes + (p.base_in_smem ? base_bytes : 0);
    void (*kern)(const psh::Params) =
        fused ? (small ? psh::psh_kernel<psh::kPerLaneSmall, true> : psh::psh_kernel<psh::kPerLaneLarge, true>)
              : (small ? psh::psh_kernel<psh::kPerLaneSmall, false> : psh::psh_kernel<psh::kPerLaneLarge, false>);
    static int attr_smem[4] = {0, 0, 0, 0};
    int& at = attr_smem[2 * fused + small];
    if ((int)smem > 48 * 1024 && (int)smem > at) {
        F3D_CUDA_TRY(cudaFuncSetAttribute((const void*)kern,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        at = (int)smem;
    }
    int per_sm = 0;
    F3D_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, psh::kThreads, smem));
    if (per_sm < 1) return F3D_ERR_CONFIG;
    int grid = std::min(per_sm * f3d_num_sms(), p.max_tiles);
    // Phase B needs nbatch*(K+1) column-warps; more CTAs than tiles only help it.
    const int col_ctas = cdiv((int64_t)nbatch * (K + 1), psh::kWarps * 2);
    grid = std::max(grid, std::min(col_ctas, per_sm * f3d_num_sms()));
    grid = std::max(grid, 1);
    if (fused) grid = std::min(grid, kMaxGrid);
    // a kernel, not a memset node (which may queue behind copy-engine traffic)
    F3D_CUDA_TRY(f3d_zero_i32x2((int32_t*)p.bar, 1, info4, 4, st));
    void* args[] = {(void*)&p};
    F3D_CUDA_TRY(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(psh::kThreads), args,
                                             smem, st));
    return F3D_OK;
}
}  // namespace

extern "C" int f3d_psh_assign(const int32_t* vox32, const int32_t* home, const int32_t* batch,
                              int64_t n, int32_t nbatch, int32_t K, int32_t S, int kind,
                              int64_t S_div, int bits, int strict,
                              const int8_t* probe_offsets_host, int32_t P, int32_t max_sweeps,
                              int32_t* bucket_id, int32_t* bucket_offset, int32_t* counts,
                              int32_t* base, int32_t* dest, int32_t* info_out, void* ws,
                              size_t ws_bytes, const int32_t* n_dev, void* stream) {
    if (n <= 0) return F3D_ERR_EMPTY;
    if (n >= INT_MAX / 2 || K < 1 || S < 1 || nbatch < 1 || P < 0 || P > psh::kMaxProbes ||
        bits < 1 || bits > 21 || S_div < 1 || kind < 0 || kind > 3)
        return F3D_ERR_CONFIG;
    if (n_dev && nbatch > 1) return F3D_ERR_CONFIG;
    if (max_sweeps < 1) max_sweeps = 1;
    if (max_sweeps > psh::kMaxSweepsCap) max_sweeps = psh::kMaxSweepsCap;
    const psh::WsLayout L = psh::layout(n, nbatch, K, max_sweeps);
    if (ws_bytes < L.total) return F3D_ERR_CONFIG;
    cudaStream_t st = (cudaStream_t)stream;
    char* w = (char*)ws;

    psh::Params p{};
    p.vox = vox32;
    p.home = home;
    p.batch = nbatch > 1 ? batch : nullptr;
    p.n = (int)n;
    p.n_dev = n_dev;
    p.nbatch = nbatch;
    p.K = K;
    p.S = S;
    p.P = P;
    p.max_sweeps = max_sweeps;
    p.hp = hash_params(kind, K, S_div, bits, strict);
    p.vmax = (1 << bits) - 1;
    for (int i = 0; i < 3 * P; ++i) p.probe[i] = probe_offsets_host[i];
    p.bucket_id = bucket_id;
    p.bucket_offset = bucket_offset;
    p.counts = counts;
    p.base = base;
    p.dest = dest;
    p.info = info_out;
    p.pk = (int4*)(w + L.pk);
    p.D = (int32_t*)(w + L.D);
    p.off = (int32_t*)(w + L.off);
    p.orig = (int32_t*)(w + L.orig);
    p.T0 = (int32_t*)(w + L.T0);
    p.T1 = (int32_t*)(w + L.T1);
    p.hist = (int32_t*)(w + L.hist);
    p.tile_p0 = (int32_t*)(w + L.tile_p0);
    p.tile_b = (int32_t*)(w + L.tile_b);
    p.btile = (int32_t*)(w + L.btile);
    p.bstart = (int32_t*)(w + L.bstart);
    p.flags = (int32_t*)(w + L.flags);
    p.bar = (unsigned*)(w + L.bar);
    const bool small = n < psh::kSmallTileMaxN;
    const int tile = small ? psh::TileC<psh::kPerLaneSmall>::kTile
                           : psh::TileC<psh::kPerLaneLarge>::kTile;
    p.max_tiles = (int)(n / tile + nbatch + 1);

    const int nbins = nbatch > 1 ? std::max(K + 1, nbatch) : K + 1;
    if (nbins > psh::kMaxBins) {
        F3D_CUDA_TRY(f3d_zero_i32(info_out, 4, st));
        psh_warp_exact_kernel<<<nbatch, 32, 0, st>>>(p);
        F3D_LAUNCH_CHECK();
        psh_exact_finish_kernel<<<1, 1024, 0, st>>>(p);
        F3D_LAUNCH_CHECK();
        return F3D_OK;
    }
    return launch_psh(p, false, st, info_out);
}

// ---------------------------------------------------------------------------
// Voxelize + remap + range statistics + home hash + PSH in ONE cooperative
// launch (single batch; the backbone's per-stage bucketing):
//   bw/geometry.py:69-72 -> bw/hashing.py:128-149 -> bw/hashing.py:60-125 ->
//   bw/bucketing.py:275-320 (+ compute_bucket_base, dest_index).
// The coordinates are read twice (per-axis extrema, then the hash in the
// first sweep); stats gets the 7 range words f3d_voxel_hash produces.
static psh::WsLayout coords_layout(int64_t n, int32_t K, int max_sweeps, size_t* part_off) {
    psh::WsLayout L = psh::layout(n, 1, K, max_sweeps);
    *part_off = L.total;
    L.total = psh::align256(L.total + 8 * sizeof(long long) * kMaxGrid);
    return L;
}

extern "C" size_t f3d_psh_coords_workspace_size(int64_t n, int32_t K) {
    size_t po;
    return coords_layout(n, K, psh::kMaxSweepsCap, &po).total;
}

extern "C" int f3d_psh_assign_coords(const double* coords, int64_t n,
                                     const double* origin3_host, double voxel_size, int kind,
                                     int32_t K, int32_t S, int64_t S_div, int bits, int strict,
                                     const int8_t* probe_offsets_host, int32_t P,
                                     int32_t max_sweeps, int32_t* bucket_id,
                                     int32_t* bucket_offset, int32_t* counts, int32_t* base,
                                     int32_t* dest, int32_t* info_out, int64_t* stats_out,
                                     void* ws, size_t ws_bytes, const int32_t* n_dev,
                                     void* stream) {
    if (n <= 0) return F3D_ERR_EMPTY;
    if (n >= INT_MAX / 2 || K < 1 || S < 1 || P < 0 || P > psh::kMaxProbes || bits < 1 ||
        bits > 21 || S_div < 1 || kind < 0 || kind > 3 || !(voxel_size > 0) ||
        K + 1 > psh::kMaxBins)
        return F3D_ERR_CONFIG;
    if (max_sweeps < 1) max_sweeps = 1;
    if (max_sweeps > psh::kMaxSweepsCap) max_sweeps = psh::kMaxSweepsCap;
    size_t part_off;
    const psh::WsLayout L = coords_layout(n, K, max_sweeps, &part_off);
    if (ws_bytes < L.total) return F3D_ERR_CONFIG;
    char* w = (char*)ws;
    psh::Params p{};
    p.coords = coords;
    for (int a = 0; a < 3; ++a) p.org[a] = origin3_host[a];
    p.vs = voxel_size;
    p.stats = stats_out;
    p.part = (long long*)(w + part_off);
    p.n = (int)n;
    p.n_dev = n_dev;
    p.nbatch = 1;
    p.K = K;
    p.S = S;
    p.P = P;
    p.max_sweeps = max_sweeps;
    p.hp = hash_params(kind, K, S_div, bits, strict);
    p.vmax = (1 << bits) - 1;
    for (int i = 0; i < 3 * P; ++i) p.probe[i] = probe_offsets_host[i];
    p.bucket_id = bucket_id;
    p.bucket_offset = bucket_offset;
    p.counts = counts;
    p.base = base;
    p.dest = dest;
    p.info = info_out;
    p.pk = (int4*)(w + L.pk);
    p.D = (int32_t*)(w + L.D);
    p.off = (int32_t*)(w + L.off);
    p.orig = (int32_t*)(w + L.orig);
    p.T0 = (int32_t*)(w + L.T0);
    p.T1 = (int32_t*)(w + L.T1);
    p.hist = (int32_t*)(w + L.hist);
    p.flags = (int32_t*)(w + L.flags);
    p.bar = (unsigned*)(w + L.bar);
    const bool small = n < psh::kSmallTileMaxN;
    const int tile = small ? psh::TileC<psh::kPerLaneSmall>::kTile
                           : psh::TileC<psh::kPerLaneLarge>::kTile;
    p.max_tiles = (int)(n / tile + 2);
    return launch_psh(p, true, (cudaStream_t)stream);
}
