// Voxelize, per-batch remap, range statistics and bucket hash (HBM-bound).
//
// bw/geometry.py:69-72   voxelize: floor((c - origin) / size), IEEE f64 ops
// bw/hashing.py:128-149  remap_nonnegative: subtract the per-batch axis minimum
// bw/hashing.py:60-125   _check_range + morton_encode + hash_bucket
#include <climits>

#include <algorithm>

#include "f3d_common.cuh"

namespace f3d {
namespace hashk {

constexpr int kThreads = 256;

struct Origin {
    double o[3];
};

// floor((c - o) / vs) with no contraction: __dsub_rn then the rounded
// division (vox_floor_inv: reciprocal multiply, exact division near integers).
__device__ __forceinline__ long long vox1(double c, double o, double vs, double inv) {
    return vox_floor_inv(c, o, vs, inv);
}

__device__ __forceinline__ void warp_min_max_atomic(long long v, long long* mn, long long* mx) {
    long long a = v, b = v;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    // read before the atomic: once the running extremum has settled almost no
    // warp improves it, so the per-address atomic traffic (one L2 slice for
    // the whole grid) collapses to a few hundred operations
    if ((threadIdx.x & 31) == 0) {
        if (mn && a < *(volatile long long*)mn) atomicMin(mn, a);
        if (mx && b > *(volatile long long*)mx) atomicMax(mx, b);
    }
}

// Block-level aggregation of up to 8 64-bit extrema (kMin of them minima):
// warp shuffles, then shared-memory atomics, then one filtered global atomic
// per block and value.  Every thread of the block must call it.
template <int N, int kMin>
__device__ __forceinline__ void block_extrema_atomic(const long long (&v)[N], int64_t* const (&dst)[N]) {
    __shared__ long long sh[N];
    if (threadIdx.x < N) sh[threadIdx.x] = threadIdx.x < kMin ? LLONG_MAX : LLONG_MIN;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < N; ++k) {
        long long a = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long b = __shfl_xor_sync(0xffffffffu, a, o);
            a = k < kMin ? min(a, b) : max(a, b);
        }
        if ((threadIdx.x & 31) == 0) {
            if (k < kMin) atomicMin(&sh[k], a);
            else atomicMax(&sh[k], a);
        }
    }
    __syncthreads();
    if (threadIdx.x < N && dst[threadIdx.x]) {
        const int k = threadIdx.x;
        const long long a = sh[k];
        long long* p = (long long*)dst[k];
        if (k < kMin) {
            if (a < *(volatile long long*)p) atomicMin(p, a);
        } else if (a > *(volatile long long*)p) {
            atomicMax(p, a);
        }
    }
}

// per-(batch, axis) minimum of one point per lane: warp-reduced when every
// lane holds the same batch (sorted / contiguous batches), else per lane
__device__ __forceinline__ void batch_min_atomic(const long long (&v)[3], int b, bool ok,
                                                 int64_t* ws_min) {
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    const int b0 = __shfl_sync(0xffffffffu, b, __ffs(act | 1u) - 1);
    const bool uniform = __all_sync(0xffffffffu, !ok || b == b0);
    if (uniform) {
        if (act == 0u) return;
        for (int a = 0; a < 3; ++a)
            warp_min_max_atomic(ok ? v[a] : LLONG_MAX, (long long*)ws_min + 3 * b0 + a, nullptr);
    } else if (ok) {
        for (int a = 0; a < 3; ++a) {
            long long* p = (long long*)ws_min + 3 * b + a;
            if (v[a] < *(volatile long long*)p) atomicMin(p, v[a]);
        }
    }
}

__global__ void init_stats_kernel(int64_t* stats, int64_t* ws_min, int nmin) {
    f3d::pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (stats && i < 7) stats[i] = (i < 3) ? LLONG_MAX : LLONG_MIN;
    if (ws_min && i < nmin) ws_min[i] = LLONG_MAX;
}

__global__ void voxelize_kernel(const double* __restrict__ coords, int64_t n, Origin org,
                                double vs, int64_t* __restrict__ out) {
    const int64_t pt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // one point per thread
    if (pt >= n) return;
    const double inv = __drcp_rn(vs);
#pragma unroll
    for (int a = 0; a < 3; ++a) out[3 * pt + a] = vox1(coords[3 * pt + a], org.o[a], vs, inv);
}

// per-(batch, axis) minimum; batch == null means one batch.  Grid-stride
// (a capped grid): one block-level atomic per axis per block for one batch.
__global__ void batch_min_kernel(const int64_t* __restrict__ vox, const int32_t* __restrict__ batch,
                                 int64_t n, int nbatch, int64_t* ws_min) {
    const bool single = !batch || nbatch == 1;
    long long acc[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX};
    const int64_t step = (int64_t)gridDim.x * blockDim.x;
    const int64_t n_it = (n + step - 1) / step * step;     // warp-uniform trip count
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_it; i += step) {
        const bool ok = i < n;
        long long v[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX};
        int b = 0;
        if (ok) {
            v[0] = vox[3 * i];
            v[1] = vox[3 * i + 1];
            v[2] = vox[3 * i + 2];
            if (batch) b = batch[i];
        }
        if (single) {
#pragma unroll
            for (int a = 0; a < 3; ++a) acc[a] = min(acc[a], v[a]);
        } else {
            batch_min_atomic(v, b, ok && b >= 0 && b < nbatch, ws_min);
        }
    }
    if (single) {
        int64_t* const dst[3] = {ws_min, ws_min + 1, ws_min + 2};
        block_extrema_atomic<3, 3>(acc, dst);
    }
}

__global__ void remap_kernel(const int64_t* __restrict__ vox, const int32_t* __restrict__ batch,
                             int64_t n, int nbatch, const int64_t* __restrict__ ws_min,
                             int64_t* __restrict__ out) {
    // one thread per point (a 64-bit divide per component dominated before)
    const int64_t pt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pt >= n) return;
    int b = (batch && nbatch > 1) ? batch[pt] : 0;
    if (b < 0 || b >= nbatch) b = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) out[3 * pt + a] = vox[3 * pt + a] - ws_min[3 * b + a];
}

struct HashArgs {
    HashParams hp;
    int want_quot;
};

// Home hash of one (remapped) voxel; range statistics accumulated in acc:
// [min x, y, z, max x, y, z, max quotient].
__device__ __forceinline__ void hash_one(long long x, long long y, long long z, int64_t i,
                                         const HashArgs& ha, int32_t* home, int32_t* vox32,
                                         bool valid, long long (&acc)[7]) {
    if (!valid) return;
    const long long lim = 1ll << ha.hp.bits;
    const bool in = x >= 0 && y >= 0 && z >= 0 && x < lim && y < lim && z < lim;
    int h = 0;
    if (in) {
        int64_t key;
        if (ha.hp.kind <= XOR_DIV) key = x ^ y ^ z;
        else key = morton3(x, y, z);
        if (ha.hp.kind == XOR_DIV || ha.hp.kind == ZORDER_DIV) {
            key = (key < 0x7FFFFFFFll && ha.hp.S_div < 0x7FFFFFFFll)
                      ? (int64_t)ha.hp.fdiv.div((uint32_t)key)
                      : key / ha.hp.S_div;
            acc[6] = max(acc[6], (long long)key);
        }
        h = key < 0x7FFFFFFFll ? (int)ha.hp.fk.mod((uint32_t)key) : (int)(key % ha.hp.K);
    }
    home[i] = h;
    if (vox32) {
        vox32[3 * i] = (int)x;
        vox32[3 * i + 1] = (int)y;
        vox32[3 * i + 2] = (int)z;
    }
    acc[0] = min(acc[0], x);
    acc[1] = min(acc[1], y);
    acc[2] = min(acc[2], z);
    acc[3] = max(acc[3], x);
    acc[4] = max(acc[4], y);
    acc[5] = max(acc[5], z);
}

// one global atomic per statistic per block (filtered by the current value)
__device__ __forceinline__ void flush_stats(const long long (&acc)[7], const HashArgs& ha,
                                            int64_t* stats) {
    if (!stats) return;
    int64_t* const dst[7] = {stats, stats + 1, stats + 2, stats + 3, stats + 4, stats + 5,
                             ha.want_quot ? stats + 6 : nullptr};
    block_extrema_atomic<7, 3>(acc, dst);
}

#define F3D_STATS_INIT {LLONG_MAX, LLONG_MAX, LLONG_MAX, LLONG_MIN, LLONG_MIN, LLONG_MIN, LLONG_MIN}

__global__ void hash_kernel(const int64_t* __restrict__ vox, int64_t n, HashArgs ha,
                            int32_t* __restrict__ home, int32_t* __restrict__ vox32,
                            int64_t* stats) {
    long long acc[7] = F3D_STATS_INIT;
    const int64_t step = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += step)
        hash_one(vox[3 * i], vox[3 * i + 1], vox[3 * i + 2], i, ha, home, vox32, true, acc);
    flush_stats(acc, ha, stats);
}

__global__ void morton_kernel(const int64_t* __restrict__ vox, int64_t n, int bits,
                              int64_t* __restrict__ codes, int64_t* stats) {
    long long acc[7] = F3D_STATS_INIT;
    const uint64_t m = (1ull << bits) - 1;
    const int64_t step = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += step) {
        const long long x = vox[3 * i], y = vox[3 * i + 1], z = vox[3 * i + 2];
        codes[i] = morton3((int64_t)(x & m), (int64_t)(y & m), (int64_t)(z & m));
        acc[0] = min(acc[0], x);
        acc[1] = min(acc[1], y);
        acc[2] = min(acc[2], z);
        acc[3] = max(acc[3], x);
        acc[4] = max(acc[4], y);
        acc[5] = max(acc[5], z);
    }
    int64_t* const dst[7] = {stats, stats + 1, stats + 2, stats + 3, stats + 4, stats + 5, nullptr};
    block_extrema_atomic<7, 3>(acc, dst);
}

// Fused pass 1: voxelize + per-batch axis minimum (voxels are not stored).
__global__ void fused_min_kernel(const double* __restrict__ coords,
                                 const int32_t* __restrict__ batch, int64_t n,
                                 const int32_t* n_dev, int nbatch, Origin org, double vs,
                                 int64_t* ws_min) {
    f3d::pdl_wait();
    const int64_t nn = dyn_n(n, n_dev);
    const bool single = !batch || nbatch == 1;
    const double inv = __drcp_rn(vs);
    long long acc[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX};
    const int64_t step = (int64_t)gridDim.x * blockDim.x;
    const int64_t n_it = (nn + step - 1) / step * step;    // warp-uniform trip count
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_it; i += step) {
        const bool ok = i < nn;
        long long v[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX};
        int b = 0;
        if (ok) {
            for (int a = 0; a < 3; ++a) v[a] = vox1(coords[3 * i + a], org.o[a], vs, inv);
            if (batch) b = batch[i];
        }
        if (single) {
#pragma unroll
            for (int a = 0; a < 3; ++a) acc[a] = min(acc[a], v[a]);
        } else {
            batch_min_atomic(v, b, ok && b >= 0 && b < nbatch, ws_min);
        }
    }
    if (single) {
        int64_t* const dst[3] = {ws_min, ws_min + 1, ws_min + 2};
        block_extrema_atomic<3, 3>(acc, dst);
    }
}

// Fused pass 2: re-voxelize, remap by the batch minimum, range stats, hash.
__global__ void fused_hash_kernel(const double* __restrict__ coords,
                                  const int32_t* __restrict__ batch, int64_t n,
                                  const int32_t* n_dev, int nbatch, Origin org, double vs,
                                  const int64_t* __restrict__ ws_min, HashArgs ha,
                                  int32_t* __restrict__ home, int32_t* __restrict__ vox32,
                                  int64_t* stats) {
    f3d::pdl_wait();
    const int64_t nn = dyn_n(n, n_dev);
    long long acc[7] = F3D_STATS_INIT;
    const double inv = __drcp_rn(vs);
    const int64_t step = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += step) {
        int b = (batch && nbatch > 1) ? batch[i] : 0;
        if (b < 0 || b >= nbatch) b = 0;
        long long v[3];
        for (int a = 0; a < 3; ++a) v[a] = vox1(coords[3 * i + a], org.o[a], vs, inv) - ws_min[3 * b + a];
        hash_one(v[0], v[1], v[2], i, ha, home, vox32, true, acc);
    }
    flush_stats(acc, ha, stats);
}

}  // namespace hashk
}  // namespace f3d

using namespace f3d;
using namespace f3d::hashk;

static inline int nblk(int64_t work) { return (int)((work + kThreads - 1) / kThreads); }
// grid-stride kernels with per-block statistics: at most 8 blocks per SM
static inline int nblk_capped(int64_t work) {
    return std::max(1, std::min(nblk(work), 8 * f3d_num_sms()));
}

extern "C" int f3d_voxelize(const double* coords, int64_t n, const double* origin3_host,
                            double voxel_size, int64_t* vox_out, void* stream) {
    if (n < 0 || !(voxel_size > 0)) return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    Origin o{{origin3_host[0], origin3_host[1], origin3_host[2]}};
    voxelize_kernel<<<nblk(n), kThreads, 0, (cudaStream_t)stream>>>(coords, n, o, voxel_size,
                                                                       vox_out);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

extern "C" int f3d_remap_nonnegative(const int64_t* vox, const int32_t* batch, int64_t n,
                                     int32_t nbatch, int64_t* vox_out, int64_t* ws,
                                     void* stream) {
    if (n < 0 || nbatch < 1) return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    cudaStream_t st = (cudaStream_t)stream;
    init_stats_kernel<<<nblk(3 * nbatch + 7), kThreads, 0, st>>>(nullptr, ws, 3 * nbatch);
    batch_min_kernel<<<nblk_capped(n), kThreads, 0, st>>>(vox, batch, n, nbatch, ws);
    remap_kernel<<<nblk(n), kThreads, 0, st>>>(vox, batch, n, nbatch, ws, vox_out);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

static bool bad_hash_cfg(int kind, int32_t K, int64_t S_div, int bits) {
    return kind < 0 || kind > 3 || K < 1 || S_div < 1 || bits < 1 || bits > 21;
}

extern "C" int f3d_hash_bucket(const int64_t* vox, int64_t n, int kind, int32_t K,
                               int64_t S_div, int bits, int32_t* home_out, int32_t* vox32_out,
                               int64_t* stats_out, void* stream) {
    if (n < 0 || bad_hash_cfg(kind, K, S_div, bits)) return F3D_ERR_CONFIG;
    cudaStream_t st = (cudaStream_t)stream;
    init_stats_kernel<<<1, 32, 0, st>>>(stats_out, nullptr, 0);
    if (n > 0) {
        HashArgs ha{hash_params(kind, K, S_div, bits, 0), 1};
        hash_kernel<<<nblk_capped(n), kThreads, 0, st>>>(vox, n, ha, home_out, vox32_out, stats_out);
    }
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

extern "C" int f3d_morton_encode(const int64_t* vox, int64_t n, int bits, int64_t* codes_out,
                                 int64_t* stats_out, void* stream) {
    if (n < 0 || bits < 1 || bits > 21) return F3D_ERR_CONFIG;
    cudaStream_t st = (cudaStream_t)stream;
    init_stats_kernel<<<1, 32, 0, st>>>(stats_out, nullptr, 0);
    if (n > 0) morton_kernel<<<nblk_capped(n), kThreads, 0, st>>>(vox, n, bits, codes_out, stats_out);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

extern "C" int f3d_voxel_hash(const double* coords, const int32_t* batch, int64_t n,
                              int32_t nbatch, const double* origin3_host, double voxel_size,
                              int kind, int32_t K, int64_t S_div, int bits, int32_t* vox32_out,
                              int32_t* home_out, int64_t* stats_out, int64_t* ws,
                              const int32_t* n_dev, void* stream) {
    if (n < 0 || nbatch < 1 || !(voxel_size > 0) || bad_hash_cfg(kind, K, S_div, bits))
        return F3D_ERR_CONFIG;
    if (n_dev && nbatch > 1) return F3D_ERR_CONFIG;
    cudaStream_t st = (cudaStream_t)stream;
    Origin o{{origin3_host[0], origin3_host[1], origin3_host[2]}};
    F3D_CUDA_TRY(f3d_launch(init_stats_kernel, dim3(nblk(3 * nbatch + 7)), dim3(kThreads), 0, st,
                            stats_out, ws, 3 * nbatch));
    if (n > 0) {
        F3D_CUDA_TRY(f3d_launch(fused_min_kernel, dim3(nblk_capped(n)), dim3(kThreads), 0, st,
                                coords, batch, n, n_dev, nbatch, o, voxel_size, ws));
        HashArgs ha{hash_params(kind, K, S_div, bits, 0), 1};
        F3D_CUDA_TRY(f3d_launch(fused_hash_kernel, dim3(nblk_capped(n)), dim3(kThreads), 0, st,
                                coords, batch, n, n_dev, nbatch, o, voxel_size, (const int64_t*)ws,
                                ha, home_out, vox32_out, stats_out));
    }
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}
