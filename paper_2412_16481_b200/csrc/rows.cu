// Row scatter / gather (bw/bucketing.py:385-401) and assignment validation
// (bw/bucketing.py:116-145).  HBM-bound: 16-byte vectors, one warp-row.
#include <cuda_bf16.h>

#include <climits>

#include "f3d_common.cuh"

namespace f3d {
namespace rows {

constexpr int kThreads = 256;

// Each thread moves one 16 B (or 4 B) chunk; consecutive threads cover a row
// contiguously so both the read and the write side are coalesced per row.
template <typename V, bool kScatter>
__global__ void move_rows_kernel(const V* __restrict__ src, const int32_t* __restrict__ idx,
                                 int64_t n, const int32_t* n_dev, int64_t vec_per_row,
                                 V* __restrict__ dst) {
    f3d::pdl_wait();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t tot = dyn_n(n, n_dev) * vec_per_row;
    if (t >= tot) return;
    const int64_t r = t / vec_per_row;
    const int64_t k = t - r * vec_per_row;
    const int64_t j = __ldg(idx + r);
    if (kScatter) dst[j * vec_per_row + k] = src[r * vec_per_row + k];
    else dst[r * vec_per_row + k] = src[j * vec_per_row + k];
}

template <bool kScatter>
int move_rows(const void* src, const int32_t* idx, int64_t n, const int32_t* n_dev,
              int64_t row_bytes, void* dst, cudaStream_t st) {
    if (n < 0 || row_bytes <= 0 || (row_bytes & 3)) return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    const bool v16 = ((row_bytes & 15) == 0) && ((uintptr_t)src & 15) == 0 &&
                     ((uintptr_t)dst & 15) == 0;
    if (v16) {
        const int64_t vpr = row_bytes / 16;
        const int64_t tot = n * vpr;
        F3D_CUDA_TRY(f3d_launch(move_rows_kernel<int4, kScatter>,
                                dim3((unsigned)((tot + kThreads - 1) / kThreads)), dim3(kThreads), 0,
                                st, (const int4*)src, idx, n, n_dev, vpr, (int4*)dst));
    } else {
        const int64_t vpr = row_bytes / 4;
        const int64_t tot = n * vpr;
        F3D_CUDA_TRY(f3d_launch(move_rows_kernel<int, kScatter>,
                                dim3((unsigned)((tot + kThreads - 1) / kThreads)), dim3(kThreads), 0,
                                st, (const int*)src, idx, n, n_dev, vpr, (int*)dst));
    }
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

// Scatter of bf16 rows into fp32 rows (the backbone's feature upload is bf16,
// the residual stream fp32): one thread per 8 columns, 16-byte in, 2x16 out.
__global__ void scatter_bf16_f32_kernel(const uint4* __restrict__ src, int64_t ld_src8,
                                        const int32_t* __restrict__ dest, int64_t n,
                                        const int32_t* n_dev, int d8, float4* __restrict__ dst,
                                        int64_t ld_dst4) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= dyn_n(n, n_dev) * d8) return;
    const int64_t r = t / d8;
    const int k = (int)(t - r * d8);
    const uint4 w = src[r * ld_src8 + k];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
    const float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
    const float2 c = __bfloat1622float2(h[2]), e = __bfloat1622float2(h[3]);
    float4* o = dst + (int64_t)__ldg(dest + r) * ld_dst4 + 2 * k;
    o[0] = make_float4(a.x, a.y, b.x, b.y);
    o[1] = make_float4(c.x, c.y, e.x, e.y);
}

// ------------------------------------------------------------- validate

enum {
    V_SUM = 1, V_CAP = 2, V_NEG = 4, V_BASE = 8, V_ID = 16, V_OFF = 32, V_BIJ = 64
};

// Slot checks: capacity, negativity, exclusive-scan consistency, total.
__global__ void validate_slots_kernel(const int32_t* __restrict__ counts,
                                      const int32_t* __restrict__ base, int64_t nslots, int K,
                                      int S, int64_t n, int32_t* flags) {
    // single block: sequential-in-chunks scan check
    __shared__ long long part[kThreads];
    const int tid = threadIdx.x;
    const int64_t per = (nslots + kThreads - 1) / kThreads;
    const int64_t a0 = min((int64_t)tid * per, nslots), a1 = min(a0 + per, nslots);
    long long s = 0;
    int f = 0;
    for (int64_t i = a0; i < a1; ++i) {
        const int c = counts[i];
        if (c < 0) f |= V_NEG;
        if ((i % (K + 1)) != K && c > S) f |= V_CAP;
        s += c;
    }
    part[tid] = s;
    __syncthreads();
    if (tid == 0) {
        long long run = 0;
        for (int w = 0; w < kThreads; ++w) {
            const long long v = part[w];
            part[w] = run;
            run += v;
        }
        if (run != n) f |= V_SUM;
    }
    __syncthreads();
    long long run = part[tid];
    for (int64_t i = a0; i < a1; ++i) {
        if (base[i] != run) f |= V_BASE;
        run += counts[i];
    }
    if (f) atomicOr(flags, f);
}

__global__ void validate_points_kernel(const int32_t* __restrict__ id,
                                       const int32_t* __restrict__ off,
                                       const int32_t* __restrict__ batch,
                                       const int32_t* __restrict__ counts,
                                       const int32_t* __restrict__ base, int64_t n, int nbatch,
                                       int K, int32_t* seen, int32_t* flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int f = 0;
    if (i < n) {
        const int d = id[i];
        const int b = (batch && nbatch > 1) ? batch[i] : 0;
        if (d < 0 || d > K || b < 0 || b >= nbatch) {
            f |= V_ID;
        } else {
            const int64_t slot = (int64_t)b * (K + 1) + d;
            const int o = off[i];
            if (o < 0 || o >= counts[slot]) {
                f |= V_OFF;
            } else {
                const int64_t dst = (int64_t)base[slot] + o;
                if (dst < 0 || dst >= n) f |= V_BIJ;
                else atomicAdd(seen + dst, 1);
            }
        }
    }
    f = __reduce_or_sync(0xffffffffu, f);
    if (f && (threadIdx.x & 31) == 0) atomicOr(flags, f);
}

__global__ void validate_seen_kernel(const int32_t* __restrict__ seen, int64_t n, int32_t* flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int f = (i < n && seen[i] != 1) ? V_BIJ : 0;
    f = __reduce_or_sync(0xffffffffu, f);
    if (f && (threadIdx.x & 31) == 0) atomicOr(flags, f);
}

}  // namespace rows
}  // namespace f3d

using namespace f3d;

extern "C" int f3d_scatter_rows(const void* src, const int32_t* dest, int64_t n,
                                int64_t row_bytes, void* dst, const int32_t* n_dev, void* stream) {
    return rows::move_rows<true>(src, dest, n, n_dev, row_bytes, dst, (cudaStream_t)stream);
}

extern "C" int f3d_scatter_rows_bf16_f32(const void* src, int64_t ld_src, const int32_t* dest,
                                         int64_t n, int d, void* dst, int64_t ld_dst,
                                         const int32_t* n_dev, void* stream) {
    if (n < 0 || d < 8 || (d & 7) || (ld_src & 7) || (ld_dst & 3) ||
        (((uintptr_t)src | (uintptr_t)dst) & 15))
        return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    const int64_t tot = n * (d / 8);
    rows::scatter_bf16_f32_kernel<<<(unsigned)((tot + rows::kThreads - 1) / rows::kThreads),
                                    rows::kThreads, 0, (cudaStream_t)stream>>>(
        (const uint4*)src, ld_src / 8, dest, n, n_dev, d / 8, (float4*)dst, ld_dst / 4);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

extern "C" int f3d_gather_rows(const void* src, const int32_t* idx, int64_t n, int64_t row_bytes,
                               void* dst, const int32_t* n_dev, void* stream) {
    return rows::move_rows<false>(src, idx, n, n_dev, row_bytes, dst, (cudaStream_t)stream);
}

extern "C" size_t f3d_validate_workspace_size(int64_t n, int64_t nslots) {
    (void)nslots;
    return (size_t)(n > 0 ? n : 1) * sizeof(int32_t);
}

extern "C" int f3d_validate_assignment(const int32_t* bucket_id, const int32_t* bucket_offset,
                                       const int32_t* batch, const int32_t* counts,
                                       const int32_t* base, int64_t n, int32_t nbatch, int32_t K,
                                       int32_t S, int32_t* flags_out, void* ws, void* stream) {
    if (n < 0 || nbatch < 1 || K < 0) return F3D_ERR_CONFIG;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nslots = (int64_t)nbatch * (K + 1);
    F3D_CUDA_TRY(f3d_zero_i32(flags_out, 1, st));
    rows::validate_slots_kernel<<<1, rows::kThreads, 0, st>>>(counts, base, nslots, K, S, n,
                                                              flags_out);
    if (n > 0) {
        int32_t* seen = (int32_t*)ws;
        F3D_CUDA_TRY(f3d_zero_i32(seen, n, st));
        const unsigned g = (unsigned)((n + rows::kThreads - 1) / rows::kThreads);
        rows::validate_points_kernel<<<g, rows::kThreads, 0, st>>>(
            bucket_id, bucket_offset, batch, counts, base, n, nbatch, K, seen, flags_out);
        rows::validate_seen_kernel<<<g, rows::kThreads, 0, st>>>(seen, n, flags_out);
    }
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}
