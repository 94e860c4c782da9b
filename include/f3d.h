/*
 * libf3d — C ABI of the B200-native Flash3D hot path (sm_100a).
 *
 * Drop-in boundary for the reference package `bucketswin`
 * (/root/reference/pkg/src/bucketswin, cited below as bw/).  Every entry point
 * replaces one reference function (or its numba native sub-boundary) and is
 * bound from Python by paper_2412_16481_b200/_lib.py via ctypes.
 *
 * Conventions:
 *   - plain pointers and sizes only; every array argument is a DEVICE pointer
 *     owned by the caller unless its name ends in `_host`;
 *   - every call takes an explicit cudaStream_t (passed as void*), is
 *     asynchronous and re-entrant per stream; the library allocates nothing;
 *   - scratch memory comes from a *_workspace_size() query + caller buffer;
 *   - int status: F3D_OK or an F3D_ERR_* code that the Python layer maps onto
 *     the reference exception classes (bw/errors.py:9-30).  Data-dependent
 *     errors (range, integrity) are reported through small device-side
 *     status arrays that the caller reads after the stream drains.
 */
#ifndef F3D_H_
#define F3D_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    F3D_OK = 0,
    F3D_ERR_CONFIG = 1,     /* bw/errors.py ConfigError    */
    F3D_ERR_RANGE = 2,      /* bw/errors.py RangeError     */
    F3D_ERR_INTEGRITY = 3,  /* bw/errors.py IntegrityError */
    F3D_ERR_CUDA = 4,       /* CUDA runtime failure        */
    F3D_ERR_EMPTY = 5,      /* bw/errors.py EmptyInputError */
    F3D_ERR_NUMERIC = 6     /* bw/errors.py NumericError   */
};

int f3d_abi_version(void);
/* Human-readable text of the last error raised on this host thread. */
const char *f3d_last_error(void);

/* ------------------------------------------------------------ a1: voxelize
 * Replaces bw/geometry.py:69-72 voxelize(): floor((c - origin) / voxel_size)
 * computed with an IEEE f64 subtract and divide (no FMA, no reciprocal).
 * coords (n,3) f64 -> vox_out (n,3) int64. */
int f3d_voxelize(const double *coords, int64_t n, const double *origin3_host,
                 double voxel_size, int64_t *vox_out, void *stream);

/* ---------------------------------------------------- a2: remap_nonnegative
 * Replaces bw/hashing.py:128-149: subtract the per-batch, per-axis minimum.
 * batch may be NULL (single batch).  ws: nbatch*3 int64 scratch. */
int f3d_remap_nonnegative(const int64_t *vox, const int32_t *batch, int64_t n,
                          int32_t nbatch, int64_t *vox_out, int64_t *ws, void *stream);

/* ------------------------------------------------------- a3: hash_bucket
 * Replaces bw/hashing.py:60-125 (_check_range + morton_encode + hash_bucket)
 * and the numba _hash (bw/_kernels.py:27-38).  kind: 0 xor-mod, 1 xor-div,
 * 2 zorder-mod, 3 zorder-div.  stats_out (device, 7 x int64) receives
 * [min_x, min_y, min_z, max_x, max_y, max_z, max_quotient] so the caller can
 * raise RangeError with the reference's message (axis + value).  vox32_out
 * (nullable) receives the voxels narrowed to int32 for f3d_psh_assign. */
int f3d_hash_bucket(const int64_t *vox, int64_t n, int kind, int32_t K, int64_t S_div,
                    int bits, int32_t *home_out, int32_t *vox32_out, int64_t *stats_out,
                    void *stream);

/* Morton code only (bw/hashing.py:78-98): codes_out (n) int64. */
int f3d_morton_encode(const int64_t *vox, int64_t n, int bits, int64_t *codes_out,
                      int64_t *stats_out, void *stream);

/* ---------------------------------------------- a1-a3 fused (pipeline path)
 * coords -> voxelize -> per-batch min remap -> range stats -> home hash, in
 * two passes over the points.  ws: nbatch*3 int64.  Outputs as above. */
int f3d_voxel_hash(const double *coords, const int32_t *batch, int64_t n, int32_t nbatch,
                   const double *origin3_host, double voxel_size, int kind, int32_t K,
                   int64_t S_div, int bits, int32_t *vox32_out, int32_t *home_out,
                   int64_t *stats_out, int64_t *ws, void *stream);

/* ------------------------------------------------------ a5-a7: PSH assign
 * Replaces bw/bucketing.py:275-320 assign_buckets (and :323-382
 * assign_buckets_two_stage, which the reference proves bit-identical) with
 * its numba sub-boundary bw/_kernels.py:69-90 assign_one_stage.
 * Exact parallel fill-time fixed point in one
 * cooperative launch; bit-identical bucket_id / bucket_offset / counts.
 * Also writes base (exclusive scan of counts, bw/bucketing.py:169-179) and
 * dest = base[batch*(K+1)+id] + offset (bw/bucketing.py:100-101).
 * probe_offsets_host: P x 3 int8 offsets (bw/bucketing.py:51-66), already cut
 * to min(max_probes, len).  info_out (device, 4 x int32): [sweeps,
 * used_sequential_fallback, batch_error, reserved]. */
size_t f3d_psh_workspace_size(int64_t n, int32_t nbatch, int32_t K);
int f3d_psh_assign(const int32_t *vox32, const int32_t *home, const int32_t *batch, int64_t n,
                   int32_t nbatch, int32_t K, int32_t S, int kind, int64_t S_div, int bits,
                   int strict, const int8_t *probe_offsets_host, int32_t P, int32_t max_sweeps,
                   int32_t *bucket_id, int32_t *bucket_offset, int32_t *counts, int32_t *base,
                   int32_t *dest, int32_t *info_out, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------- a7: validate()
 * Replaces BucketAssignment.validate (bw/bucketing.py:116-145).
 * flags_out (device int32) receives a bit set: 1 counts sum != n,
 * 2 regular bucket over S, 4 negative count, 8 base not the exclusive scan,
 * 16 id outside [0,K], 32 offset outside [0,count), 64 not a bijection.
 * ws: f3d_validate_workspace_size(n, nslots) bytes. */
size_t f3d_validate_workspace_size(int64_t n, int64_t nslots);
int f3d_validate_assignment(const int32_t *bucket_id, const int32_t *bucket_offset,
                            const int32_t *batch, const int32_t *counts, const int32_t *base,
                            int64_t n, int32_t nbatch, int32_t K, int32_t S, int32_t *flags_out,
                            void *ws, void *stream);

/* ------------------------------------------------- a8: scatter / gather
 * Replaces bw/bucketing.py:385-401 scatter: dst[dest[i]] = src[i]; and its
 * inverse out = scattered[perm] (pkg/tests/test_stage.py:165).  row_bytes
 * must be a multiple of 4; rows are moved with 16-byte vectors when aligned. */
int f3d_scatter_rows(const void *src, const int32_t *dest, int64_t n, int64_t row_bytes,
                     void *dst, void *stream);
int f3d_gather_rows(const void *src, const int32_t *idx, int64_t n, int64_t row_bytes,
                    void *dst, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* F3D_H_ */
