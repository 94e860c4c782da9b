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
 *     status arrays that the caller reads after the stream drains;
 *   - arguments named n_dev / ntiles_dev / npool_dev (nullable) hold a row
 *     count in device memory: the launch is sized for the host capacity and
 *     processes min(capacity, *count) rows, so a pipeline whose sizes are
 *     data dependent (pooled rows) runs with no host read-back and can be
 *     captured in a CUDA graph.
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
 * two passes over the points.  ws: nbatch*3 int64.  Outputs as above.
 * n_dev (nullable, single batch only): device point count <= n. */
int f3d_voxel_hash(const double *coords, const int32_t *batch, int64_t n, int32_t nbatch,
                   const double *origin3_host, double voxel_size, int kind, int32_t K,
                   int64_t S_div, int bits, int32_t *vox32_out, int32_t *home_out,
                   int64_t *stats_out, int64_t *ws, const int32_t *n_dev, void *stream);

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
 * used_sequential_fallback, batch_error, reserved].  n_dev (nullable, single
 * batch only): device point count <= n; points past it are not touched. */
size_t f3d_psh_workspace_size(int64_t n, int32_t nbatch, int32_t K);
int f3d_psh_assign(const int32_t *vox32, const int32_t *home, const int32_t *batch, int64_t n,
                   int32_t nbatch, int32_t K, int32_t S, int kind, int64_t S_div, int bits,
                   int strict, const int8_t *probe_offsets_host, int32_t P, int32_t max_sweeps,
                   int32_t *bucket_id, int32_t *bucket_offset, int32_t *counts, int32_t *base,
                   int32_t *dest, int32_t *info_out, void *ws, size_t ws_bytes,
                   const int32_t *n_dev, void *stream);

/* Voxelize + per-axis remap + range statistics + home hash + PSH assignment
 * in one cooperative launch, for one batch (the backbone's per-stage
 * bucketing): bw/geometry.py:69-72, bw/hashing.py:60-149,
 * bw/bucketing.py:275-320 and compute_bucket_base (:169-179).  coords: n x 3
 * float64 (device); outputs as f3d_psh_assign, plus stats_out = the 7 range
 * words of f3d_voxel_hash (axis minima / maxima of the remapped voxels, the
 * largest div quotient).  K + 1 <= 12288.  ws: f3d_psh_coords_workspace_size. */
size_t f3d_psh_coords_workspace_size(int64_t n, int32_t K);
int f3d_psh_assign_coords(const double *coords, int64_t n, const double *origin3_host,
                          double voxel_size, int kind, int32_t K, int32_t S, int64_t S_div,
                          int bits, int strict, const int8_t *probe_offsets_host, int32_t P,
                          int32_t max_sweeps, int32_t *bucket_id, int32_t *bucket_offset,
                          int32_t *counts, int32_t *base, int32_t *dest, int32_t *info_out,
                          int64_t *stats_out, void *ws, size_t ws_bytes, const int32_t *n_dev,
                          void *stream);

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
                     void *dst, const int32_t *n_dev, void *stream);
int f3d_gather_rows(const void *src, const int32_t *idx, int64_t n, int64_t row_bytes,
                    void *dst, const int32_t *n_dev, void *stream);
/* Scatter with a dtype change: dst (fp32, row stride ld_dst)[dest[i]] =
 * src (bf16, row stride ld_src)[i]; d % 8 == 0, 16-byte aligned rows. */
int f3d_scatter_rows_bf16_f32(const void *src, int64_t ld_src, const int32_t *dest, int64_t n,
                              int d, void *dst, int64_t ld_dst, const int32_t *n_dev,
                              void *stream);


/* ------------------------------------------ a9-a11: bucket-swin attention
 * Replaces bw/attention.py:188-268 tiled_attention (and the per-scope loop of
 * bw/stage.py:141-156).  One launch covers every scope of a round: scope s is
 * the concatenation of segments j in [scope_seg[s], scope_seg[s]+scope_nseg[s])
 * with physical start seg_start[j] and virtual start seg_vstart[j];
 * scope_len[s] = m_s.  live (nullable, device): [nwork, nlive, max_len] as
 * written by f3d_plan_round; nwork / nlive / max_len are then upper bounds.
 * work: nwork x (scope, q_start) pairs (128-row query tiles, streaming
 * kernel); scope_order: the nlive non-empty scopes, longest first, and
 * max_len = max m_s (whole-scope-resident kernel, chosen when head dim <= 64
 * and the scope's K/V fit in shared memory).  q/k/v are bf16 rows with head h
 * at columns [h*dh, (h+1)*dh) and row strides ld_*; o is bf16 (out_f32 = 0)
 * or f32 with the same layout, written at the fixed rows.  mask (nullable):
 * per-row uint8 validity; 0 = masked (excluded as key, query gives 0), 1 = present,
 * 2 = query only (excluded as key; lets reference_attention take a key set of its
 * own size, bw/attention.py:147-166).
 * starved (nullable): count of rows with no valid key. */
int f3d_bswin_attention(const void *q, const void *k, const void *v, int64_t ld_q,
                        int64_t ld_k, int64_t ld_v, void *o, int64_t ld_o, int out_f32, int H,
                        int dh, const int32_t *scope_seg, const int32_t *scope_nseg,
                        const int32_t *seg_start, const int32_t *seg_vstart,
                        const int32_t *scope_len, const int32_t *work, int nwork,
                        const int32_t *scope_order, int nlive, int max_len, const int32_t *live,
                        const uint8_t *mask, int32_t *starved, void *stream);

/* Same contract on the 5th-generation tensor cores (tcgen05.mma into TMEM,
 * persistent warp-specialised CTAs: TMA loads of in-segment tiles with a
 * cp.async row gather for tiles straddling segments, one elected MMA-issuing
 * lane, softmax warpgroups reading S / writing P with tcgen05.ld / st).  The
 * work list must step q_start by f3d_attention_tc_qstep(dh) (two 128-row Q
 * tiles share each K/V tile).  n_rows: rows of q/k/v (bounds of the TMA
 * tensor maps; 0 disables TMA).  lse (nullable, training): lse[row*ld_lse + h] =
 * log2-domain logsumexp of the row's scaled scores, so P = exp2(s*scale*log2e -
 * lse).  Requires dh % 8 == 0, dh <= 128, 16-byte aligned q/k/v and row strides
 * that are multiples of 8; no mask.  With live (8 words from f3d_plan_round)
 * the CTAs take work items from the counter live[4] (dynamic balance);
 * without it, item i goes to CTA i mod grid. */
int f3d_bswin_attention_tc(const void *q, const void *k, const void *v, int64_t ld_q,
                           int64_t ld_k, int64_t ld_v, void *o, int64_t ld_o, int out_f32, int H,
                           int dh, const int32_t *scope_seg, const int32_t *scope_nseg,
                           const int32_t *seg_start, const int32_t *seg_vstart,
                           const int32_t *scope_len, const int32_t *work, int nwork,
                           const int32_t *live, int64_t n_rows, float *lse, int64_t ld_lse,
                           void *stream);

int f3d_attention_tc_qstep(int dh);

/* Device planner for one round (bw/attention.py:84-139 over the split table
 * of bw/bucketing.py:147-166, built from the PSH counts/base in HBM).
 * The table size nb = K + ceil(counts[K] / S) is read on the device; nb_cap
 * is the host's upper bound and nscopes = ceil(nb_cap / (W*stride)) * stride;
 * segment arrays hold nscopes*W entries (fixed stride W per scope); work
 * holds max_work (scope, q_start) pairs with q_start stepping by qstep
 * (f3d_attention_tc_qstep for the tcgen05 kernel); live receives [nwork,
 * nlive, max_len, status, 0, 0, -, -] (8 words) with status bits 1 (window_w >
 * nb, ConfigError), 2 (nb > nb_cap), 4 (work list truncated); words 4-5 are
 * the tcgen05 attention kernel's dynamic item counter and CTA-done counter
 * (zeroed here, left zeroed by every attention launch: launches sharing one
 * plan must be stream-ordered).  The work list holds every scope's full
 * qstep groups first, then the partial last groups.  off = (t*shift) mod W. */
int f3d_plan_round(const int32_t *counts, const int32_t *base, int K, int S, int nb_cap, int W,
                   int stride, int off, int nscopes, int32_t *scope_seg, int32_t *scope_nseg,
                   int32_t *seg_start, int32_t *seg_vstart, int32_t *scope_len,
                   int32_t *scope_order, int32_t *work, int max_work, int qstep, int32_t *live,
                   void *stream);
/* All rounds of a schedule in one launch: round t (block t) uses rotation
 * (t*shift) mod W and writes its tables round_stride int32 elements after
 * round t-1's (every output pointer is round 0's). */
int f3d_plan_rounds(const int32_t *counts, const int32_t *base, int K, int S, int nb_cap, int W,
                    int stride, int shift, int nrounds, int64_t round_stride, int nscopes,
                    int32_t *scope_seg, int32_t *scope_nseg, int32_t *seg_start,
                    int32_t *seg_vstart, int32_t *scope_len, int32_t *scope_order,
                    int32_t *work, int max_work, int qstep, int32_t *live, void *stream);
/* Device pooling tile table (bw/pooling.py:211-225): tiles of <= cap rows per
 * slot in scatter order; totals receives [ntiles, npooled]. */
int f3d_plan_pool(const int32_t *counts, const int32_t *base, int nslots, int cap, int rho,
                  int32_t *tile_start, int32_t *tile_m, int32_t *tile_out, int32_t *totals,
                  void *stream);

/* ---------------------------------------------- a12: positional encoding
 * bw/attention.py:271-288 (d % 6 == 0).  out_f64: 1 -> double, 0 -> float. */
int f3d_positional_encoding(const double *coords, int64_t n, int d, double base, int out_f64,
                            void *out, int64_t ld, void *stream);
/* Stage form: coords normalised by lo_ext = [lo[3], extent[3]] first
 * (bw/stage.py:129-132).  out_kind: 1 float, 2 double. */
int f3d_stage_pe(const double *coords, int64_t n, int d, double base, const double *lo_ext,
                 int out_kind, void *out, int64_t ld, void *stream);
/* Per-axis bbox: lo_ext[0..2] = min, lo_ext[3..5] = max - min (0 -> 1).
 * ws: 6 * 296 doubles. */
int f3d_coord_bbox(const double *coords, int64_t n, double *ws, double *lo_ext,
                   const int32_t *n_dev, void *stream);

/* ------------------------------------------------------ a13: stage rows
 * Fused residual + LayerNorm (+PE) (bw/stage.py:84-88, 135, 157-158):
 *   if y:   F[r] += y[r] + ybias           (F float or double, y bf16)
 *   if out: out[r] = LN(F[r]) * gain + beta (+ PE(pe_coords[r]))  (population var)
 * The PE term (bw/attention.py:271-288) is computed on the fly from the f64
 * coords, normalised by lo_ext (nullable; bw/stage.py:129-132), when
 * pe_coords is non-null (d % 6 == 0).  out_kind: 0 bf16, 1 float, 2 double. */
int f3d_row_ln(void *F, int f_is_f64, int64_t ldf, const void *y, int64_t ldy,
               const float *ybias, const float *gain, const float *beta,
               const double *pe_coords, const double *lo_ext, double pe_base, void *out,
               int out_kind, int64_t ldo, int64_t n, int d, double eps, void *stream);
/* y = 0.5 x (1 + erf(x / sqrt 2)) in float64 (bw/stage.py:91-92). */
int f3d_gelu_f64(const double *x, int64_t n, double *y, void *stream);
/* u = gelu(u + bias) with the exact erf form (bw/stage.py:91-96), bf16 rows. */
int f3d_bias_gelu(void *u_bf16, int64_t n, int dh, const float *bias, void *stream);

/* ------------------------------------------------ a14-a15: pooling
 * Replaces bw/pooling.py:68-163 build_subbuckets for every <=1024-row tile
 * of every bucket slot (tile_start/tile_m/tile_out: first scattered row, row
 * count and first pooled row of each tile; bw/pooling.py:211-225).  Writes,
 * per pooled row j, sizes_out[j], seeds_out[j] (tile-local seed row,
 * nullable) and members[j*rho + r] = r-th member row in index order (-1
 * padded); sub_out (nullable) gets each row's tile-local sub-bucket id.
 * flags (device int32) collects integrity failures (1 allocation short,
 * 2 no candidate, 4 over rho, 8 empty, 16 >1 under-filled, 32 bad id).
 * rho <= 64.  ntiles_dev (nullable): device tile count <= ntiles (e.g. the
 * totals[0] written by f3d_plan_pool). */
int f3d_pool_build(const double *coords, const int32_t *tile_start, const int32_t *tile_m,
                   const int32_t *tile_out, int ntiles, int rho, int32_t *sub_out,
                   int32_t *members, int32_t *sizes_out, int32_t *seeds_out,
                   int32_t *passes_out, int32_t *flags, const int32_t *ntiles_dev,
                   void *stream);
/* Pooling map for unpooling (no reference counterpart):
 * parent[members[j*rho + r]] = j for r < sizes[j]. */
int f3d_pool_parent(const int32_t *members, const int32_t *sizes, int64_t npool, int rho,
                    int32_t *parent, const int32_t *npool_dev, void *stream);
/* Replaces bw/pooling.py:166-184 pool_features: out[j] = reduce over
 * members of x (sequential in index order; mean = sum / size).
 * dtype: 0 bf16, 1 float, 2 double.  op: 0 sum, 1 mean, 2 min, 3 max.
 * npool_dev (nullable): device pooled-row count <= npool (totals[1]). */
int f3d_pool_reduce(const void *x, int dtype, int64_t ldx, int d, const int32_t *members,
                    const int32_t *sizes, int64_t npool, int rho, int op, void *out,
                    int64_t ldo, const int32_t *npool_dev, void *stream);

/* A stage's last residual and the bf16 copy of the result in one pass:
 * F += y + ybias (f3d_row_ln's arithmetic; ybias NULL = zero), out = bf16(F).  d % 4 == 0.
 * Replaces the MLP residual of the last round (bw/stage.py:156-158) + a cast. */
int f3d_residual_out(float *F, int64_t ldf, const void *y_bf16, int64_t ldy, const float *ybias,
                     void *out_bf16, int64_t ldo, int64_t n, int d, void *stream);

/* f3d_pool_reduce of fp32 rows with the stage's pending residual folded in:
 * each member row is x + (y + ybias) (y bf16, f3d_row_ln's arithmetic), so the
 * last residual pass of a pooled stage is skipped.  d % 4 == 0.
 * Replaces bw/stage.py:156-158 (last residual) + bw/pooling.py:166-184 (reduce). */
int f3d_pool_reduce_res(const float *x, int64_t ldx, const void *y_bf16, int64_t ldy,
                        const float *ybias, int d, const int32_t *members, const int32_t *sizes,
                        int64_t npool, int rho, int op, float *out, int64_t ldo,
                        const int32_t *npool_dev, void *stream);

/* A stage's input scatter fused with its first LayerNorm + PE: row i of src
 * (bf16, or fp32 when src_is_f32; input order) goes to F[dest[i]] (fp32) and
 * x[dest[i]] = LN(F)*gain + beta + PE(coords[i]) (bf16) -- bit-identical to
 * f3d_scatter_rows(_bf16_f32) followed by f3d_row_ln.  d % 12 == 0, d <= 128;
 * n_dev (nullable): device row count <= n.  Replaces bw/bucketing.py:385-401
 * (scatter) + bw/stage.py:129-136 (LN1 + PE of the first round). */
int f3d_scatter_ln_pe(const void *src, int src_is_f32, int64_t lds, const int32_t *dest,
                      const double *coords, const double *lo_ext, double pe_base,
                      const float *gain, const float *beta, float *F, int64_t ldf, void *out_bf16,
                      int64_t ldo, int64_t n, int d, double eps, const int32_t *n_dev,
                      void *stream);

/* Stage projection GEMM on the tensor cores: y = x W (+ bias) (GELU-erf when
 * gelu != 0) as bf16 rows, fp32 accumulation in TMEM.  x: n x K bf16 (row
 * stride ldx), w_t = W^T (N x K row-major bf16), bias: N fp32 (nullable), y:
 * n x N bf16 (row stride ldy).  The QKV, O-projection and MLP GEMMs of
 * bw/stage.py:135-138, 146-158.  K % 32 == 0, N % 16 == 0, N <= 4096
 * (f3d_gemm_supported); 16-byte aligned rows.  n_dev (nullable): device row
 * count <= n. */
int f3d_gemm_supported(int K, int N);
int f3d_gemm(const void *x, int64_t ldx, int64_t n, int K, const void *w_t, int N,
             const float *bias, int gelu, void *y, int64_t ldy, const int32_t *n_dev,
             void *stream);

/* The O-projection / MLP-output GEMM with the residual + LayerNorm (+PE) row
 * pass in its epilogue (bw/stage.py:134-158: F += attn W_o + b_o, x = LN2(F);
 * F += MLP W_out + b_out, x = LN1(F) + PE for the next round):
 *   F[r] += x[r] W + bias   (F: n x N fp32, row stride ldf, in place)
 *   y[r]  = (F[r] - mean) / sqrt(var + eps) * gain + beta (+ PE) as bf16
 * gain == NULL: residual only (y unused).  pe_coords (nullable): (n,3) f64 rows
 * and lo_ext the bbox [lo x,y,z, extent x,y,z] (as f3d_row_ln; N % 6 == 0).
 * The fp32 residual tile is TMA-loaded into shared memory and leaves with F
 * and y by TMA stores.  N % 32 == 0, N <= 256 (f3d_gemm_res_ln_supported). */
int f3d_gemm_res_ln_supported(int K, int N);
int f3d_gemm_res_ln(const void *x, int64_t ldx, int64_t n, int K, const void *w_t, int N,
                    const float *bias, float *F, int64_t ldf, const float *gain,
                    const float *beta, const double *pe_coords, const double *lo_ext,
                    double pe_base, double eps, void *y, int64_t ldy, const int32_t *n_dev,
                    void *stream);

/* ------------------------------------------------ training
 * LayerNorm backward fused with the residual add: dx = dres + rstd*(g*dy -
 * mean(g*dy) - xhat*mean(g*dy*xhat)); dgain += sum dy*xhat, dbeta += sum dy
 * (fp32 atomics).  x is the LN input (fp32), dy bf16 (dy_bf16=1) or fp32. */
int f3d_ln_bwd(const float *x, int64_t ldx, const void *dy, int dy_bf16, int64_t ldy,
               const float *gain, const float *dres, int64_t ldr, float *dx, int64_t ldd,
               float *dgain, float *dbeta, int64_t n, int d, double eps, void *stream);
/* du = dg * GELU'(u + bias) (exact erf form), dbias += sum du. */
int f3d_gelu_bwd(const void *u_bf16, int64_t ldu, const float *bias, const float *dg,
                 int64_t ldg, float *du, int64_t ldd, float *dbias, int64_t n, int h,
                 void *stream);
/* out[c] += sum_r x[r, c] (bias gradients). */
int f3d_colsum(const void *x, int is_bf16, int64_t ldx, int64_t n, int d, float *out,
               void *stream);
/* Padded per-(scope, head) score tiles [B, M, M] (M % 8 == 0): T is the fp32
 * GEMM output, out the bf16 operand of the next GEMM.  mode 0: out = P =
 * exp2(T*scale_log2 - rowv[b,i]) (rowv = lse); mode 1 (T = dP, P = the mode-0
 * bf16 output): out = dS = P*(dP - rowv[b,i])*scale (rowv = D = rowsum(dO*O)), or
 * with rowv = NULL, D = sum_j P*dP computed per row in the kernel (the consistent,
 * cancellation-safe form).  Zero outside len[b] rows/keys. */
int f3d_softmax_bwd(const float *T, const void *P, const float *rowv, const int32_t *len, int B,
                    int M, double scale_log2, double scale, int mode, void *out, void *stream);

/* Fused bucket-swin attention backward (training; the gradient of
 * bw/attention.py:188-268 per scope, which the reference does not provide):
 * dQ, dK, dV (fp32, head h at column h*dh, written at the fixed rows) from the
 * forward's bf16 q/k/v, the bf16 upstream gradient dout and the forward's
 * log2-domain row logsumexp lse (f3d_bswin_attention_tc's lse output), for the scopes
 * of one round (the same scope tables as the forward; nscopes / max_len are
 * upper bounds, empty scopes are skipped on the device).  Never forms an
 * m x m tile: a query-block kernel computes D = sum_j P dP / sum_j P per
 * (row, head) into the caller's delta buffer (rows x ld_delta fp32) and dQ,
 * then a key-block kernel accumulates dK, dV over the scope's query blocks
 * (bf16 mma.sync, fp32 accumulation).  Requires dh % 8 == 0, 8 <= dh <= 32. */
int f3d_attn_bwd(const void *q, const void *k, const void *v, const void *dout, int64_t ld_q,
                 int64_t ld_k, int64_t ld_v, int64_t ld_do, const float *lse, int64_t ld_lse,
                 float *delta, int64_t ld_delta, float *dq, int64_t ld_dq, float *dk,
                 int64_t ld_dk, float *dv, int64_t ld_dv, int H, int dh,
                 const int32_t *scope_seg, const int32_t *scope_nseg, const int32_t *seg_start,
                 const int32_t *seg_vstart, const int32_t *scope_len, int nscopes, int max_len,
                 void *stream);

#ifdef __cplusplus
}
#endif
#endif /* F3D_H_ */
