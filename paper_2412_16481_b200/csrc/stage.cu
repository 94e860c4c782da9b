// Stage row kernels around the GEMMs of bw/stage.py:99-159 (HBM-bound):
//   positional encoding of bbox-normalised coords (bw/attention.py:271-288,
//   bw/stage.py:129-132), fused residual + LayerNorm (+PE) -> bf16
//   (bw/stage.py:84-88, 135, 157-158), and bias + exact-erf GELU
//   (bw/stage.py:91-96).  One warp per row, fp32 (or f64) math.
#include <cuda_bf16.h>

#include <cstdlib>

#include <algorithm>
#include <cfloat>

#include "f3d_common.cuh"

namespace f3d {
namespace stage {

constexpr int kThreads = 256;
constexpr int kMaxPerLane = 32;   // d <= 1024

// ---------------------------------------------------------------- bbox

__global__ void bbox_partial_kernel(const double* __restrict__ c, int64_t n,
                                    const int32_t* n_dev, double* part) {
    f3d::pdl_wait();
    n = dyn_n(n, n_dev);
    __shared__ double s[6][kThreads / 32];
    double mn[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, mx[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        for (int a = 0; a < 3; ++a) {
            const double v = c[3 * i + a];
            mn[a] = fmin(mn[a], v);
            mx[a] = fmax(mx[a], v);
        }
    }
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[a] = fmin(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = fmax(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0)
        for (int a = 0; a < 3; ++a) {
            s[a][w] = mn[a];
            s[3 + a][w] = mx[a];
        }
    __syncthreads();
    if (threadIdx.x < 6) {
        double r = threadIdx.x < 3 ? DBL_MAX : -DBL_MAX;
        for (int j = 0; j < kThreads / 32; ++j)
            r = threadIdx.x < 3 ? fmin(r, s[threadIdx.x][j]) : fmax(r, s[threadIdx.x][j]);
        part[blockIdx.x * 6 + threadIdx.x] = r;
    }
}

// lo[3], ext[3] with ext == 0 -> 1 (bw/stage.py:129-131)
// one warp per axis: lanes stride over the partial results (min / max are
// exact in any order)
__global__ void bbox_final_kernel(const double* part, int nparts, double* lo_ext) {
    f3d::pdl_wait();
    const int a = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (a >= 3) return;
    double mn = DBL_MAX, mx = -DBL_MAX;
    for (int j = lane; j < nparts; j += 32) {
        mn = fmin(mn, part[6 * j + a]);
        mx = fmax(mx, part[6 * j + 3 + a]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane) return;
    double e = __dsub_rn(mx, mn);
    if (e == 0.0) e = 1.0;
    lo_ext[a] = mn;
    lo_ext[3 + a] = e;
}

// --------------------------------------------------------------------- PE

template <typename OutT>
__global__ void pe_kernel(const double* __restrict__ c, int64_t n, int d, double base,
                          const double* __restrict__ lo_ext, OutT* __restrict__ out, int64_t ld) {
    const int npair = d / 6;
    const int blk = 2 * npair;
    const int64_t tot = n * 3 * npair;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / (3 * npair);
        const int r = (int)(t - i * 3 * npair);
        const int a = r / npair, j = r - a * npair;
        double x = c[3 * i + a];
        if (lo_ext) x = __ddiv_rn(__dsub_rn(x, lo_ext[a]), lo_ext[3 + a]);
        const double inv = pow(base, -(double)j / (double)npair);
        const double ang = __dmul_rn(x, inv);
        double sv, cv;
        sincos(ang, &sv, &cv);
        out[i * ld + a * blk + 2 * j] = (OutT)sv;
        out[i * ld + a * blk + 2 * j + 1] = (OutT)cv;
    }
}

// ------------------------------------------------------- residual + LN

template <typename T> struct Acc { using type = float; };
template <> struct Acc<double> { using type = double; };

__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float to_f(float v) { return v; }

// F[r] += y[r] + bias (if y); out[r] = LN(F[r]) * g + b + pe[r] (if out).
__device__ __forceinline__ void store_out(__nv_bfloat16* p, double v) { *p = __float2bfloat16((float)v); }
__device__ __forceinline__ void store_out(float* p, double v) { *p = (float)v; }
__device__ __forceinline__ void store_out(double* p, double v) { *p = v; }

template <typename FT, typename OT, int PER>
__global__ void __launch_bounds__(kThreads) row_ln_kernel(
    FT* __restrict__ F, int64_t ldf, const __nv_bfloat16* __restrict__ y, int64_t ldy,
    const float* __restrict__ ybias, const float* __restrict__ gain,
    const float* __restrict__ beta, const double* __restrict__ pec,
    const double* __restrict__ lo_ext, float pe_log2base, OT* __restrict__ out, int64_t ldo,
    int64_t n, int d, double eps) {
    using A = typename Acc<FT>::type;
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
    if (row >= n) return;
    FT* fr = F + row * ldf;
    // issue every load of the row first (ILP), then reduce
    A v[PER];
    A yv[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int c = lane + 32 * j;
        v[j] = (c < d) ? (A)fr[c] : (A)0;
        yv[j] = (y && c < d) ? (A)to_f(y[row * ldy + c]) : (A)0;
    }
    if (y) {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int c = lane + 32 * j;
            if (c < d) {
                v[j] += yv[j] + (ybias ? (A)ybias[c] : (A)0);
                fr[c] = (FT)v[j];
            }
        }
    }
    if (!out) return;
    A s = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) s += v[j];
    s = warp_sum(s);
    const A mean = s / (A)d;
    A q = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int c = lane + 32 * j;
        const A t = (c < d) ? v[j] - mean : (A)0;
        q += t * t;
    }
    q = warp_sum(q);
    const A rstd = (A)1 / sqrt(q / (A)d + (A)eps);
    // positional encoding of the bbox-normalised coordinate, computed on the
    // fly (bw/attention.py:271-288; bw/stage.py:129-132): d/3 dims per axis,
    // alternating sin/cos of x * base^(-j/npair)
    float xn[3] = {0.f, 0.f, 0.f};
    const int npair = d / 6, blk = 2 * npair;
    if (pec) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            double x = pec[3 * row + a];
            if (lo_ext) x = __ddiv_rn(__dsub_rn(x, lo_ext[a]), lo_ext[3 + a]);
            xn[a] = (float)x;
        }
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int c = lane + 32 * j;
        if (c < d) {
            A o = (v[j] - mean) * rstd * (A)gain[c] + (A)beta[c];
            if (pec) {
                // |ang| <= ~1 for normalised coords: the fast MUFU forms are
                // accurate to ~1e-6 absolute, far inside the bf16 output
                const int a = c / blk, k = c - a * blk, jj = k >> 1;
                const float ang = xn[a] * exp2f(-(float)jj / (float)npair * pe_log2base);
                o += (A)((k & 1) ? __cosf(ang) : __sinf(ang));
            }
            store_out(out + row * ldo + c, (double)o);
        }
    }
}

// GELU with the erf form (bw/stage.py:91-92).  erf via Abramowitz & Stegun
// 7.1.26 (|error| <= 1.5e-7, below the bf16 rounding of the result):
// erf(z) = 1 - (a1 t + ... + a5 t^5) e^{-z^2}, t = 1 / (1 + p z), odd in z;
// one MUFU.RCP + one MUFU.EX2 and 7 FMA instead of erff's polynomial chain.
__device__ __forceinline__ float gelu_f(float x) {
    const float z = fabsf(x) * 0.70710678118654752f;
    float t;   // MUFU reciprocal / exp2 (approx): 1-2 ulp, far inside the 1.5e-7 formula error
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, z, 1.f)));
    float pl = fmaf(1.061405429f, t, -1.453152027f);
    pl = fmaf(pl, t, 1.421413741f);
    pl = fmaf(pl, t, -0.284496736f);
    pl = fmaf(pl, t, 0.254829592f);
    pl *= t;
    float ez;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ez) : "f"(-z * z * 1.4426950408889634f));
    const float e = 1.f - pl * ez;   // erf(|x|/sqrt2)
    const float phi2 = 1.f + copysignf(e, x);                          // 1 + erf(x/sqrt2)
    return 0.5f * x * phi2;
}

// 16-byte vector form: 8 bf16 per vector (dh % 8 == 0); each thread loads
// kU vectors before computing any (memory-level parallelism: one 16-byte load
// in flight per thread left the kernel latency-bound).  IT = uint32_t when the
// element count allows it (a 64-bit modulo per vector costs more than the
// GELU itself).
template <typename IT>
__global__ void bias_gelu8_kernel(uint4* __restrict__ u, IT n8, int dh8,
                                  const float4* __restrict__ b) {
    constexpr int kU = 4;
    const IT stride = (IT)gridDim.x * blockDim.x;
    for (IT t0 = (IT)blockIdx.x * blockDim.x + threadIdx.x; t0 < n8; t0 += stride * kU) {
        uint4 w[kU];
#pragma unroll
        for (int q = 0; q < kU; ++q) {
            const IT t = t0 + q * stride;
            if (t < n8) w[q] = u[t];
        }
#pragma unroll
        for (int q = 0; q < kU; ++q) {
            const IT t = t0 + q * stride;
            if (t >= n8) break;
            const int c8 = (int)(t % (IT)dh8);
            const float4 b0 = __ldg(b + 2 * c8), b1 = __ldg(b + 2 * c8 + 1);
            const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&w[q]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float2 f = __bfloat1622float2(h[e]);
                f2_split(fadd2(f2(f.x, f.y), f2(bb[2 * e], bb[2 * e + 1])), f.x, f.y);
                const float2 g = gelu2(f.x, f.y);
                h[e] = __floats2bfloat162_rn(g.x, g.y);
            }
            u[t] = w[q];
        }
    }
}

// u = gelu(u + b), exact erf form, in place on bf16 rows.
__global__ void bias_gelu_kernel(__nv_bfloat16* __restrict__ u, int64_t n, int dh,
                                 const float* __restrict__ b) {
    const int64_t tot2 = n * dh / 2;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot2;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)((2 * t) % dh);
        __nv_bfloat162 p = reinterpret_cast<__nv_bfloat162*>(u)[t];
        float x0 = __bfloat162float(p.x) + b[c], x1 = __bfloat162float(p.y) + b[c + 1];
        x0 = 0.5f * x0 * (1.f + erff(x0 * 0.70710678118654752f));
        x1 = 0.5f * x1 * (1.f + erff(x1 * 0.70710678118654752f));
        reinterpret_cast<__nv_bfloat162*>(u)[t] = __floats2bfloat162_rn(x0, x1);
    }
}

}  // namespace stage
}  // namespace f3d

using namespace f3d;

static inline unsigned grid_for(int64_t work, int threads) {
    int64_t g = (work + threads - 1) / threads;
    const int64_t cap = (int64_t)f3d_num_sms() * 16;
    if (g > cap) g = cap;
    return (unsigned)(g < 1 ? 1 : g);
}

extern "C" int f3d_coord_bbox(const double* coords, int64_t n, double* ws, double* lo_ext,
                              const int32_t* n_dev, void* stream) {
    if (n < 1) return F3D_ERR_EMPTY;
    cudaStream_t st = (cudaStream_t)stream;
    const int parts = (int)std::min<int64_t>((n + 1023) / 1024, 296);
    F3D_CUDA_TRY(f3d_launch(stage::bbox_partial_kernel, dim3(parts), dim3(stage::kThreads), 0, st,
                            coords, n, n_dev, ws));
    F3D_CUDA_TRY(f3d_launch(stage::bbox_final_kernel, dim3(1), dim3(96), 0, st, (const double*)ws,
                            parts, lo_ext));
    return F3D_OK;
}

extern "C" int f3d_positional_encoding(const double* coords, int64_t n, int d, double base,
                                       int out_f64, void* out, int64_t ld, void* stream) {
    return f3d_stage_pe(coords, n, d, base, nullptr, out_f64 ? 2 : 1, out, ld, stream);
}

extern "C" int f3d_stage_pe(const double* coords, int64_t n, int d, double base,
                            const double* lo_ext, int out_kind, void* out, int64_t ld,
                            void* stream) {
    if (d % 6 || d < 6 || n < 0) return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t work = n * 3 * (d / 6);
    const unsigned g = grid_for(work, stage::kThreads);
    if (out_kind == 2)
        stage::pe_kernel<double><<<g, stage::kThreads, 0, st>>>(coords, n, d, base, lo_ext,
                                                                (double*)out, ld);
    else
        stage::pe_kernel<float><<<g, stage::kThreads, 0, st>>>(coords, n, d, base, lo_ext,
                                                               (float*)out, ld);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

namespace f3d {
namespace stage {

// Vector form of row_ln for the pipeline's common case: fp32 residual rows,
// bf16 y / out, d % 4 == 0, d <= 128.  Lane q owns columns [4q, 4q+4) (one
// 16-byte F load, one 8-byte y load); each warp carries RPW rows at once so
// every load of all of them is in flight before the first reduction.
template <int RPW, bool HAS_Y, bool HAS_OUT, bool HAS_PE>
__global__ void __launch_bounds__(kThreads, HAS_PE ? 4 : 5) row_ln_vec_kernel(
    float* __restrict__ F, int64_t ldf, const __nv_bfloat16* __restrict__ y, int64_t ldy,
    const float* __restrict__ ybias, const float* __restrict__ gain,
    const float* __restrict__ beta, const double* __restrict__ pec,
    const double* __restrict__ lo_ext, float pl2, __nv_bfloat16* __restrict__ out, int64_t ldo,
    int64_t n, int d, float eps) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const bool act = lane < (d >> 2);
    const int64_t row0 = ((int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * RPW;
    const int c0 = 4 * lane;
    float4 v[RPW];
    uint2 yy[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int64_t row = row0 + i;
        const bool ok = act && row < n;
        v[i] = ok ? *reinterpret_cast<const float4*>(F + row * ldf + c0) : make_float4(0, 0, 0, 0);
        if (HAS_Y) yy[i] = ok ? *reinterpret_cast<const uint2*>(y + row * ldy + c0) : make_uint2(0, 0);
    }
    if (HAS_Y) {
        const float4 yb = (ybias && act) ? *reinterpret_cast<const float4*>(ybias + c0)
                                         : make_float4(0, 0, 0, 0);
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&yy[i]);
            const float2 y01 = __bfloat1622float2(h[0]), y23 = __bfloat1622float2(h[1]);
            v[i].x += y01.x + yb.x;
            v[i].y += y01.y + yb.y;
            v[i].z += y23.x + yb.z;
            v[i].w += y23.y + yb.w;
            const int64_t row = row0 + i;
            if (act && row < n) *reinterpret_cast<float4*>(F + row * ldf + c0) = v[i];
        }
    }
    if (!HAS_OUT) return;
    float s[RPW], q[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) s[i] = (v[i].x + v[i].y) + (v[i].z + v[i].w);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < RPW; ++i) s[i] += __shfl_xor_sync(0xffffffffu, s[i], o);
    const float inv_d = 1.f / (float)d;
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const float m = s[i] * inv_d;
        const float a = act ? v[i].x - m : 0.f, b = act ? v[i].y - m : 0.f;
        const float c = act ? v[i].z - m : 0.f, e = act ? v[i].w - m : 0.f;
        q[i] = (a * a + b * b) + (c * c + e * e);
        s[i] = m;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < RPW; ++i) q[i] += __shfl_xor_sync(0xffffffffu, q[i], o);
    if (!act) return;
    const float4 gg = *reinterpret_cast<const float4*>(gain + c0);
    const float4 bb = *reinterpret_cast<const float4*>(beta + c0);
    // PE: columns (c0, c0+1) and (c0+2, c0+3) are (sin, cos) pairs (d % 6 == 0,
    // so blk = d/3 is even); bw/attention.py:271-288 on the bbox-normalised
    // coordinate (bw/stage.py:129-132)
    const int npair = d / 6, blk = 2 * npair;
    // per lane: the axis and frequency of its two pairs, the axis offset and
    // reciprocal extent (fp32 angles: the normalised coordinate is in [0, 1])
    int pa[2];
    float fq[2], pinv[2];
    double plo[2];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const int c = c0 + 2 * p;
        pa[p] = c / blk;
        const int pj = (c - pa[p] * blk) >> 1;
        fq[p] = exp2f(-(float)pj / (float)npair * pl2);
        plo[p] = lo_ext ? lo_ext[pa[p]] : 0.0;
        pinv[p] = lo_ext ? (float)(1.0 / lo_ext[3 + pa[p]]) : 1.f;
    }
    // PE inputs: only this lane's two axes, loaded after the reductions (short
    // live ranges: the PE variant stays at the non-PE occupancy)
    double pcv[RPW][2];
    if (HAS_PE) {
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            const int64_t row = row0 + i < n ? row0 + i : 0;
            pcv[i][0] = pec[3 * row + pa[0]];
            pcv[i][1] = pec[3 * row + pa[1]];
        }
    }
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int64_t row = row0 + i;
        if (row >= n) break;
        const float rstd = rsqrtf(q[i] * inv_d + eps);
        const float m = s[i];
        float o0 = (v[i].x - m) * rstd * gg.x + bb.x;
        float o1 = (v[i].y - m) * rstd * gg.y + bb.y;
        float o2 = (v[i].z - m) * rstd * gg.z + bb.z;
        float o3 = (v[i].w - m) * rstd * gg.w + bb.w;
        if (HAS_PE) {
            float sn[2], cs[2];
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const float xn = (float)__dsub_rn(pcv[i][p], plo[p]) * pinv[p];
                __sincosf(xn * fq[p], &sn[p], &cs[p]);
            }
            o0 += sn[0];
            o1 += cs[0];
            o2 += sn[1];
            o3 += cs[1];
        }
        __nv_bfloat162 h0 = __floats2bfloat162_rn(o0, o1), h1 = __floats2bfloat162_rn(o2, o3);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&h0);
        w.y = *reinterpret_cast<uint32_t*>(&h1);
        *reinterpret_cast<uint2*>(out + row * ldo + c0) = w;
    }
}

// ---- 8 lanes per row (d % 32 == 0, d <= 128): VPL = d / 32 float4 per lane,
// lane l of a group owning the 16-byte chunks l, l + 8, ..; four rows per warp
// at once, RB row batches per warp.  Every lane is busy at d = 96 (the
// 32-lane form above leaves lanes 24..31 idle) and the row reductions take
// three shuffle steps instead of five.  Used for the plain LayerNorm (no PE).
template <int VPL>
__device__ __forceinline__ float2 ln8_stats(const float4 (&v)[VPL], float inv_d, float eps) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    const float m = s * inv_d;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
        const float a = v[k].x - m, b = v[k].y - m, c = v[k].z - m, e = v[k].w - m;
        q += (a * a + b * b) + (c * c + e * e);
    }
    q += __shfl_xor_sync(0xffffffffu, q, 1);
    q += __shfl_xor_sync(0xffffffffu, q, 2);
    q += __shfl_xor_sync(0xffffffffu, q, 4);
    return make_float2(m, rsqrtf(q * inv_d + eps));
}

// LN(v) * gain + beta -> bf16 at out_row
template <int VPL>
__device__ __forceinline__ void ln8_out(const float4 (&v)[VPL], float2 st, int gl,
                                        const float4 (&gg)[VPL], const float4 (&bb)[VPL],
                                        __nv_bfloat16* out_row) {
    const float m = st.x, rstd = st.y;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
        const float o0 = (v[k].x - m) * rstd * gg[k].x + bb[k].x;
        const float o1 = (v[k].y - m) * rstd * gg[k].y + bb[k].y;
        const float o2 = (v[k].z - m) * rstd * gg[k].z + bb[k].z;
        const float o3 = (v[k].w - m) * rstd * gg[k].w + bb[k].w;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(o0, o1), h1 = __floats2bfloat162_rn(o2, o3);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&h0);
        w.y = *reinterpret_cast<uint32_t*>(&h1);
        *reinterpret_cast<uint2*>(out_row + 4 * (gl + 8 * k)) = w;
    }
}

constexpr int kRB8 = 2;   // row batches per warp (8 rows per warp)

template <int VPL, bool HAS_Y, bool HAS_OUT>
__global__ void __launch_bounds__(kThreads, 3) row_ln8_kernel(
    float* __restrict__ F, int64_t ldf, const __nv_bfloat16* __restrict__ y, int64_t ldy,
    const float* __restrict__ ybias, const float* __restrict__ gain,
    const float* __restrict__ beta, __nv_bfloat16* __restrict__ out, int64_t ldo, int64_t n, int d,
    float eps) {
    pdl_wait();
    const int lane = threadIdx.x & 31, grp = lane >> 3, gl = lane & 7;
    const int64_t rw = ((int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * (4 * kRB8);
    if (rw >= n) return;
    float4 v[kRB8][VPL];
#pragma unroll
    for (int b = 0; b < kRB8; ++b) {
        const int64_t row = rw + 4 * b + grp;
        const bool ok = row < n;
#pragma unroll
        for (int k = 0; k < VPL; ++k)
            v[b][k] = ok ? *reinterpret_cast<const float4*>(F + row * ldf + 4 * (gl + 8 * k))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (HAS_Y) {
        uint2 yy[kRB8][VPL];
#pragma unroll
        for (int b = 0; b < kRB8; ++b) {
            const int64_t row = rw + 4 * b + grp;
#pragma unroll
            for (int k = 0; k < VPL; ++k)
                yy[b][k] = row < n ? *reinterpret_cast<const uint2*>(y + row * ldy + 4 * (gl + 8 * k))
                                   : make_uint2(0, 0);
        }
#pragma unroll
        for (int b = 0; b < kRB8; ++b) {
            const int64_t row = rw + 4 * b + grp;
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
                const int c = 4 * (gl + 8 * k);
                const float4 yb = ybias ? *reinterpret_cast<const float4*>(ybias + c)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&yy[b][k]);
                const float2 y01 = __bfloat1622float2(h[0]), y23 = __bfloat1622float2(h[1]);
                v[b][k].x += y01.x + yb.x;
                v[b][k].y += y01.y + yb.y;
                v[b][k].z += y23.x + yb.z;
                v[b][k].w += y23.y + yb.w;
                if (row < n) *reinterpret_cast<float4*>(F + row * ldf + c) = v[b][k];
            }
        }
    }
    if (!HAS_OUT) return;
    const float inv_d = 1.f / (float)d;
    float4 gg[VPL], bb[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
        gg[k] = *reinterpret_cast<const float4*>(gain + 4 * (gl + 8 * k));
        bb[k] = *reinterpret_cast<const float4*>(beta + 4 * (gl + 8 * k));
    }
#pragma unroll
    for (int b = 0; b < kRB8; ++b) {
        const float2 st = ln8_stats<VPL>(v[b], inv_d, eps);
        const int64_t row = rw + 4 * b + grp;
        if (row < n) ln8_out<VPL>(v[b], st, gl, gg, bb, out + row * ldo);
    }
}

// ---- 8 lanes per row with the positional encoding (d == 96: the only width
// with d % 6 == 0 and d % 32 == 0 up to 128).  Lane gl of a row group owns the
// 16-byte chunks gl, gl + 8, gl + 16; chunk gl + 8k holds the (sin, cos) pairs
// of axis k at frequencies 2gl and 2gl + 1.  The per-element arithmetic is
// row_ln_vec's (angles, affine, PE add); the row statistics are ln8_stats'.
// row_ln8pe (residual + LN1 + PE of the next round) and scatter_ln8pe (input
// scatter + first LN1 + PE) share it, so the fused scatter stays bit-identical
// to scatter + row_ln.
struct Pe8 {
    float fq[2];
    double plo[3];
    float pinv[3];
};
__device__ __forceinline__ Pe8 pe8_consts(int gl, const double* __restrict__ lo_ext, float pl2) {
    Pe8 c;
#pragma unroll
    for (int p = 0; p < 2; ++p) c.fq[p] = exp2f(-(float)(2 * gl + p) / 16.f * pl2);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        c.plo[a] = lo_ext ? lo_ext[a] : 0.0;
        c.pinv[a] = lo_ext ? (float)(1.0 / lo_ext[3 + a]) : 1.f;
    }
    return c;
}

// LN(v) * gain + beta + PE(coords of the row) -> bf16 at out_row (d == 96)
__device__ __forceinline__ void ln8pe_out(const float4 (&v)[3], float2 st, int gl,
                                          const float* __restrict__ gain,
                                          const float* __restrict__ beta, const Pe8& pc,
                                          const double* __restrict__ crow,
                                          __nv_bfloat16* __restrict__ out_row) {
    const float m = st.x, rstd = st.y;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int c = 4 * (gl + 8 * k);
        const float4 gg = __ldg(reinterpret_cast<const float4*>(gain + c));
        const float4 bb = __ldg(reinterpret_cast<const float4*>(beta + c));
        float o0 = (v[k].x - m) * rstd * gg.x + bb.x;
        float o1 = (v[k].y - m) * rstd * gg.y + bb.y;
        float o2 = (v[k].z - m) * rstd * gg.z + bb.z;
        float o3 = (v[k].w - m) * rstd * gg.w + bb.w;
        const float xn = (float)__dsub_rn(crow[k], pc.plo[k]) * pc.pinv[k];
        float sn[2], cs[2];
#pragma unroll
        for (int p = 0; p < 2; ++p) __sincosf(xn * pc.fq[p], &sn[p], &cs[p]);
        o0 += sn[0];
        o1 += cs[0];
        o2 += sn[1];
        o3 += cs[1];
        __nv_bfloat162 h0 = __floats2bfloat162_rn(o0, o1), h1 = __floats2bfloat162_rn(o2, o3);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&h0);
        w.y = *reinterpret_cast<uint32_t*>(&h1);
        *reinterpret_cast<uint2*>(out_row + c) = w;
    }
}

constexpr int kRB8pe = 2;   // row batches per warp of the PE kernels (8 rows per warp)

template <bool HAS_Y>
__global__ void __launch_bounds__(kThreads, 3) row_ln8pe_kernel(
    float* __restrict__ F, int64_t ldf, const __nv_bfloat16* __restrict__ y, int64_t ldy,
    const float* __restrict__ ybias, const float* __restrict__ gain,
    const float* __restrict__ beta, const double* __restrict__ pec,
    const double* __restrict__ lo_ext, float pl2, __nv_bfloat16* __restrict__ out, int64_t ldo,
    int64_t n, float eps) {
    pdl_wait();
    const int lane = threadIdx.x & 31, grp = lane >> 3, gl = lane & 7;
    const int64_t rw = ((int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * (4 * kRB8pe);
    if (rw >= n) return;
    float4 v[kRB8pe][3];
#pragma unroll
    for (int b = 0; b < kRB8pe; ++b) {
        const int64_t row = rw + 4 * b + grp;
        const bool ok = row < n;
#pragma unroll
        for (int k = 0; k < 3; ++k)
            v[b][k] = ok ? *reinterpret_cast<const float4*>(F + row * ldf + 4 * (gl + 8 * k))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (HAS_Y) {
        uint2 yy[kRB8pe][3];
#pragma unroll
        for (int b = 0; b < kRB8pe; ++b) {
            const int64_t row = rw + 4 * b + grp;
#pragma unroll
            for (int k = 0; k < 3; ++k)
                yy[b][k] = row < n ? *reinterpret_cast<const uint2*>(y + row * ldy + 4 * (gl + 8 * k))
                                   : make_uint2(0, 0);
        }
#pragma unroll
        for (int b = 0; b < kRB8pe; ++b) {
            const int64_t row = rw + 4 * b + grp;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int c = 4 * (gl + 8 * k);
                const float4 yb = ybias ? *reinterpret_cast<const float4*>(ybias + c)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&yy[b][k]);
                const float2 y01 = __bfloat1622float2(h[0]), y23 = __bfloat1622float2(h[1]);
                v[b][k].x += y01.x + yb.x;
                v[b][k].y += y01.y + yb.y;
                v[b][k].z += y23.x + yb.z;
                v[b][k].w += y23.y + yb.w;
                if (row < n) *reinterpret_cast<float4*>(F + row * ldf + c) = v[b][k];
            }
        }
    }
    const Pe8 pc = pe8_consts(gl, lo_ext, pl2);
#pragma unroll
    for (int b = 0; b < kRB8pe; ++b) {
        const float2 st = ln8_stats<3>(v[b], 1.f / 96.f, eps);
        const int64_t row = rw + 4 * b + grp;
        if (row < n) ln8pe_out(v[b], st, gl, gain, beta, pc, pec + 3 * row, out + row * ldo);
    }
}

template <typename ST>
__global__ void __launch_bounds__(kThreads, 3) scatter_ln8pe_kernel(
    const ST* __restrict__ src, int64_t lds, const int32_t* __restrict__ dest,
    const double* __restrict__ C, const double* __restrict__ lo_ext, float pl2,
    const float* __restrict__ gain, const float* __restrict__ beta, float* __restrict__ F,
    int64_t ldf, __nv_bfloat16* __restrict__ out, int64_t ldo, int64_t n,
    const int32_t* __restrict__ n_dev, float eps) {
    pdl_wait();
    const int lane = threadIdx.x & 31, grp = lane >> 3, gl = lane & 7;
    const int64_t nn = dyn_n(n, n_dev);
    const int64_t rw = ((int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * (4 * kRB8pe);
    if (rw >= nn) return;
    float4 v[kRB8pe][3];
#pragma unroll
    for (int b = 0; b < kRB8pe; ++b) {
        const int64_t row = rw + 4 * b + grp;
        const bool ok = row < nn;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int c = 4 * (gl + 8 * k);
            if (sizeof(ST) == 2) {
                if (ok) {
                    const uint2 w = *reinterpret_cast<const uint2*>(
                        reinterpret_cast<const __nv_bfloat16*>(src) + row * lds + c);
                    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
                    const float2 a = __bfloat1622float2(h[0]), bq = __bfloat1622float2(h[1]);
                    v[b][k] = make_float4(a.x, a.y, bq.x, bq.y);
                } else {
                    v[b][k] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            } else {
                v[b][k] = ok ? *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(src) +
                                                               row * lds + c)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    }
    const Pe8 pc = pe8_consts(gl, lo_ext, pl2);
#pragma unroll
    for (int b = 0; b < kRB8pe; ++b) {
        const float2 st = ln8_stats<3>(v[b], 1.f / 96.f, eps);
        const int64_t row = rw + 4 * b + grp;
        if (row >= nn) continue;
        const int64_t dr = __ldg(dest + row);
#pragma unroll
        for (int k = 0; k < 3; ++k)
            *reinterpret_cast<float4*>(F + dr * ldf + 4 * (gl + 8 * k)) = v[b][k];
        ln8pe_out(v[b], st, gl, gain, beta, pc, C + 3 * row, out + dr * ldo);
    }
}

// Scatter + first LayerNorm + PE of a stage in one pass: input row i (bf16 or
// fp32, input order) -> F[dest[i]] (fp32) and x[dest[i]] = LN(F)*g + b + PE(C[i])
// (bf16), with row_ln_vec_kernel's arithmetic (so bit-identical to the scatter
// followed by f3d_row_ln), saving the re-read of F.
template <int RPW, typename ST>
__global__ void __launch_bounds__(kThreads, 4) scatter_ln_pe_kernel(
    const ST* __restrict__ src, int64_t lds, const int32_t* __restrict__ dest,
    const double* __restrict__ C, const double* __restrict__ lo_ext, float pl2,
    const float* __restrict__ gain, const float* __restrict__ beta, float* __restrict__ F,
    int64_t ldf, __nv_bfloat16* __restrict__ out, int64_t ldo, int64_t n,
    const int32_t* __restrict__ n_dev, int d, float eps) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const bool act = lane < (d >> 2);
    const int64_t nn = dyn_n(n, n_dev);
    const int64_t row0 = ((int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * RPW;
    if (row0 >= nn) return;
    const int c0 = 4 * lane;
    float4 v[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int64_t row = row0 + i;
        const bool ok = act && row < nn;
        if (sizeof(ST) == 2) {
            if (ok) {
                const uint2 w = *reinterpret_cast<const uint2*>(
                    reinterpret_cast<const __nv_bfloat16*>(src) + row * lds + c0);
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
                const float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
                v[i] = make_float4(a.x, a.y, b.x, b.y);
            } else {
                v[i] = make_float4(0, 0, 0, 0);
            }
        } else {
            v[i] = ok ? *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(src) +
                                                         row * lds + c0)
                      : make_float4(0, 0, 0, 0);
        }
    }
    float s[RPW], q[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) s[i] = (v[i].x + v[i].y) + (v[i].z + v[i].w);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < RPW; ++i) s[i] += __shfl_xor_sync(0xffffffffu, s[i], o);
    const float inv_d = 1.f / (float)d;
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const float m = s[i] * inv_d;
        const float a = act ? v[i].x - m : 0.f, b = act ? v[i].y - m : 0.f;
        const float c = act ? v[i].z - m : 0.f, e = act ? v[i].w - m : 0.f;
        q[i] = (a * a + b * b) + (c * c + e * e);
        s[i] = m;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < RPW; ++i) q[i] += __shfl_xor_sync(0xffffffffu, q[i], o);
    if (!act) return;
    const float4 gg = *reinterpret_cast<const float4*>(gain + c0);
    const float4 bb = *reinterpret_cast<const float4*>(beta + c0);
    const int npair = d / 6, blk = 2 * npair;
    int pa[2];
    float fq[2], pinv[2];
    double plo[2];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const int c = c0 + 2 * p;
        pa[p] = c / blk;
        const int pj = (c - pa[p] * blk) >> 1;
        fq[p] = exp2f(-(float)pj / (float)npair * pl2);
        plo[p] = lo_ext ? lo_ext[pa[p]] : 0.0;
        pinv[p] = lo_ext ? (float)(1.0 / lo_ext[3 + pa[p]]) : 1.f;
    }
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int64_t row = row0 + i;
        if (row >= nn) break;
        const int64_t dr = __ldg(dest + row);
        *reinterpret_cast<float4*>(F + dr * ldf + c0) = v[i];
        const float rstd = rsqrtf(q[i] * inv_d + eps);
        const float m = s[i];
        float o0 = (v[i].x - m) * rstd * gg.x + bb.x;
        float o1 = (v[i].y - m) * rstd * gg.y + bb.y;
        float o2 = (v[i].z - m) * rstd * gg.z + bb.z;
        float o3 = (v[i].w - m) * rstd * gg.w + bb.w;
        float sn[2], cs[2];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const float xn = (float)__dsub_rn(C[3 * row + pa[p]], plo[p]) * pinv[p];
            __sincosf(xn * fq[p], &sn[p], &cs[p]);
        }
        o0 += sn[0];
        o1 += cs[0];
        o2 += sn[1];
        o3 += cs[1];
        __nv_bfloat162 h0 = __floats2bfloat162_rn(o0, o1), h1 = __floats2bfloat162_rn(o2, o3);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&h0);
        w.y = *reinterpret_cast<uint32_t*>(&h1);
        *reinterpret_cast<uint2*>(out + dr * ldo + c0) = w;
    }
}

// A stage's last residual fused with the bf16 copy of the result:
// F += y + b (f3d_row_ln's arithmetic), out = bf16(F); 4 columns per thread.
__global__ void residual_out_kernel(float* __restrict__ F, int64_t ldf,
                                    const __nv_bfloat16* __restrict__ y, int64_t ldy,
                                    const float* __restrict__ yb, __nv_bfloat16* __restrict__ out,
                                    int64_t ldo, int64_t n, int d4) {
    pdl_wait();
    const int64_t tot = n * d4;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / d4;
        const int c = 4 * (int)(t - r * d4);
        float4 v = *reinterpret_cast<const float4*>(F + r * ldf + c);
        const uint2 w = *reinterpret_cast<const uint2*>(y + r * ldy + c);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
        const float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
        const float4 bb = yb ? *reinterpret_cast<const float4*>(yb + c)
                             : make_float4(0.f, 0.f, 0.f, 0.f);   // NULL ybias = zero bias
        v.x += a.x + bb.x;
        v.y += a.y + bb.y;
        v.z += b.x + bb.z;
        v.w += b.y + bb.w;
        *reinterpret_cast<float4*>(F + r * ldf + c) = v;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(v.x, v.y), h1 = __floats2bfloat162_rn(v.z, v.w);
        uint2 o;
        o.x = *reinterpret_cast<uint32_t*>(&h0);
        o.y = *reinterpret_cast<uint32_t*>(&h1);
        *reinterpret_cast<uint2*>(out + r * ldo + c) = o;
    }
}

}  // namespace stage
}  // namespace f3d

// returns false when the vector form does not apply
static bool launch_row_ln_vec(cudaStream_t st, void* F, int64_t ldf, const void* y, int64_t ldy,
                              const float* ybias, const float* gain, const float* beta,
                              const double* pec, const double* lo_ext, float pl2, void* out,
                              int64_t ldo, int64_t n, int d, double eps) {
    auto al = [](const void* p, int a) { return ((uintptr_t)p % a) == 0; };
    if (d % 4 || d > 128 || ldf % 4 || !al(F, 16)) return false;
    if (y && (ldy % 4 || !al(y, 8) || (ybias && !al(ybias, 16)))) return false;
    if (out && (ldo % 4 || !al(out, 8) || !al(gain, 16) || !al(beta, 16))) return false;
    // 8 lanes per row for the plain LayerNorm (measured: LN2 18.9 vs 21.2 us at
    // 100K rows); the PE variants keep 32 lanes (their 8-lane form needs 118
    // registers and measured slower, 21.3 vs 18.8 us)
    static const bool ln8 = !getenv("F3D_LN8") || getenv("F3D_LN8")[0] != '0';
    // LN1 + PE at d == 96: 8 lanes per row as well (row_ln8pe; F3D_LN8PE=0: 32 lanes)
    static const bool ln8pe = !getenv("F3D_LN8PE") || getenv("F3D_LN8PE")[0] != '0';
    if (ln8pe && d == 96 && pec && out) {
        using BF = __nv_bfloat16;
        const unsigned g8 = (unsigned)((n + 8 * 4 * stage::kRB8pe - 1) / (8 * 4 * stage::kRB8pe));
        if (y)
            (void)(f3d_launch(stage::row_ln8pe_kernel<true>, dim3(g8), dim3(stage::kThreads), 0,
                                      st, (float*)F, ldf, (const BF*)y, ldy, ybias, gain, beta, pec,
                                      lo_ext, pl2, (BF*)out, ldo, n, (float)eps));
        else
            (void)(f3d_launch(stage::row_ln8pe_kernel<false>, dim3(g8), dim3(stage::kThreads), 0,
                                      st, (float*)F, ldf, (const BF*)y, ldy, ybias, gain, beta, pec,
                                      lo_ext, pl2, (BF*)out, ldo, n, (float)eps));
        return true;
    }
    if (ln8 && d % 32 == 0 && d <= 128 && !pec) {
        using BF = __nv_bfloat16;
        const unsigned g8 = (unsigned)((n + 8 * 4 * stage::kRB8 - 1) / (8 * 4 * stage::kRB8));
        const float fe = (float)eps;
#define F3D_LN8V(V, HY, HO)                                                                       \
    f3d_launch(stage::row_ln8_kernel<V, HY, HO>, dim3(g8), dim3(stage::kThreads), 0, st,          \
               (float*)F, ldf, (const BF*)y, ldy, ybias, gain, beta, (BF*)out, ldo, n, d, fe)
#define F3D_LN8D(V)                                                                               \
    if (y && out) F3D_LN8V(V, true, true);                                                        \
    else if (y) F3D_LN8V(V, true, false);                                                         \
    else if (out) F3D_LN8V(V, false, true);
        switch (d / 32) {
            case 1: F3D_LN8D(1) break;
            case 2: F3D_LN8D(2) break;
            case 3: F3D_LN8D(3) break;
            default: F3D_LN8D(4) break;
        }
#undef F3D_LN8D
#undef F3D_LN8V
        return true;
    }
#ifndef F3D_LN_RPW
#define F3D_LN_RPW 4
#endif
    constexpr int RPW = F3D_LN_RPW;
    const unsigned g = (unsigned)((n + RPW * 8 - 1) / (RPW * 8));
    using BF = __nv_bfloat16;
    float* Ff = (float*)F;
    const BF* yb = (const BF*)y;
    BF* ob = (BF*)out;
    const float fe = (float)eps;
#define F3D_LNV(HY, HO, HP)                                                                       \
    f3d_launch(stage::row_ln_vec_kernel<RPW, HY, HO, HP>, dim3(g), dim3(stage::kThreads), 0, st, \
               Ff, ldf, yb, ldy, ybias, gain, beta, pec, lo_ext, pl2, ob, ldo, n, d, fe)
    if (y && out && pec) F3D_LNV(true, true, true);
    else if (y && out) F3D_LNV(true, true, false);
    else if (y) F3D_LNV(true, false, false);
    else if (out && pec) F3D_LNV(false, true, true);
    else if (out) F3D_LNV(false, true, false);
    else return true;
#undef F3D_LNV
    return true;
}

template <typename FT, typename OT, int PER>
static void launch_row_ln_p(unsigned g, cudaStream_t st, void* F, int64_t ldf, const void* y,
                            int64_t ldy, const float* ybias, const float* gain, const float* beta,
                            const double* pec, const double* lo_ext, float pl2, void* out,
                            int64_t ldo, int64_t n, int d, double eps) {
    stage::row_ln_kernel<FT, OT, PER><<<g, stage::kThreads, 0, st>>>(
        (FT*)F, ldf, (const __nv_bfloat16*)y, ldy, ybias, gain, beta, pec, lo_ext, pl2, (OT*)out,
        ldo, n, d, eps);
}

template <typename FT, typename OT>
static void launch_row_ln_o(unsigned g, cudaStream_t st, void* F, int64_t ldf, const void* y,
                            int64_t ldy, const float* ybias, const float* gain, const float* beta,
                            const double* pec, const double* lo_ext, float pl2, void* out,
                            int64_t ldo, int64_t n, int d, double eps) {
    const int per = (d + 31) / 32;
#define F3D_LN_CASE(P)                                                                          \
    case P:                                                                                     \
        launch_row_ln_p<FT, OT, P>(g, st, F, ldf, y, ldy, ybias, gain, beta, pec, lo_ext, pl2, \
                                   out, ldo, n, d, eps);                                        \
        break;
    switch (per) {
        F3D_LN_CASE(1) F3D_LN_CASE(2) F3D_LN_CASE(3) F3D_LN_CASE(4) F3D_LN_CASE(6)
        F3D_LN_CASE(8) F3D_LN_CASE(12) F3D_LN_CASE(16)
        default:
            if (per <= 5) launch_row_ln_p<FT, OT, 6>(g, st, F, ldf, y, ldy, ybias, gain, beta, pec, lo_ext, pl2, out, ldo, n, d, eps);
            else if (per <= 12) launch_row_ln_p<FT, OT, 12>(g, st, F, ldf, y, ldy, ybias, gain, beta, pec, lo_ext, pl2, out, ldo, n, d, eps);
            else if (per <= 16) launch_row_ln_p<FT, OT, 16>(g, st, F, ldf, y, ldy, ybias, gain, beta, pec, lo_ext, pl2, out, ldo, n, d, eps);
            else launch_row_ln_p<FT, OT, 32>(g, st, F, ldf, y, ldy, ybias, gain, beta, pec, lo_ext, pl2, out, ldo, n, d, eps);
    }
#undef F3D_LN_CASE
}

template <typename FT>
static void launch_row_ln(unsigned g, cudaStream_t st, void* F, int64_t ldf, const void* y,
                          int64_t ldy, const float* ybias, const float* gain, const float* beta,
                          const double* pec, const double* lo_ext, float pl2, void* out,
                          int out_kind, int64_t ldo, int64_t n, int d, double eps) {
    if (out_kind == 2)
        launch_row_ln_o<FT, double>(g, st, F, ldf, y, ldy, ybias, gain, beta, pec, lo_ext, pl2,
                                    out, ldo, n, d, eps);
    else if (out_kind == 1)
        launch_row_ln_o<FT, float>(g, st, F, ldf, y, ldy, ybias, gain, beta, pec, lo_ext, pl2,
                                   out, ldo, n, d, eps);
    else
        launch_row_ln_o<FT, __nv_bfloat16>(g, st, F, ldf, y, ldy, ybias, gain, beta, pec, lo_ext,
                                           pl2, out, ldo, n, d, eps);
}

extern "C" int f3d_row_ln(void* F, int f_is_f64, int64_t ldf, const void* y, int64_t ldy,
                          const float* ybias, const float* gain, const float* beta,
                          const double* pe_coords, const double* lo_ext, double pe_base,
                          void* out, int out_kind, int64_t ldo, int64_t n, int d, double eps,
                          void* stream) {
    if (d < 1 || d > 32 * stage::kMaxPerLane || n < 0 || out_kind < 0 || out_kind > 2)
        return F3D_ERR_CONFIG;
    if (pe_coords && (d % 6)) return F3D_ERR_CONFIG;
    const float pl2 = pe_coords ? (float)log2(pe_base) : 0.f;
    const double* pec = pe_coords;
    if (out && (!gain || !beta)) return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (!f_is_f64 && (out_kind == 0 || !out) &&
        launch_row_ln_vec(st, F, ldf, y, ldy, ybias, gain, beta, pec, lo_ext, pl2, out, ldo, n, d,
                          eps)) {
        F3D_LAUNCH_CHECK();
        return F3D_OK;
    }
    const unsigned g = (unsigned)((n + stage::kThreads / 32 - 1) / (stage::kThreads / 32));
    if (f_is_f64)
        launch_row_ln<double>(g, st, F, ldf, y, ldy, ybias, gain, beta, pec, lo_ext, pl2, out,
                              out_kind, ldo, n, d, eps);
    else
        launch_row_ln<float>(g, st, F, ldf, y, ldy, ybias, gain, beta, pec, lo_ext, pl2, out,
                             out_kind, ldo, n, d, eps);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

namespace f3d {
namespace stage {
__global__ void gelu_f64_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ y) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = x[i];
        y[i] = 0.5 * v * (1.0 + erf(v / sqrt(2.0)));
    }
}
}  // namespace stage
}  // namespace f3d

extern "C" int f3d_gelu_f64(const double* x, int64_t n, double* y, void* stream) {
    if (n < 0) return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    stage::gelu_f64_kernel<<<grid_for(n, stage::kThreads), stage::kThreads, 0,
                             (cudaStream_t)stream>>>(x, n, y);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

extern "C" int f3d_bias_gelu(void* u_bf16, int64_t n, int dh, const float* bias, void* stream) {
    if (dh < 2 || dh % 2 || n < 0) return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (dh % 8 == 0 && ((uintptr_t)u_bf16 & 15) == 0 && ((uintptr_t)bias & 15) == 0) {
        const int64_t n8 = n * dh / 8;
        const unsigned g = grid_for((n8 + 3) / 4, stage::kThreads);
        if (n8 < (int64_t)1 << 31)
            stage::bias_gelu8_kernel<uint32_t><<<g, stage::kThreads, 0, st>>>(
                (uint4*)u_bf16, (uint32_t)n8, dh / 8, (const float4*)bias);
        else
            stage::bias_gelu8_kernel<int64_t><<<g, stage::kThreads, 0, st>>>(
                (uint4*)u_bf16, n8, dh / 8, (const float4*)bias);
    } else {
        stage::bias_gelu_kernel<<<grid_for(n * dh / 2, stage::kThreads), stage::kThreads, 0, st>>>(
            (__nv_bfloat16*)u_bf16, n, dh, bias);
    }
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

extern "C" int f3d_scatter_ln_pe(const void* src, int src_is_f32, int64_t lds,
                                 const int32_t* dest, const double* coords, const double* lo_ext,
                                 double pe_base, const float* gain, const float* beta, float* F,
                                 int64_t ldf, void* out_bf16, int64_t ldo, int64_t n, int d,
                                 double eps, const int32_t* n_dev, void* stream) {
    auto al = [](const void* p, int a) { return ((uintptr_t)p % a) == 0; };
    if (d % 12 || d > 128 || n < 0 || ldf % 4 || ldo % 4 || lds % 4 || !al(F, 16) ||
        !al(out_bf16, 8) || !al(gain, 16) || !al(beta, 16) || !al(src, src_is_f32 ? 16 : 8))
        return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    constexpr int RPW = 4;
    const unsigned g = (unsigned)((n + RPW * 8 - 1) / (RPW * 8));
    const float pl2 = (float)log2(pe_base);
    cudaStream_t st = (cudaStream_t)stream;
    // d == 96: 8 lanes per row, the statistics of row_ln8pe (bit-identical to
    // the scatter followed by f3d_row_ln); F3D_LN8PE=0: 32 lanes
    static const bool ln8pe = !getenv("F3D_LN8PE") || getenv("F3D_LN8PE")[0] != '0';
    if (ln8pe && d == 96) {
        const unsigned g8 = (unsigned)((n + 8 * 4 * stage::kRB8pe - 1) / (8 * 4 * stage::kRB8pe));
        if (src_is_f32)
            F3D_CUDA_TRY(f3d_launch(stage::scatter_ln8pe_kernel<float>, dim3(g8), dim3(stage::kThreads),
                                    0, st, (const float*)src, lds, dest, coords, lo_ext, pl2, gain,
                                    beta, F, ldf, (__nv_bfloat16*)out_bf16, ldo, n, n_dev, (float)eps));
        else
            F3D_CUDA_TRY(f3d_launch(stage::scatter_ln8pe_kernel<__nv_bfloat16>, dim3(g8),
                                    dim3(stage::kThreads), 0, st, (const __nv_bfloat16*)src, lds, dest,
                                    coords, lo_ext, pl2, gain, beta, F, ldf, (__nv_bfloat16*)out_bf16,
                                    ldo, n, n_dev, (float)eps));
        return F3D_OK;
    }
    if (src_is_f32)
        F3D_CUDA_TRY(f3d_launch(stage::scatter_ln_pe_kernel<RPW, float>, dim3(g),
                                dim3(stage::kThreads), 0, st, (const float*)src, lds, dest, coords,
                                lo_ext, pl2, gain, beta, F, ldf, (__nv_bfloat16*)out_bf16, ldo, n,
                                n_dev, d, (float)eps));
    else
        F3D_CUDA_TRY(f3d_launch(stage::scatter_ln_pe_kernel<RPW, __nv_bfloat16>, dim3(g),
                                dim3(stage::kThreads), 0, st, (const __nv_bfloat16*)src, lds, dest,
                                coords, lo_ext, pl2, gain, beta, F, ldf, (__nv_bfloat16*)out_bf16,
                                ldo, n, n_dev, d, (float)eps));
    return F3D_OK;
}

extern "C" int f3d_residual_out(float* F, int64_t ldf, const void* y_bf16, int64_t ldy,
                                const float* ybias, void* out_bf16, int64_t ldo, int64_t n, int d,
                                void* stream) {
    if (d < 4 || d % 4 || n < 0 || ldf % 4 || ldy % 4 || ldo % 4 ||
        (((uintptr_t)F | (uintptr_t)ybias) & 15) || (((uintptr_t)y_bf16 | (uintptr_t)out_bf16) & 7))
        return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    const int64_t tot = n * (d / 4);
    const unsigned g = (unsigned)std::min<int64_t>((tot + 255) / 256, (int64_t)f3d_num_sms() * 16);
    F3D_CUDA_TRY(f3d_launch(stage::residual_out_kernel, dim3(g), dim3(256), 0, (cudaStream_t)stream,
                            F, ldf, (const __nv_bfloat16*)y_bf16, ldy, ybias,
                            (__nv_bfloat16*)out_bf16, ldo, n, d / 4));
    return F3D_OK;
}
