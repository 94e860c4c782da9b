// Backward-pass kernels of the training step (the
// forward is bw/stage.py:134-158):
//   * LayerNorm backward fused with the residual add (row kernel, fp32);
//   * GELU backward with the bias gradient (erf form, fp32);
//   * column sums (bias gradients) with block partials + fp32 atomics;
//   * the softmax part of the attention backward on padded per-(scope, head)
//     score tiles: P = exp2(S*sl2 - lse) and dS = P (dP - D) * scale, fp32 GEMM
//     outputs in, bf16 GEMM operands out.
#include <cuda_bf16.h>

#include <algorithm>
#include <cfloat>

#include "f3d_common.cuh"

namespace f3d {
namespace train {

constexpr int kThreads = 256;
constexpr int kMaxPer = 16;   // d <= 512

__device__ __forceinline__ float ld_any(const void* p, int is_bf16, int64_t i) {
    return is_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i])
                   : reinterpret_cast<const float*>(p)[i];
}

// One warp per row, PER columns per lane (c = lane + 32 j).  x: LN input
// (fp32), dy: gradient of the LN output (bf16 or fp32), dres: residual
// gradient (nullable).  dx = dres + rstd * (g*dy - mean(g*dy) - xhat *
// mean(g*dy*xhat)); dgain += dy*xhat, dbeta += dy, accumulated per lane in
// registers over all rows of the warp and reduced once per block.
template <int PER>
__global__ void __launch_bounds__(kThreads) ln_bwd_kernel(
    const float* __restrict__ x, int64_t ldx, const void* __restrict__ dy, int dy_bf16,
    int64_t ldy, const float* __restrict__ gain, const float* __restrict__ dres, int64_t ldr,
    float* __restrict__ dx, int64_t ldd, float* __restrict__ dgain, float* __restrict__ dbeta,
    int64_t n, int d, float eps) {
    __shared__ float s_dg[kMaxPer * 32], s_db[kMaxPer * 32];
    for (int c = threadIdx.x; c < d; c += kThreads) s_dg[c] = s_db[c] = 0.f;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warps = kThreads / 32;
    float g[PER], adg[PER], adb[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int c = lane + 32 * j;
        g[j] = c < d ? gain[c] : 0.f;
        adg[j] = adb[j] = 0.f;
    }
    for (int64_t row = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5); row < n;
         row += (int64_t)gridDim.x * warps) {
        float xv[PER], gy[PER], yv[PER];
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int c = lane + 32 * j;
            xv[j] = c < d ? x[row * ldx + c] : 0.f;
            yv[j] = c < d ? ld_any(dy, dy_bf16, row * ldy + c) : 0.f;
            gy[j] = yv[j] * g[j];
            s += xv[j];
        }
        const float mean = warp_sum(s) / d;
        float q = 0.f;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int c = lane + 32 * j;
            const float t = c < d ? xv[j] - mean : 0.f;
            q += t * t;
        }
        const float rstd = rsqrtf(warp_sum(q) / d + eps);
        float a = 0.f, b = 0.f;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            xv[j] = (xv[j] - mean) * rstd;            // xhat
            a += gy[j];
            b += gy[j] * xv[j];
        }
        a = warp_sum(a) / d;
        b = warp_sum(b) / d;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int c = lane + 32 * j;
            if (c >= d) continue;
            float v = rstd * (gy[j] - a - xv[j] * b);
            if (dres) v += dres[row * ldr + c];
            dx[row * ldd + c] = v;
            adg[j] = fmaf(yv[j], xv[j], adg[j]);
            adb[j] += yv[j];
        }
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int c = lane + 32 * j;
        if (c < d) {
            atomicAdd(&s_dg[c], adg[j]);
            atomicAdd(&s_db[c], adb[j]);
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += kThreads) {
        if (dgain) atomicAdd(dgain + c, s_dg[c]);
        if (dbeta) atomicAdd(dbeta + c, s_db[c]);
    }
}

// Phi(z) = 0.5 (1 + erf(z / sqrt2)) with the forward's Abramowitz-Stegun
// 7.1.26 erf (|err| <= 1.5e-7); phi(z) = exp(-z^2/2) / sqrt(2 pi).
__device__ __forceinline__ float gelu_grad(float z) {
    const float a = fabsf(z) * 0.70710678118654752f;
    const float t = __frcp_rn(fmaf(0.3275911f, a, 1.f));
    float pl = fmaf(1.061405429f, t, -1.453152027f);
    pl = fmaf(pl, t, 1.421413741f);
    pl = fmaf(pl, t, -0.284496736f);
    pl = fmaf(pl, t, 0.254829592f);
    const float ez = __expf(-a * a);                 // = exp(-z^2/2)
    const float erf_a = 1.f - pl * t * ez;
    const float Phi = 0.5f * (1.f + copysignf(erf_a, z));
    return Phi + z * (0.3989422804014327f * ez);
}

// du = dg * GELU'(u + b); dbias += du.  Blocks stride over rows; thread t
// owns the column pairs t, t + blockDim, ... (coalesced bf16x2 / float2 row
// accesses, bias partials in shared memory without atomics).  h even.
__global__ void __launch_bounds__(kThreads) gelu_bwd_kernel(
    const __nv_bfloat16* __restrict__ u, int64_t ldu, const float* __restrict__ bias,
    const float* __restrict__ dg, int64_t ldg, float* __restrict__ du, int64_t ldd,
    float* __restrict__ dbias, int64_t n, int h) {
    extern __shared__ float s_db[];
    const int h2 = h / 2;
    for (int c = threadIdx.x; c < h2; c += blockDim.x) s_db[2 * c] = s_db[2 * c + 1] = 0.f;
    for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
        for (int c = threadIdx.x; c < h2; c += blockDim.x) {
            const float2 uu = __bfloat1622float2(
                reinterpret_cast<const __nv_bfloat162*>(u + r * ldu)[c]);
            const float2 bb = reinterpret_cast<const float2*>(bias)[c];
            const float2 gg = reinterpret_cast<const float2*>(dg + r * ldg)[c];
            float2 v;
            v.x = gg.x * gelu_grad(uu.x + bb.x);
            v.y = gg.y * gelu_grad(uu.y + bb.y);
            reinterpret_cast<float2*>(du + r * ldd)[c] = v;
            s_db[2 * c] += v.x;
            s_db[2 * c + 1] += v.y;
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < h; c += blockDim.x) atomicAdd(dbias + c, s_db[c]);
}

// out[c] += sum_r x[r, c]  (x bf16 or fp32)
__global__ void __launch_bounds__(kThreads) colsum_kernel(const void* __restrict__ x, int is_bf16,
                                                          int64_t ldx, int64_t n, int d,
                                                          float* __restrict__ out) {
    const int c = blockIdx.y * kThreads + threadIdx.x;
    if (c >= d) return;
    float s = 0.f;
    for (int64_t r = blockIdx.x; r < n; r += gridDim.x) s += ld_any(x, is_bf16, r * ldx + c);
    atomicAdd(out + c, s);
}

// Padded score tiles [B, M, M] (row-major, B = scopes x heads); len[b] real
// rows/keys.  T: fp32 GEMM output, out: bf16 operand of the next GEMM.
// mode 0: out = P = exp2(T*sl2 - lse[b,i]);  mode 1 (T = dP, P = mode-0 out):
// out = dS = P (dP - D[b,i]) * scale.  Zero outside len.  Eight elements per
// thread (M % 8 == 0): 32 B fp32 loads, 16 B bf16 stores.
__global__ void __launch_bounds__(kThreads) softmax_bwd_kernel(
    const float* __restrict__ T, const __nv_bfloat16* __restrict__ P,
    const float* __restrict__ rowv, const int32_t* __restrict__ len, int B, int M, float sl2,
    float scale, int mode, __nv_bfloat16* __restrict__ out) {
    const int64_t tot8 = (int64_t)B * M * M / 8;
    const int M8 = M / 8;
    for (int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x; t < tot8;
         t += (int64_t)gridDim.x * kThreads) {
        const int64_t bi = t / M8;           // (b, i)
        const int j0 = (int)(t - bi * M8) * 8;
        const int b = (int)(bi / M);
        const int i = (int)(bi - (int64_t)b * M);
        const int m = len[b];
        uint4 o = make_uint4(0, 0, 0, 0);
        if (i < m && j0 < m) {
            const float4 a = reinterpret_cast<const float4*>(T)[2 * t];
            const float4 c = reinterpret_cast<const float4*>(T)[2 * t + 1];
            float v[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
            const float r = rowv[bi];
            float p[8];
            if (mode == 1) {
                const uint4 pp = reinterpret_cast<const uint4*>(P)[t];
                const __nv_bfloat162* ph = reinterpret_cast<const __nv_bfloat162*>(&pp);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f = __bfloat1622float2(ph[e]);
                    p[2 * e] = f.x;
                    p[2 * e + 1] = f.y;
                }
            }
            __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float x0, x1;
                if (mode == 0) {
                    x0 = exp2f(fmaf(v[2 * e], sl2, -r));
                    x1 = exp2f(fmaf(v[2 * e + 1], sl2, -r));
                } else {
                    x0 = p[2 * e] * (v[2 * e] - r) * scale;
                    x1 = p[2 * e + 1] * (v[2 * e + 1] - r) * scale;
                }
                if (j0 + 2 * e >= m) x0 = 0.f;
                if (j0 + 2 * e + 1 >= m) x1 = 0.f;
                oh[e] = __floats2bfloat162_rn(x0, x1);
            }
        }
        reinterpret_cast<uint4*>(out)[t] = o;
    }
}

// mode 1 with D computed in-kernel: one warp per (b, i) row, D = sum_j P dP
// over the same bf16 P the product uses (so sum_j dS = 0 in this arithmetic:
// the stable choice when dP - D cancels), then dS = P (dP - D) * scale.
__global__ void __launch_bounds__(kThreads) softmax_bwd_rows_kernel(
    const float* __restrict__ T, const __nv_bfloat16* __restrict__ P,
    const int32_t* __restrict__ len, int B, int M, float scale, __nv_bfloat16* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t rows = (int64_t)B * M;
    for (int64_t bi = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5; bi < rows;
         bi += ((int64_t)gridDim.x * kThreads) >> 5) {
        const int b = (int)(bi / M);
        const int i = (int)(bi - (int64_t)b * M);
        const int m = len[b];
        const float* tr = T + bi * M;
        const __nv_bfloat16* pr = P + bi * M;
        uint4* orow = reinterpret_cast<uint4*>(out + bi * M);
        float acc = 0.f;
        if (i < m) {
            for (int j0 = lane * 8; j0 < m; j0 += 256) {
                const uint4 pp = *reinterpret_cast<const uint4*>(pr + j0);
                const float4 a = *reinterpret_cast<const float4*>(tr + j0);
                const float4 c = *reinterpret_cast<const float4*>(tr + j0 + 4);
                const float v[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
                const __nv_bfloat162* ph = reinterpret_cast<const __nv_bfloat162*>(&pp);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f = __bfloat1622float2(ph[e]);
                    if (j0 + 2 * e < m) acc = fmaf(f.x, v[2 * e], acc);
                    if (j0 + 2 * e + 1 < m) acc = fmaf(f.y, v[2 * e + 1], acc);
                }
            }
        }
        const float D = warp_sum(acc);
        for (int j0 = lane * 8; j0 < M; j0 += 256) {
            uint4 o = make_uint4(0, 0, 0, 0);
            if (i < m && j0 < m) {
                const uint4 pp = *reinterpret_cast<const uint4*>(pr + j0);
                const float4 a = *reinterpret_cast<const float4*>(tr + j0);
                const float4 c = *reinterpret_cast<const float4*>(tr + j0 + 4);
                const float v[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
                const __nv_bfloat162* ph = reinterpret_cast<const __nv_bfloat162*>(&pp);
                __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f = __bfloat1622float2(ph[e]);
                    float x0 = f.x * (v[2 * e] - D) * scale, x1 = f.y * (v[2 * e + 1] - D) * scale;
                    if (j0 + 2 * e >= m) x0 = 0.f;
                    if (j0 + 2 * e + 1 >= m) x1 = 0.f;
                    oh[e] = __floats2bfloat162_rn(x0, x1);
                }
            }
            orow[j0 / 8] = o;
        }
    }
}

}  // namespace train
}  // namespace f3d

using namespace f3d;

static unsigned grid_cap(int64_t work, int threads, int per_sm = 8) {
    int64_t g = (work + threads - 1) / threads;
    const int64_t cap = (int64_t)f3d_num_sms() * per_sm;
    if (g > cap) g = cap;
    return (unsigned)(g < 1 ? 1 : g);
}

extern "C" int f3d_ln_bwd(const float* x, int64_t ldx, const void* dy, int dy_bf16, int64_t ldy,
                          const float* gain, const float* dres, int64_t ldr, float* dx,
                          int64_t ldd, float* dgain, float* dbeta, int64_t n, int d, double eps,
                          void* stream) {
    if (n < 0 || d < 1 || d > 32 * train::kMaxPer) return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    const int per = (d + 31) / 32;
    const unsigned grid = grid_cap(n * 32, train::kThreads, 4);
    cudaStream_t st = (cudaStream_t)stream;
#define F3D_LNB(P)                                                                             \
    train::ln_bwd_kernel<P><<<grid, train::kThreads, 0, st>>>(x, ldx, dy, dy_bf16, ldy, gain,  \
                                                              dres, ldr, dx, ldd, dgain, dbeta, \
                                                              n, d, (float)eps)
    if (per <= 1) F3D_LNB(1);
    else if (per <= 2) F3D_LNB(2);
    else if (per <= 3) F3D_LNB(3);
    else if (per <= 4) F3D_LNB(4);
    else if (per <= 8) F3D_LNB(8);
    else F3D_LNB(16);
#undef F3D_LNB
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

extern "C" int f3d_gelu_bwd(const void* u_bf16, int64_t ldu, const float* bias, const float* dg,
                            int64_t ldg, float* du, int64_t ldd, float* dbias, int64_t n, int h,
                            void* stream) {
    if (n < 0 || h < 2 || h % 2 || h > 8192 || ldu % 2 || ldg % 2 || ldd % 2)
        return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    // one column pair per thread when h/2 <= 256 (h = 384: 192 threads)
    const int threads = std::min(train::kThreads, ((h / 2 + 31) / 32) * 32);
    train::gelu_bwd_kernel<<<grid_cap(n, 1, 8), threads, h * sizeof(float),
                             (cudaStream_t)stream>>>((const __nv_bfloat16*)u_bf16, ldu, bias, dg,
                                                     ldg, du, ldd, dbias, n, h);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

extern "C" int f3d_colsum(const void* x, int is_bf16, int64_t ldx, int64_t n, int d, float* out,
                          void* stream) {
    if (n < 0 || d < 1) return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    dim3 grid((unsigned)std::min<int64_t>(n, 1024), (unsigned)((d + train::kThreads - 1) / train::kThreads));
    train::colsum_kernel<<<grid, train::kThreads, 0, (cudaStream_t)stream>>>(x, is_bf16, ldx, n, d,
                                                                            out);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

extern "C" int f3d_softmax_bwd(const float* T, const void* P, const float* rowv,
                               const int32_t* len, int B, int M, double scale_log2, double scale,
                               int mode, void* out, void* stream) {
    if (B < 0 || M < 8 || M % 8 || mode < 0 || mode > 1 || (mode == 1 && !P))
        return F3D_ERR_CONFIG;
    if (B == 0) return F3D_OK;
    if (mode == 1 && !rowv) {
        train::softmax_bwd_rows_kernel<<<grid_cap((int64_t)B * M * 32, train::kThreads, 16),
                                         train::kThreads, 0, (cudaStream_t)stream>>>(
            T, (const __nv_bfloat16*)P, len, B, M, (float)scale, (__nv_bfloat16*)out);
        F3D_LAUNCH_CHECK();
        return F3D_OK;
    }
    train::softmax_bwd_kernel<<<grid_cap((int64_t)B * M * M / 8, train::kThreads, 16),
                                train::kThreads, 0, (cudaStream_t)stream>>>(
        T, (const __nv_bfloat16*)P, rowv, len, B, M, (float)scale_log2, (float)scale, mode,
        (__nv_bfloat16*)out);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}
