// Backward-pass kernels of the training step (the
// forward is bw/stage.py:134-158):
//   * LayerNorm backward fused with the residual add (row kernel, fp32);
//   * GELU backward with the bias gradient (erf form, fp32);
//   * column sums (bias gradients) with block partials + fp32 atomics;
//   * the softmax part of the attention backward on padded per-(scope, head)
//     score tiles: P = exp2(S*sl2 - lse) and dS = P (dP - D) * scale, in place.
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

// One warp per row.  x: LN input (fp32), dy: gradient of the LN output
// (bf16 or fp32), dres: residual gradient (nullable).  dx = dres + rstd *
// (g*dy - mean(g*dy) - xhat * mean(g*dy*xhat)); dgain += dy*xhat, dbeta += dy.
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
    for (int64_t row = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5); row < n;
         row += (int64_t)gridDim.x * warps) {
        float xv[kMaxPer], gy[kMaxPer], yv[kMaxPer];
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < kMaxPer; ++j) {
            const int c = lane + 32 * j;
            xv[j] = c < d ? x[row * ldx + c] : 0.f;
            yv[j] = c < d ? ld_any(dy, dy_bf16, row * ldy + c) : 0.f;
            gy[j] = c < d ? yv[j] * gain[c] : 0.f;
            s += xv[j];
        }
        const float mean = warp_sum(s) / d;
        float q = 0.f;
#pragma unroll
        for (int j = 0; j < kMaxPer; ++j) {
            const int c = lane + 32 * j;
            const float t = c < d ? xv[j] - mean : 0.f;
            q += t * t;
        }
        const float rstd = rsqrtf(warp_sum(q) / d + eps);
        float a = 0.f, b = 0.f;
#pragma unroll
        for (int j = 0; j < kMaxPer; ++j) {
            xv[j] = (xv[j] - mean) * rstd;            // xhat
            a += gy[j];
            b += gy[j] * xv[j];
        }
        a = warp_sum(a) / d;
        b = warp_sum(b) / d;
#pragma unroll
        for (int j = 0; j < kMaxPer; ++j) {
            const int c = lane + 32 * j;
            if (c >= d) continue;
            float v = rstd * (gy[j] - a - xv[j] * b);
            if (dres) v += dres[row * ldr + c];
            dx[row * ldd + c] = v;
            atomicAdd(&s_dg[c], yv[j] * xv[j]);
            atomicAdd(&s_db[c], yv[j]);
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += kThreads) {
        if (dgain) atomicAdd(dgain + c, s_dg[c]);
        if (dbeta) atomicAdd(dbeta + c, s_db[c]);
    }
}

// du = dg * GELU'(u + b), GELU'(z) = Phi(z) + z phi(z); dbias += du (columns).
__global__ void __launch_bounds__(kThreads) gelu_bwd_kernel(
    const __nv_bfloat16* __restrict__ u, int64_t ldu, const float* __restrict__ bias,
    const float* __restrict__ dg, int64_t ldg, float* __restrict__ du, int64_t ldd,
    float* __restrict__ dbias, int64_t n, int h) {
    extern __shared__ float s_db[];
    for (int c = threadIdx.x; c < h; c += kThreads) s_db[c] = 0.f;
    __syncthreads();
    const int64_t tot = n * h;
    for (int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * kThreads) {
        const int64_t r = t / h;
        const int c = (int)(t - r * h);
        const float z = __bfloat162float(u[r * ldu + c]) + bias[c];
        const float phi = 0.3989422804014327f * __expf(-0.5f * z * z);
        const float Phi = 0.5f * (1.f + erff(z * 0.70710678118654752f));
        const float v = dg[r * ldg + c] * (Phi + z * phi);
        du[r * ldd + c] = v;
        atomicAdd(&s_db[c], v);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < h; c += kThreads) atomicAdd(dbias + c, s_db[c]);
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
// rows/keys.  mode 0: S -> P = exp2(S*sl2 - lse[b,i]) (0 outside len);
// mode 1: dP -> dS = P (dP - D[b,i]) * scale.
__global__ void __launch_bounds__(kThreads) softmax_bwd_kernel(
    float* __restrict__ T, const float* __restrict__ P, const float* __restrict__ rowv,
    const int32_t* __restrict__ len, int B, int M, float sl2, float scale, int mode) {
    const int64_t tot = (int64_t)B * M * M;
    for (int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * kThreads) {
        const int64_t bi = t / M;            // (b, i)
        const int j = (int)(t - bi * M);
        const int b = (int)(bi / M);
        const int i = (int)(bi - (int64_t)b * M);
        const int m = len[b];
        if (i >= m || j >= m) {
            T[t] = 0.f;
            continue;
        }
        if (mode == 0) T[t] = exp2f(T[t] * sl2 - rowv[bi]);
        else T[t] = P[t] * (T[t] - rowv[bi]) * scale;
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
    train::ln_bwd_kernel<<<grid_cap(n * 32, train::kThreads), train::kThreads, 0,
                           (cudaStream_t)stream>>>(x, ldx, dy, dy_bf16, ldy, gain, dres, ldr, dx,
                                                   ldd, dgain, dbeta, n, d, (float)eps);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}

extern "C" int f3d_gelu_bwd(const void* u_bf16, int64_t ldu, const float* bias, const float* dg,
                            int64_t ldg, float* du, int64_t ldd, float* dbias, int64_t n, int h,
                            void* stream) {
    if (n < 0 || h < 1 || h > 8192) return F3D_ERR_CONFIG;
    if (n == 0) return F3D_OK;
    train::gelu_bwd_kernel<<<grid_cap(n * h, train::kThreads), train::kThreads, h * sizeof(float),
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

extern "C" int f3d_softmax_bwd(float* T, const float* P, const float* rowv, const int32_t* len,
                               int B, int M, double scale_log2, double scale, int mode,
                               void* stream) {
    if (B < 0 || M < 1 || mode < 0 || mode > 1) return F3D_ERR_CONFIG;
    if (B == 0) return F3D_OK;
    train::softmax_bwd_kernel<<<grid_cap((int64_t)B * M * M, train::kThreads, 32),
                                train::kThreads, 0, (cudaStream_t)stream>>>(
        T, P, rowv, len, B, M, (float)scale_log2, (float)scale, mode);
    F3D_LAUNCH_CHECK();
    return F3D_OK;
}
