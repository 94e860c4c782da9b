// Microbenchmark: per-SM throughput of the softmax instruction mix on sm_100a
// (elements per clock per SM): MUFU ex2 f32, ex2 bf16x2, 2- and 3-input fp32
// max, packed FFMA2, cvt f32x2 -> bf16x2.  One CTA of 512 threads per SM,
// 8 independent chains per thread.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o sfu_rate sfu_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096, kCh = 8;

template <int OP>
__global__ void k(float* out, long long* clk, float seed) {
    float v[kCh];
    uint32_t u[kCh];
#pragma unroll
    for (int c = 0; c < kCh; ++c) {
        v[c] = seed * (threadIdx.x + c) * 1e-7f - 3.f;
        u[c] = 0x3f80bf80u + c + threadIdx.x;
    }
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kCh; ++c) {
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[c]));
            if (OP == 1) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u[c]));
            if (OP == 2) asm volatile("max.f32 %0, %0, %1;" : "+f"(v[c]) : "f"(v[(c + 1) % kCh]));
            if (OP == 3) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(v[c]) : "f"(v[(c + 1) % kCh]), "f"(v[(c + 2) % kCh]));
            if (OP == 4) {
                uint64_t a;
                asm volatile("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(v[c]), "f"(v[(c + 1) % kCh]));
                asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(a));
                asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(v[c]), "=f"(v[(c + 1) % kCh]) : "l"(a));
            }
            if (OP == 5) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[c]) : "f"(v[c]), "f"(__uint_as_float(u[c])));
            if (OP == 6) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[c]));
        }
    }
    long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kCh; ++c) s += v[c] + __uint_as_float(u[c]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int elems_per_op) {
    float* o; long long* c;
    const int nb = 148, nt = 512;
    cudaMalloc(&o, nb * nt * 4); cudaMalloc(&c, nb * 8);
    k<OP><<<nb, nt>>>(o, c, 1.f);
    k<OP><<<nb, nt>>>(o, c, 1.f);
    long long h[148]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0; for (int i = 0; i < nb; ++i) mx = h[i] > mx ? h[i] : mx;
    const double ops = (double)nt * kIters * kCh;      // per SM
    printf("%-26s %7.2f ops/clk/SM  %7.2f elem/clk/SM (%s)\n", name, ops / mx, ops * elems_per_op / mx,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(o); cudaFree(c);
}

int main() {
    run<0>("ex2.approx.ftz.f32", 1);
    run<1>("ex2.approx.ftz.bf16x2", 2);
    run<6>("ex2.approx.f16x2", 2);
    run<2>("max.f32 (2-input)", 1);
    run<3>("max.f32 (3-input)", 2);
    run<4>("fma.rn.f32x2", 2);
    run<5>("cvt.rn.bf16x2.f32", 2);
    return 0;
}
