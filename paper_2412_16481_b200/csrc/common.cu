// Library-wide state: error text, device properties.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "f3d_common.cuh"

static thread_local char g_last_error[512] = "";

void f3d_set_last_cuda_error(cudaError_t e) {
    snprintf(g_last_error, sizeof(g_last_error), "CUDA error %d: %s", (int)e,
             cudaGetErrorString(e));
}

bool f3d_pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("F3D_PDL");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

int f3d_num_sms() {
    static int sms[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (sms[dev] == 0) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        sms[dev] = v > 0 ? v : 148;
    }
    return sms[dev];
}

extern "C" int f3d_abi_version(void) { return 1; }

extern "C" const char* f3d_last_error(void) { return g_last_error; }

__global__ void f3d_zero_i32_kernel(int32_t* p, int64_t n) {
    f3d::pdl_wait();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = 0;
}

// two small ranges in one launch (a cooperative kernel's barrier word and its
// status words)
__global__ void f3d_zero_i32x2_kernel(int32_t* p, int n, int32_t* q, int m) {
    f3d::pdl_wait();
    const int i = threadIdx.x;
    if (i < n) p[i] = 0;
    if (q && i < m) q[i] = 0;
}

cudaError_t f3d_zero_i32x2(int32_t* p, int n, int32_t* q, int m, cudaStream_t st) {
    return f3d_launch(f3d_zero_i32x2_kernel, dim3(1), dim3(32), 0, st, p, n, q, m);
}

cudaError_t f3d_zero_i32(int32_t* p, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    int64_t g = (n + 255) / 256;
    if (g > 1024) g = 1024;
    return f3d_launch(f3d_zero_i32_kernel, dim3((unsigned)g), dim3(256), 0, st, p, n);
}
