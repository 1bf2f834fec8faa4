#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dadd(double* out, double a, double b, int n, long long* cyc) {
    double x = a;
    long long t0 = clock64();
    #pragma unroll 1
    for (int i = 0; i < n; ++i) {
        x = x + b; x = x + b; x = x + b; x = x + b; x = x + b; x = x + b; x = x + b; x = x + b;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_dmul(double* out, double a, double b, int n, long long* cyc) {
    double x = a;
    long long t0 = clock64();
    #pragma unroll 1
    for (int i = 0; i < n; ++i) {
        x = x * b; x = x * b; x = x * b; x = x * b; x = x * b; x = x * b; x = x * b; x = x * b;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_dfma(double* out, double a, double b, int n, long long* cyc) {
    double x = a;
    long long t0 = clock64();
    #pragma unroll 1
    for (int i = 0; i < n; ++i) {
        x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a);
        x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_fadd(float* out, float a, float b, int n, long long* cyc) {
    float x = a;
    long long t0 = clock64();
    #pragma unroll 1
    for (int i = 0; i < n; ++i) {
        x = x + b; x = x + b; x = x + b; x = x + b; x = x + b; x = x + b; x = x + b; x = x + b;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_shfl(double* out, double a, int n, long long* cyc) {
    double x = a + threadIdx.x;
    long long t0 = clock64();
    #pragma unroll 1
    for (int i = 0; i < n; ++i) {
        x = __shfl_up_sync(0xffffffffu, x, 1); x = __shfl_up_sync(0xffffffffu, x, 1);
        x = __shfl_up_sync(0xffffffffu, x, 1); x = __shfl_up_sync(0xffffffffu, x, 1);
        x = __shfl_up_sync(0xffffffffu, x, 1); x = __shfl_up_sync(0xffffffffu, x, 1);
        x = __shfl_up_sync(0xffffffffu, x, 1); x = __shfl_up_sync(0xffffffffu, x, 1);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double* d; float* f; long long* c; long long h;
    cudaMalloc(&d, 1024 * 8); cudaMalloc(&f, 1024 * 4); cudaMalloc(&c, 8);
    const int n = 4096;
    for (int w = 1; w <= 32; w *= 32) {
        k_dadd<<<1, 32 * w>>>(d, 1.0, 1e-9, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("warps %d DADD %.1f cyc\n", w, double(h) / (8.0 * n));
        k_dmul<<<1, 32 * w>>>(d, 1.0, 1.0000001, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("warps %d DMUL %.1f cyc\n", w, double(h) / (8.0 * n));
        k_dfma<<<1, 32 * w>>>(d, 1.0, 0.5, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("warps %d DFMA %.1f cyc\n", w, double(h) / (8.0 * n));
        k_fadd<<<1, 32 * w>>>(f, 1.0f, 1e-9f, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("warps %d FADD %.1f cyc\n", w, double(h) / (8.0 * n));
        k_shfl<<<1, 32 * w>>>(d, 1.0, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("warps %d SHFL64 %.1f cyc\n", w, double(h) / (8.0 * n));
    }
    return 0;
}
