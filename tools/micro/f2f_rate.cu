// Issue rates of F2F.F64.F32 vs DADD/DMUL (per SM per clock, from clock64()).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_cvt(const float *in, double *out, long long *cyc, int iters) {
    float f[8];
    for (int i = 0; i < 8; i++) f[i] = in[(threadIdx.x + i) & 255];
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            acc[i] = acc[i] + (double)f[i];  // F2F + DADD (+ FADD)
            f[i] = f[i] + 1.0f;
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; i++) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_cvtonly(const float *in, double *out, long long *cyc, int iters) {
    float f[8];
    for (int i = 0; i < 8; i++) f[i] = in[(threadIdx.x + i) & 255];
    unsigned long long x[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            x[i] ^= (unsigned long long)__double_as_longlong((double)f[i]);
            f[i] = f[i] + 1.0f;
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; i++) s += (double)x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_dadd(const float *in, double *out, long long *cyc, int iters) {
    double f[8];
    for (int i = 0; i < 8; i++) f[i] = in[(threadIdx.x + i) & 255];
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            acc[i] = acc[i] + f[i];
            f[i] = f[i] * 1.0000001;
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; i++) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    float *in;
    double *out;
    long long *cyc, h[148];
    cudaMalloc(&in, 256 * 4);
    cudaMemset(in, 0, 256 * 4);
    cudaMalloc(&out, 148 * 1024 * 8);
    cudaMalloc(&cyc, 148 * 8);
    const int iters = 4096;
    for (int rep = 0; rep < 2; rep++) {
        k_cvt<<<148, 1024>>>(in, out, cyc, iters);
        cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
        // per SM: 1024 threads x iters x 8 (F2F + DADD)
        printf("cvt+dadd: %.2f lane-ops/clk/SM each\n", 1024.0 * iters * 8 / h[0]);
        k_cvtonly<<<148, 1024>>>(in, out, cyc, iters);
        cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
        printf("cvt (+fadd+2 lop): %.2f lane-ops/clk/SM\n", 1024.0 * iters * 8 / h[0]);
        k_dadd<<<148, 1024>>>(in, out, cyc, iters);
        cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
        printf("dadd+dmul: %.2f lane-ops/clk/SM each\n", 1024.0 * iters * 8 / h[0]);
    }
    return 0;
}
