// Shared-load wavefronts per LDS.128 / LDS.64 for broadcast patterns
// (ncu: l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum per launch).
#include <cstdio>
#include <cuda_runtime.h>

template <int PAT, int W128>
__global__ void k_lds(double *out, int iters) {
    __shared__ __align__(16) double buf[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int row;
    switch (PAT) {
        case 0: row = 0; break;               // 1 unique
        case 1: row = lane >> 2; break;       // 8 unique, 4 lanes each (lanes 4r..4r+3)
        case 2: row = lane & 3; break;        // 4 unique, strided lanes
        case 3: row = lane >> 3; break;       // 4 unique, one per quarter-warp
        case 4: row = lane & 7; break;        // 8 unique, strided lanes
        case 5: row = lane; break;            // 32 unique
        default: row = lane >> 4; break;      // 2 unique
    }
    const int S = 102;  // row stride in doubles (S/2 odd)
    double acc = 0.0;
    const double *p = buf + row * S;
    for (int it = 0; it < iters; it++) {
        const int t = (it & 15) * 2;
        if (W128) {
            const double2 v = *reinterpret_cast<const double2 *>(p + t);
            acc += v.x + v.y;
        } else {
            acc += p[t];
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    double *out;
    cudaMalloc(&out, 148 * 256 * sizeof(double));
#define RUN(P, W) k_lds<P, W><<<148, 256>>>(out, 4096);
    RUN(0, 1) RUN(1, 1) RUN(2, 1) RUN(3, 1) RUN(4, 1) RUN(5, 1) RUN(6, 1)
    RUN(0, 0) RUN(1, 0) RUN(2, 0) RUN(3, 0) RUN(4, 0) RUN(5, 0) RUN(6, 0)
    cudaDeviceSynchronize();
    printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
