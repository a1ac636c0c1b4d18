// Does a warp shuffle occupy the L1 data pipe?  Two kernels with the same
// dependency structure: a chain of 64-bit shuffles vs a chain of 64-bit
// shared-memory store+load pairs.  Profile with
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,gpu__time_duration.sum
#include <cstdio>
__global__ void k_shfl(double* out, int iters) {
    double v = threadIdx.x * 1.0;
    for (int i = 0; i < iters; ++i) {
        v = v + __shfl_up_sync(0xffffffffu, v, 1);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = v;
}
__global__ void k_smem(double* out, int iters) {
    __shared__ double s[256];
    double v = threadIdx.x * 1.0;
    for (int i = 0; i < iters; ++i) {
        s[threadIdx.x] = v;
        __syncwarp();
        v = v + s[threadIdx.x ^ 1];
        __syncwarp();
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = v;
}
int main() {
    double* o;
    cudaMalloc(&o, 148 * 8 * 256 * sizeof(double));
    for (int r = 0; r < 2; ++r) {
        k_shfl<<<148 * 8, 256>>>(o, 4096);
        k_smem<<<148 * 8, 256>>>(o, 4096);
    }
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    cudaEventRecord(a); k_shfl<<<148 * 8, 256>>>(o, 4096); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("shfl %.3f ms\n", ms);
    cudaEventRecord(a); k_smem<<<148 * 8, 256>>>(o, 4096); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("smem %.3f ms\n", ms);
    return 0;
}
