// fp64 dependent-chain latency and throughput on this GPU (clock64 cycles).
#include <cstdio>
__global__ void lat(double* out, double a, double b, int n, long long* cyc) {
    double x = a, y = b;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        x = x * y; x = x * y; x = x * y; x = x * y;
        x = x * y; x = x * y; x = x * y; x = x * y;
    }
    long long t1 = clock64();
    double z = a;
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) {
        z = z + y; z = z + y; z = z + y; z = z + y;
        z = z + y; z = z + y; z = z + y; z = z + y;
    }
    long long t3 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t3 - t2; }
    out[threadIdx.x] = x + z;
}
__global__ void tput(double* out, double a, double b, int n, long long* cyc) {
    double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        x0 = x0 * b; x1 = x1 * b; x2 = x2 * b; x3 = x3 * b; x4 = x4 * b; x5 = x5 * b; x6 = x6 * b; x7 = x7 * b;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[2] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
    double* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMallocManaged(&cyc, 64);
    int n = 4096;
    lat<<<1, 32>>>(out, 1.0000001, 0.9999999, n, cyc); cudaDeviceSynchronize();
    lat<<<1, 32>>>(out, 1.0000001, 0.9999999, n, cyc); cudaDeviceSynchronize();
    printf("DMUL dep latency %.2f cyc, DADD dep latency %.2f cyc\n", (double)cyc[0] / (8.0 * n), (double)cyc[1] / (8.0 * n));
    for (int w : {1, 2, 4, 8, 16}) {
        tput<<<1, 32 * w>>>(out, 1.0, 0.9999999, n, cyc); cudaDeviceSynchronize();
        printf("1 SM, %2d warps: %.3f cyc per warp-DMUL per SM\n", w, (double)cyc[2] / (8.0 * n * w));
    }
    return 0;
}
