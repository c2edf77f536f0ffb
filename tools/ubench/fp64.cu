// FP64 FMA and fp32->fp64 conversion throughput per SM on this GPU (148 blocks x 256 threads, independent chains).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64 fp64.cu
#include <cstdio>

__global__ void k_dfma(int iters, double* out, unsigned long long* cyc) {
    double a[8];
    for (int u = 0; u < 8; ++u) a[u] = threadIdx.x * 1e-3 + u;
    const double b = 1.0000001, c = 1e-9;
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = fma(a[u], b, c);
    const unsigned long long t1 = clock64();
    double s = 0;
    for (int u = 0; u < 8; ++u) s += a[u];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_f2f(int iters, const float* in, double* out, unsigned long long* cyc) {
    float f[8];
    for (int u = 0; u < 8; ++u) f[u] = in[(threadIdx.x + u) & 255];
    double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < 8; ++u) { s[u] += (double)f[u]; f[u] = __int_as_float(__float_as_int(f[u]) ^ 1); }
    const unsigned long long t1 = clock64();
    double t = 0;
    for (int u = 0; u < 8; ++u) t += s[u];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    double* out; float* in; unsigned long long* cyc;
    cudaMalloc(&out, 8 * 148 * 256); cudaMalloc(&in, 4 * 256); cudaMalloc(&cyc, 8 * 148);
    cudaMemset(in, 0, 4 * 256);
    const int iters = 4096;
    unsigned long long h[148];
    for (int rep = 0; rep < 2; ++rep) {
        k_dfma<<<148, 256>>>(iters, out, cyc);
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, 8 * 148, cudaMemcpyDeviceToHost);
        printf("DFMA: %.1f FMA/clk/SM (%s)\n", 256.0 * 8 * iters / h[0], cudaGetErrorString(cudaGetLastError()));
        k_f2f<<<148, 256>>>(iters, in, out, cyc);
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, 8 * 148, cudaMemcpyDeviceToHost);
        printf("F2F.F64.F32 + DADD: %.1f per clk/SM\n", 256.0 * 8 * iters / h[0]);
    }
    return 0;
}
