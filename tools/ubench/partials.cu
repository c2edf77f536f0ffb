// Cost of k_inner's block partials (12 values: warp shuffles, a barrier, the per-warp combine, a barrier) with a hot
// instruction cache, to compare with the in-kernel phase timers.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o partials partials.cu
#include <cstdio>

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
template <int N>
__device__ __forceinline__ void partials(const double (&v)[N], unsigned maxmask, double* sh_w, double* part, int slot0) {
    const int W = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const double t = ((maxmask >> k) & 1u) ? warp_max(v[k]) : warp_sum(v[k]);
        if (lane == 0) sh_w[wid * N + k] = t;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        double t = sh_w[k];
        for (int w = 1; w < W; ++w) {
            const double x = sh_w[w * N + k];
            t = ((maxmask >> k) & 1u) ? fmax(t, x) : t + x;
        }
        part[(size_t)(slot0 + k) * gridDim.x + blockIdx.x] = t;
        sh_w[8 * N + k] = t;
    }
    __syncthreads();
}
__global__ void __launch_bounds__(256, 1) k_part(int iters, const double* in, double* part, unsigned long long* cyc) {
    __shared__ double sh_w[8 * 12 + 12];
    double v[12];
    for (int k = 0; k < 12; ++k) v[k] = in[threadIdx.x] * (k + 1);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        partials<12>(v, (1u << 10) | (1u << 11), sh_w, part, 0);
        v[0] += sh_w[8 * 12 + 3] * 1e-30;
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
}
int main() {
    double *in, *part; unsigned long long* cyc;
    cudaMalloc(&in, 8 * 256); cudaMalloc(&part, 8 * 148 * 16); cudaMalloc(&cyc, 8 * 148);
    cudaMemset(in, 0, 8 * 256);
    unsigned long long h[148];
    for (int rep = 0; rep < 2; ++rep) {
        k_part<<<148, 256>>>(1000, in, part, cyc);
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, 8 * 148, cudaMemcpyDeviceToHost);
        printf("block partials<12>: %llu cycles per call (%.2f us at 1965 MHz) %s\n", h[0], h[0] / 1965.0,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
