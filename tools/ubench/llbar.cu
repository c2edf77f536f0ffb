// A grid barrier that carries the block totals with it ("payload barrier"), against cg grid.sync() followed by a
// separate read of the block partials (what k_inner does now).  Every block publishes N doubles, each as two 64-bit
// words (32-bit half of the value | 32-bit tag); a block has passed the barrier once it has read every block's words
// with the current tag.  The publisher fences (release) before its tagged stores and the reader fences (acquire)
// after its tagged loads, so all writes a block made before the barrier are visible to every block after it.  Two
// alternating buffers: a block is at most one barrier ahead of the slowest.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o llbar llbar.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr int N = 12, GMAX = 160;
#ifndef BACKOFF
#define BACKOFF 100
#endif

__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// buf: [2][N][2][G] words.  mine: this block's N totals (shared).  out: the N grid totals (shared), block order.
__device__ void ll_barrier(const double* mine, unsigned long long* buf, unsigned tag, double* out) {
    const int G = gridDim.x, wid = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
    unsigned long long* B = buf + (size_t)(tag & 1u) * N * 2 * G;
    __syncthreads();   // every thread's earlier writes precede the publication
    if (threadIdx.x == 0) {
        __threadfence();   // release (cumulative over the block's writes ordered by the barrier)
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const unsigned long long bits = (unsigned long long)__double_as_longlong(mine[k]);
            st_relaxed(B + ((size_t)k * 2 + 0) * G + blockIdx.x, (bits & 0xffffffff00000000ull) | tag);
            st_relaxed(B + ((size_t)k * 2 + 1) * G + blockIdx.x, (bits << 32) | tag);
        }
    }
    if (wid < N) {   // warp w polls slots w and w + W of every block (5 blocks per lane) together
        unsigned long long w[2][5][2];
        while (true) {
            bool ok = true;
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                const int k = wid + s2 * W;
#pragma unroll
                for (int j = 0; j < 5; ++j) {
                    const int b = lane + 32 * j;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        w[s2][j][h] = (b < G && k < N) ? ld_relaxed(B + ((size_t)k * 2 + h) * G + b) : (unsigned long long)tag;
                        ok &= (unsigned)(w[s2][j][h] & 0xffffffffu) == tag;
                    }
                }
            }
            if (__all_sync(0xffffffffu, ok)) break;
            if (BACKOFF) __nanosleep(BACKOFF);
        }
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
            const int k = wid + s2 * W;
            double t = 0.0;
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                const int b = lane + 32 * j;
                const unsigned long long bits = (w[s2][j][0] & 0xffffffff00000000ull) | (w[s2][j][1] >> 32);
                if (b < G) t += __longlong_as_double((long long)bits);
            }
            t = warp_sum(t);
            if (lane == 0 && k < N) out[k] = t;
        }
        if (lane == 0) __threadfence();   // acquire
    }
    __syncthreads();
}

__global__ void k_ll(int iters, unsigned long long* buf, double* data, unsigned tag0, unsigned long long* cyc, int* bad) {
    __shared__ double mine[N], out[N];
    const int G = gridDim.x;
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x < N) mine[threadIdx.x] = (double)((blockIdx.x + 1) * (threadIdx.x + 1) + i);
        if (threadIdx.x == 0) data[blockIdx.x] = (double)i;   // a plain write the barrier must order
        ll_barrier(mine, buf, tag0 + (unsigned)i, out);
        if (threadIdx.x < N) {
            const double want = (double)(threadIdx.x + 1) * G * (G + 1) / 2 + (double)i * G;
            if (out[threadIdx.x] != want) atomicOr(bad, 1);
        }
        if (threadIdx.x == 0 && data[(blockIdx.x + 1) % G] < (double)i) atomicOr(bad, 2);   // ordering check
        __syncthreads();
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = (clock64() - t0) / iters;
}
__global__ void k_cgtot(int iters, double* part, unsigned long long* cyc) {
    cg::grid_group g = cg::this_grid();
    __shared__ double out[N];
    const int G = gridDim.x, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x < N) part[(size_t)threadIdx.x * G + blockIdx.x] = (double)(blockIdx.x + i);
        g.sync();
        for (int k = wid; k < N; k += 8) {
            double t = 0.0;
            for (int j = 0; j < 5; ++j) { const int b = lane + 32 * j; if (b < G) t += __ldcg(part + (size_t)k * G + b); }
            t = warp_sum(t);
            if (lane == 0) out[k] = t;
        }
        __syncthreads();
        part[GMAX * N + blockIdx.x] = out[0];
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = (clock64() - t0) / iters;
}
int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *buf, *cyc; double *data, *part; int* bad;
    cudaMalloc(&buf, 8 * 2 * N * 2 * GMAX); cudaMalloc(&cyc, 8 * GMAX); cudaMalloc(&data, 8 * GMAX);
    cudaMalloc(&part, 8 * (GMAX * N + GMAX)); cudaMalloc(&bad, 4);
    cudaMemset(buf, 0, 8 * 2 * N * 2 * GMAX); cudaMemset(bad, 0, 4); cudaMemset(data, 0, 8 * GMAX);
    int iters = 2000;
    unsigned tag0 = 1;
    unsigned long long h[GMAX];
    for (int rep = 0; rep < 2; ++rep) {
        void* a[] = {&iters, &buf, &data, &tag0, &cyc, &bad};
        cudaLaunchCooperativeKernel((void*)k_ll, sms, 256, a, 0, 0);
        cudaError_t e = cudaDeviceSynchronize();
        int hb = 0;
        cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost);
        printf("payload barrier (12 totals): %llu cycles = %.2f us per barrier, bad=%d (%s)\n", h[0], h[0] / 1965.0, hb,
               cudaGetErrorString(e));
        tag0 += iters;
        void* b[] = {&iters, &part, &cyc};
        cudaLaunchCooperativeKernel((void*)k_cgtot, sms, 256, b, 0, 0);
        e = cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost);
        printf("cg grid.sync + totals (12): %llu cycles = %.2f us per barrier (%s)\n", h[0], h[0] / 1965.0,
               cudaGetErrorString(e));
    }
    return 0;
}
