// Grid-barrier latency on this GPU: cooperative-groups grid.sync() vs a sense-reversing barrier built from one
// global atomic counter (release/acquire).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gs gridsync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned long long* out) {
    cg::grid_group g = cg::this_grid();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}
__device__ __forceinline__ void bar_arrive_wait(unsigned* ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned v;
        asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(v) : "l"(ctr) : "memory");
        do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
    }
    __syncthreads();
}
__global__ void k_atom(int iters, unsigned* ctr, unsigned long long* out) {
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) bar_arrive_wait(ctr, (unsigned)(i + 1) * gridDim.x);
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}
int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d;
    unsigned* ctr;
    cudaMalloc(&d, 8);
    cudaMalloc(&ctr, 4);
    int iters = 2000;
    for (int rep = 0; rep < 2; ++rep) {
        void* a[] = {&iters, &d};
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)k_cg, sms, 256, a, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("cg grid.sync: %d blocks: %.3f us per barrier\n", sms, ms * 1e3 / iters);
        cudaMemset(ctr, 0, 4);
        void* b[] = {&iters, &ctr, &d};
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)k_atom, sms, 256, b, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("atomic barrier: %d blocks: %.3f us per barrier (%s)\n", sms, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
