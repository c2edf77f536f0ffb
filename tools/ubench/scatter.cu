// Cost of the small-m S phase (X_A s into a block-shared m-vector) for one block of 256 threads, chunks already in
// shared memory: (1) the k_inner loop (a __syncthreads per chunk), (2) the same without the per-chunk barrier
// (racy, timing only), (3) warps owning row ranges (no barrier; each warp locates its range in every chunk).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scatter scatter.cu
#include <cstdio>
#include <cstdlib>

constexpr int SCH = 2048, NCH = 5, M = 2000, UB = SCH / 256;

template <int MODE>
__global__ void __launch_bounds__(256, 1) k_sc(const int* __restrict__ gidx, const float* __restrict__ gval, int ncol_nnz, int reps,
                                               const double* coef, double* out, unsigned long long* cyc) {
    extern __shared__ __align__(16) unsigned char sm[];
    int* s_idx = reinterpret_cast<int*>(sm);
    float* s_val = reinterpret_cast<float*>(sm + 4 * NCH * SCH);
    double* xs = reinterpret_cast<double*>(sm + 8 * NCH * SCH);
    for (int k = threadIdx.x; k < NCH * SCH; k += blockDim.x) { s_idx[k] = gidx[k]; s_val[k] = gval[k]; }
    __syncthreads();
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long tot = 0;
    for (int rep = 0; rep < reps; ++rep) {
        for (int i = threadIdx.x; i < M; i += blockDim.x) xs[i] = 0.0;
        __syncthreads();
        const unsigned long long t0 = clock64();
        for (int c = 0; c < NCH; ++c) {
            const double cf = coef[c];
            const int* ci = s_idx + c * SCH;
            const float* cv = s_val + c * SCH;
            if (MODE == 3) {   // the k_inner shape: smem part [vb, kend), global tail [kend, ve)
                const int kend = ncol_nnz - (reps < 0 ? 1 : 0), ve = ncol_nnz;
                for (int k0 = threadIdx.x; k0 < ve; k0 += UB * (int)blockDim.x) {
                    int r[UB];
                    double xv[UB], a[UB];
#pragma unroll
                    for (int u = 0; u < UB; ++u) {
                        const int k = k0 + u * blockDim.x;
                        r[u] = -1;
                        if (k < kend) { r[u] = ci[k]; xv[u] = (double)cv[k]; }
                        else if (k < ve) { r[u] = __ldg(gidx + k); xv[u] = (double)__ldg(gval + k); }
                    }
#pragma unroll
                    for (int u = 0; u < UB; ++u) a[u] = r[u] >= 0 ? xs[r[u]] : 0.0;
#pragma unroll
                    for (int u = 0; u < UB; ++u)
                        if (r[u] >= 0) xs[r[u]] = fma(xv[u], cf, a[u]);
                }
                __syncthreads();
            } else if (MODE == 4) {   // smem part with float values converted after the loads; global tail apart
                const int kend = ncol_nnz - (reps < 0 ? 1 : 0), ve = ncol_nnz;
                for (int k0 = threadIdx.x; k0 < kend; k0 += UB * (int)blockDim.x) {
                    int r[UB];
                    float fv[UB];
                    double a[UB];
#pragma unroll
                    for (int u = 0; u < UB; ++u) {
                        const int k = k0 + u * blockDim.x;
                        const bool in = k < kend;
                        r[u] = in ? ci[k] : -1;
                        fv[u] = in ? cv[k] : 0.0f;
                    }
#pragma unroll
                    for (int u = 0; u < UB; ++u) a[u] = r[u] >= 0 ? xs[r[u]] : 0.0;
#pragma unroll
                    for (int u = 0; u < UB; ++u)
                        if (r[u] >= 0) xs[r[u]] = fma((double)fv[u], cf, a[u]);
                }
                for (int k = kend + threadIdx.x; k < ve; k += blockDim.x) {
                    const int rr = __ldg(gidx + k);
                    xs[rr] = fma((double)__ldg(gval + k), cf, xs[rr]);
                }
                __syncthreads();
            } else if (MODE <= 1) {
                for (int k0 = threadIdx.x; k0 < ncol_nnz; k0 += UB * (int)blockDim.x) {
                    int r[UB];
                    double xv[UB], a[UB];
#pragma unroll
                    for (int u = 0; u < UB; ++u) {
                        const int k = k0 + u * blockDim.x;
                        r[u] = -1;
                        if (k < ncol_nnz) { r[u] = ci[k]; xv[u] = (double)cv[k]; }
                    }
#pragma unroll
                    for (int u = 0; u < UB; ++u) a[u] = r[u] >= 0 ? xs[r[u]] : 0.0;
#pragma unroll
                    for (int u = 0; u < UB; ++u)
                        if (r[u] >= 0) xs[r[u]] = fma(xv[u], cf, a[u]);
                }
                if (MODE == 0) __syncthreads();
            } else {   // rows [lo, hi) of warp wid; chunk rows ascending: two ballot rounds find the start
                const int lo = wid * ((M + 7) / 8), hi = min(M, lo + (M + 7) / 8);
                const int seg = (ncol_nnz + 31) / 32;
                const int p = lane * seg;
                const int rv = p < ncol_nnz ? ci[p] : 0x7fffffff;
                const unsigned b = __ballot_sync(0xffffffffu, rv < lo);
                const int s0 = b ? (31 - __clz(b)) * seg : 0;   // last sample below lo
                int k = s0 + lane;
                unsigned bb = 0xffffffffu;
                // advance to the first element >= lo (within one segment)
                while (true) {
                    const int rr = k < ncol_nnz ? ci[k] : 0x7fffffff;
                    bb = __ballot_sync(0xffffffffu, rr < lo);
                    if (bb != 0xffffffffu) break;
                    k += 32;
                }
                k = k - lane + __popc(bb);
                for (k += lane; k < ncol_nnz; k += 32) {
                    const int rr = ci[k];
                    if (rr >= hi) break;
                    xs[rr] = fma((double)cv[k], cf, xs[rr]);
                }
            }
        }
        __syncthreads();
        tot += clock64() - t0;
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = tot / reps;
    for (int i = threadIdx.x; i < M; i += blockDim.x) out[(size_t)blockIdx.x * M + i] = xs[i];
}

int main() {
    int* hidx = (int*)malloc(4 * NCH * SCH);
    float* hval = (float*)malloc(4 * NCH * SCH);
    for (int c = 0; c < NCH; ++c)
        for (int k = 0; k < SCH; ++k) { hidx[c * SCH + k] = k < M ? k : 0; hval[c * SCH + k] = 1.0f + 0.001f * (k % 17); }
    int *gidx; float *gval; double *coef, *out; unsigned long long* cyc;
    cudaMalloc(&gidx, 4 * NCH * SCH); cudaMalloc(&gval, 4 * NCH * SCH);
    cudaMalloc(&coef, 8 * NCH); cudaMalloc(&out, 8 * 148 * M); cudaMalloc(&cyc, 8 * 148);
    cudaMemcpy(gidx, hidx, 4 * NCH * SCH, cudaMemcpyHostToDevice);
    cudaMemcpy(gval, hval, 4 * NCH * SCH, cudaMemcpyHostToDevice);
    double hc[NCH] = {0.5, -0.25, 0.125, 1.0, -2.0};
    cudaMemcpy(coef, hc, 8 * NCH, cudaMemcpyHostToDevice);
    const size_t smem = 8 * NCH * SCH + 8 * M;
    void (*ks[5])(const int*, const float*, int, int, const double*, double*, unsigned long long*) = {k_sc<0>, k_sc<1>, k_sc<2>, k_sc<3>, k_sc<4>};
    const char* names[5] = {"sync per chunk", "no sync (racy)", "row-owned warps", "k_inner shape", "split tail"};
    double ref = 0;
    for (int v = 0; v < 5; ++v) {
        cudaFuncSetAttribute(ks[v], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        ks[v]<<<148, 256, smem>>>(gidx, gval, M, 200, coef, out, cyc);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long hc2[148];
        double hout[M];
        cudaMemcpy(hc2, cyc, 8 * 148, cudaMemcpyDeviceToHost);
        cudaMemcpy(hout, out, 8 * M, cudaMemcpyDeviceToHost);
        double s = 0; for (int i = 0; i < M; ++i) s += hout[i];
        if (v == 0) ref = s;
        unsigned long long mx = 0, sm2 = 0;
        for (int b = 0; b < 148; ++b) { mx = hc2[b] > mx ? hc2[b] : mx; sm2 += hc2[b]; }
        printf("%-18s %s: cycles per 5-chunk S phase: avg %.0f max %llu  (%.2f us at 1965 MHz)  checksum %.6f (ref %.6f)\n",
               names[v], cudaGetErrorString(e), (double)sm2 / 148, mx, mx / 1965.0, s, ref);
    }
    return 0;
}
