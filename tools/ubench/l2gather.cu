// The L2 ceiling of the gather passes (A2's (r, D) gathers, A5's D o X sigma gathers): how many random sectors per
// clock the chip serves, against the ~6300 B/clk streaming cap of B300_MICROARCH.md.  Each lane streams indices
// (coalesced int4 loads, as the column passes do) and gathers one EB-byte element per index from a table of TB
// megabytes (L2-resident), U gathers in flight per lane.  Index patterns: uniform random, and "columns" of a given
// density (sorted rows with a geometric gap, the shape of a Zipf column).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2gather l2gather.cu ; run: ./l2gather
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

template <int EB> struct Elt;
template <> struct Elt<8> { typedef double T; };
template <> struct Elt<16> { typedef double2 T; };
__device__ __forceinline__ double val(double x) { return x; }
__device__ __forceinline__ double val(double2 x) { return x.x + x.y; }

template <int EB, int U, bool CG>
__global__ void __launch_bounds__(256) k_gather(const int* __restrict__ idx, long long n, const typename Elt<EB>::T* __restrict__ tab,
                                                double* out) {
    typedef typename Elt<EB>::T T;
    double acc = 0.0;
    const long long stride = (long long)gridDim.x * blockDim.x * 4 * (U / 4);
    for (long long k = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4; k + stride * 0 < n; k += stride) {
        int q[U];
#pragma unroll
        for (int u = 0; u < U / 4; ++u) {
            const long long ku = k + (long long)u * gridDim.x * blockDim.x * 4;
            int4 v = ku + 3 < n ? *reinterpret_cast<const int4*>(idx + ku) : make_int4(0, 0, 0, 0);
            q[4 * u] = v.x; q[4 * u + 1] = v.y; q[4 * u + 2] = v.z; q[4 * u + 3] = v.w;
        }
        T g[U];
#pragma unroll
        for (int u = 0; u < U; ++u) g[u] = CG ? __ldcg(tab + q[u]) : __ldg(tab + q[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += val(g[u]);
    }
    if (acc == 12345.678) out[0] = acc;
}

// the same index stream, one 64-bit red.global.add per index (the X_A s reductions of the light columns)
template <int U>
__global__ void __launch_bounds__(256) k_red(const int* __restrict__ idx, long long n, unsigned long long* tab) {
    const long long stride = (long long)gridDim.x * blockDim.x * 4 * (U / 4);
    for (long long k = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4; k < n; k += stride) {
        int q[U];
#pragma unroll
        for (int u = 0; u < U / 4; ++u) {
            const long long ku = k + (long long)u * gridDim.x * blockDim.x * 4;
            int4 v = ku + 3 < n ? *reinterpret_cast<const int4*>(idx + ku) : make_int4(0, 0, 0, 0);
            q[4 * u] = v.x; q[4 * u + 1] = v.y; q[4 * u + 2] = v.z; q[4 * u + 3] = v.w;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            asm volatile("red.global.add.u64 [%0], %1;" ::"l"(tab + q[u]), "l"((unsigned long long)(q[u] + 1)) : "memory");
    }
}
static void run_red(const char* name, const int* d_idx, long long n, void* tab, int blocks_per_sm, double clk_ghz) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = 148 * blocks_per_sm;
    for (int w = 0; w < 2; ++w) k_red<8><<<grid, 256>>>(d_idx, n, (unsigned long long*)tab);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k_red<8><<<grid, 256>>>(d_idx, n, (unsigned long long*)tab);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double gps = n / (ms * 1e-3);
    printf("%-34s red.global.add.u64 blk/SM=%d : %7.3f ms  %7.1f G reds/s  %5.2f per SM clk\n", name, blocks_per_sm, ms, gps * 1e-9,
           gps / (148 * clk_ghz * 1e9));
}

template <int EB, int U, bool CG>
static void run(const char* name, const int* d_idx, long long n, const void* tab, double* out, int blocks_per_sm, double clk_ghz) {
    typedef typename Elt<EB>::T T;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = 148 * blocks_per_sm;
    for (int w = 0; w < 2; ++w) k_gather<EB, U, CG><<<grid, 256>>>(d_idx, n, (const T*)tab, out);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k_gather<EB, U, CG><<<grid, 256>>>(d_idx, n, (const T*)tab, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double gps = n / (ms * 1e-3);
    printf("%-34s EB=%2d U=%2d %s blk/SM=%d : %7.3f ms  %7.1f G gathers/s  %5.2f per SM clk  (idx stream %6.1f GB/s)\n", name, EB, U,
           CG ? "cg" : "nc", blocks_per_sm, ms, gps * 1e-9, gps / (148 * clk_ghz * 1e9), 4.0 * gps * 1e-9);
}

int main() {
    const long long n = 1LL << 26;   // 67 M gathers per launch
    int dev = 0, khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
    const double ghz = khz * 1e-6;
    std::vector<int> h(n);
    int* d_idx;
    void* tab;
    double* out;
    cudaMalloc(&d_idx, n * 4);
    cudaMalloc(&tab, 64 << 20);
    cudaMemset(tab, 0, 64 << 20);
    cudaMalloc(&out, 8);
    const int rows = 2000000;
    for (int pat = 0; pat < 4; ++pat) {
        uint64_t s = 88172645463325252ull;
        auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };
        const char* name;
        if (pat == 0) {
            name = "uniform random rows";
            for (long long k = 0; k < n; ++k) h[k] = (int)(rnd() % rows);
        } else {
            const double dens = pat == 1 ? 0.5 : pat == 2 ? 0.05 : 0.005;
            name = pat == 1 ? "sorted columns, density 0.5" : pat == 2 ? "sorted columns, density 0.05" : "sorted columns, density 0.005";
            const double il = 1.0 / log(1.0 - dens);   // geometric gaps between the rows of a column
            long long r = 0;
            for (long long k = 0; k < n; ++k) {
                const double u = ((rnd() >> 11) + 1) * (1.0 / 9007199254740993.0);
                r += 1 + (long long)(log(u) * il);
                if (r >= rows) r %= rows;   // (the next column)
                h[k] = (int)r;
            }
        }
        cudaMemcpy(d_idx, h.data(), n * 4, cudaMemcpyHostToDevice);
        run<8, 8, true>(name, d_idx, n, tab, out, 1, ghz);
        run<8, 8, true>(name, d_idx, n, tab, out, 4, ghz);
        run<8, 16, true>(name, d_idx, n, tab, out, 1, ghz);
        run<8, 16, true>(name, d_idx, n, tab, out, 4, ghz);
        run<8, 16, true>(name, d_idx, n, tab, out, 8, ghz);
        run<8, 8, false>(name, d_idx, n, tab, out, 4, ghz);
        run<16, 8, true>(name, d_idx, n, tab, out, 3, ghz);
        run<16, 8, false>(name, d_idx, n, tab, out, 3, ghz);
        run<16, 16, false>(name, d_idx, n, tab, out, 3, ghz);
        run<16, 8, false>(name, d_idx, n, tab, out, 6, ghz);
        run_red(name, d_idx, n, tab, 1, ghz);
        run_red(name, d_idx, n, tab, 4, ghz);
        run_red(name, d_idx, n, tab, 8, ghz);
    }
    return 0;
}
