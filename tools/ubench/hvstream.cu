// Streaming rate of the heavy-column path's chunk engine (ml_heavy.cuh) in isolation, on a synthetic S copy shaped
// like cfg 5's (130 M entries, rows of ~65 heavy entries, tiles of whole rows <= 4090 entries).  Per stage count:
// TMA ring only (wait + release), and the ring with hv_chunk's segmented reduction.  One block per SM, 256 threads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o hvstream hvstream.cu
#include <cstdio>
#include <vector>
#include <random>
#include "../../paper_1607_00315_b200/csrc/ml_heavy.cuh"
using namespace ml;

template <int STG, bool COMPUTE>
__global__ void __launch_bounds__(256, 1) k_stream(const HvChunk* chunks, int nch, const float* gv, const uint16_t* gk,
                                                   const int* offs, const uint16_t* blk, const double* sH,
                                                   double* Xh, unsigned long long* cyc) {
    extern __shared__ __align__(16) unsigned char sm[];
    double* s = reinterpret_cast<double*>(sm);
    unsigned char* ring = sm + HV_SRING_OFF;
    for (int i = threadIdx.x; i < HV_HMAX; i += blockDim.x) s[i] = sH[i];
    __syncthreads();
    const int2 rng = hv_my_chunks(chunks, nch);
    HvOpS<1> op{Xh, nullptr};
    const unsigned long long t0 = clock64();
    if (COMPUTE) {
        hv_stream<1>(chunks, rng.x, rng.y, gv, gk, offs, blk, HV_SRING_OFF, op, [](const HvChunk&) {});
    } else {
        uint64_t* bar = reinterpret_cast<uint64_t*>(ring + (size_t)STG * HV_STAGE);
        auto issue = [&](int c, int st) {
            const int a0 = chunks[c].e0 & ~15, a1 = (chunks[c].e1 + 15) & ~15;
            const int o0 = chunks[c].s0 & ~3, o1 = (chunks[c].s0 + chunks[c].ns + 4) & ~3;
            const uint32_t nn = (uint32_t)(a1 - a0), no = (uint32_t)(o1 - o0);
            mbar_arrive_expect_tx(bar + st, 6u * nn + 4u * no);
            bulk_g2s(ring + (size_t)st * HV_STAGE, gv + a0, 4u * nn, bar + st);
            bulk_g2s(ring + (size_t)st * HV_STAGE + HV_CAP * 4, gk + a0, 2u * nn, bar + st);
            bulk_g2s(ring + (size_t)st * HV_STAGE + HV_CAP * 6, offs + o0, 4u * no, bar + st);
        };
        if (threadIdx.x == 0) {
            for (int k = 0; k < STG; ++k) mbar_init(bar + k, 1);
            fence_mbar_init();
            for (int k = 0; k < STG && rng.x + k < rng.y; ++k) issue(rng.x + k, k);
        }
        __syncthreads();
        uint32_t phase = 0;
        for (int c = rng.x, st = 0; c < rng.y; ++c, st = (st + 1) % STG) {
            mbar_wait(bar + st, (phase >> st) & 1u);
            phase ^= 1u << st;
            __syncthreads();
            if (threadIdx.x == 0 && c + STG < rng.y) issue(c + STG, st);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(cyc, clock64() - t0);
}

template <int STG, bool COMPUTE>
void run(const HvChunk* ch, int nch, const float* v, const uint16_t* k, const int* offs, const uint16_t* blk,
         const double* sH, double* Xh, long long E, int sms) {
    auto kf = k_stream<STG, COMPUTE>;
    const size_t smem = HV_SRING_OFF + (size_t)(STG > HV_STG ? STG : HV_STG) * HV_STAGE + 64;
    cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    unsigned long long* cyc;
    cudaMalloc(&cyc, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(cyc, 0, 8);
        cudaEventRecord(e0);
        kf<<<sms, 256, smem>>>(ch, nch, v, k, offs, blk, sH, Xh, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    printf("stages %d compute %d: %.3f ms, %.0f GB/s (6 B per entry), err %s\n", STG, (int)COMPUTE, best,
           6.0 * E / best / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
    const int m = 2000000;
    const int rowlen = argc > 1 ? atoi(argv[1]) : 65;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    std::mt19937 rng(1);
    std::vector<int> rp(m + 1, 0);
    std::poisson_distribution<int> pois(rowlen);
    int mx = 0;
    for (int i = 0; i < m; ++i) { const int c = std::min(pois(rng), 8000); rp[i + 1] = rp[i] + c; mx = std::max(mx, c); }
    const long long E = rp[m];
    std::vector<float> v(E + 16, 1.0f);
    std::vector<uint16_t> k(E + 16, 0);
    const bool spread = argc > 2 ? atoi(argv[2]) != 0 : true;
    for (int i = 0; i < m; ++i) {   // random heavy ids per row, in bank-spread order (as the library's build writes them)
        std::vector<int> hs;
        for (int e = rp[i]; e < rp[i + 1]; ++e) hs.push_back((int)(rng() % HV_HMAX));
        int sz[16] = {0}, rk[16] = {0};
        for (int h : hs) sz[h & 15]++;
        (void)spread; (void)rk;
        for (size_t q = 0; q < hs.size(); ++q) k[hv_phys_i(rp[i] + (long long)q)] = (uint16_t)hs[q];
    }
    // chunks of whole rows (<= HV_CHMAX entries, <= HV_SMAX rows)
    std::vector<HvChunk> ch;
    for (int r = 0; r < m;) {
        const int r0 = r;
        while (r < m && rp[r + 1] - rp[r0] <= HV_CHMAX && r - r0 < HV_SMAX) ++r;
        ch.push_back(HvChunk{rp[r0], rp[r], r0, r0, r - r0, hv_lg(rp[r] - rp[r0], r - r0), 0, 0});
    }
    printf("entries %lld, max row %d, chunks %zu (avg %.0f entries), lg %d\n", E, mx, ch.size(), (double)E / ch.size(), ch[0].lg);
    HvChunk* dch; float* dv; uint16_t* dk; int* doff; double *dsH, *dXh;
    cudaMalloc(&dch, ch.size() * sizeof(HvChunk));
    cudaMalloc(&dv, v.size() * 4);
    cudaMalloc(&dk, k.size() * 2);
    cudaMalloc(&doff, (rp.size() + 8) * 4);
    cudaMalloc(&dsH, HV_HMAX * 8);
    cudaMalloc(&dXh, (size_t)m * 8);
    cudaMemcpy(dch, ch.data(), ch.size() * sizeof(HvChunk), cudaMemcpyHostToDevice);
    cudaMemcpy(dv, v.data(), v.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dk, k.data(), k.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(doff, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dsH, 0, HV_HMAX * 8);
    uint16_t* dblk;
    cudaMalloc(&dblk, ch.size() * 512);
    k_hv_blocks<<<592, 256>>>(dch, (int)ch.size(), doff, dblk);
    const int nch = (int)ch.size();
    run<2, false>(dch, nch, dv, dk, doff, dblk, dsH, dXh, E, sms);
    run<3, false>(dch, nch, dv, dk, doff, dblk, dsH, dXh, E, sms);
    run<4, false>(dch, nch, dv, dk, doff, dblk, dsH, dXh, E, sms);
    run<HV_STG, true>(dch, nch, dv, dk, doff, dblk, dsH, dXh, E, sms);
    return 0;
}
