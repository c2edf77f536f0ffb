// ml_heavy.cuh — the heavy-column path of the large-m inner solver (A5: X_A s and H sigma = X_A^T D X_A sigma,
// PAPER.md P:793; DESIGN section 8.2 "heavy columns").
//
// On the Zipf designs (cfg 3-5) a few thousand columns hold most of X's nonzeros (cfg 5: the 8192 longest columns
// hold 65 % of 2e8), and they are the columns of every free set.  Through the column units of k_inner their X_A s
// products are fp64 reductions into global memory and their H sigma products are 8-byte L2 gathers of D o X sigma:
// both bound by L2 operations, not by HBM.  Here the heavy set H (at most HV_HMAX columns, the longest, chosen once
// at ml_create) gets two extra copies of its nonzeros (fp32 value + 16-bit index, 6 bytes), each ordered so that
// the vector it multiplies sits in shared memory:
//   * S copy (row-major): the heavy entries of each row, index = h.  s_H (the direction on H, HV_HMAX doubles) is
//     staged in shared memory; every row's sum is written once (Xh): no atomics.
//   * G copy ("band CSC"): rows cut into bands of HV_RB rows; within a band the heavy entries ordered by (h, row),
//     index = row - band row0.  D o X sigma of one band sits in shared memory; every (band, h) segment sum is written
//     once to hpart[h * nb + band]; the owner of position h sums its nb band partials in band order.
// Heavy ids h are assigned by decreasing column length, so the segments of a band come longest first and a chunk
// holds segments of similar length.  Both copies are cut into chunks (S: whole rows; G: whole segments) of at most
// HV_CHMAX entries and HV_SMAX segments, streamed by one thread of the block with TMA bulk copies through a
// HV_STG-stage ring together with the chunk's slice of segment offsets (S: the heavy row pointers; G: the (band, h)
// segment starts).  Groups of L = 2^lg lanes (lg fixed per chunk from its mean segment length) take the segments in
// turn, each lane summing every L-th entry, then a fixed shuffle tree; chunks of a few long segments are reduced by
// the whole block, one segment at a time.  Every result is a fixed-order sum: bitwise reproducible.
#pragma once
#include "ml_common.cuh"

namespace ml {

constexpr int HV_HMAX = 8192;              // heavy columns at most (s_H: 64 KB of shared memory)
constexpr int HV_CAP = 4096;               // entries per ring stage
constexpr int HV_CHMAX = HV_CAP - 32;      // entries per chunk (its span of whole 16-entry blocks is <= HV_CAP)
constexpr int HV_SMAX = 1024;              // segments per chunk
constexpr int HV_OFFCAP = HV_SMAX + 8;     // offsets per stage (the chunk's HV_SMAX + 1, from a 16-byte boundary)
constexpr int HV_RB = HV_CHMAX;            // rows per band of the G copy (16-bit row index; a segment fits a chunk)
constexpr int HV_STG = 3;                  // ring stages (two chunks in flight while one is reduced)
constexpr int HV_MINLEN = 32;              // shortest heavy column
constexpr int HV_W = 8;                    // warps per block (k_inner)
constexpr int HV_LGBLK = 8;                // lg of a chunk reduced by the whole block, segment by segment
constexpr size_t HV_STAGE = (size_t)HV_CAP * 6 + (size_t)HV_OFFCAP * 4 + 512;   // values, indices, offsets, block segs
// dynamic shared memory of the sub-phases (they alias the column rings of k_inner)
constexpr size_t HV_SH_OFF = 0;                                            // S: s_H
constexpr size_t HV_ZH_OFF = (size_t)8 * HV_HMAX;                          // S: zeroing bits of H
constexpr size_t HV_SRING_OFF = HV_ZH_OFF + (size_t)4 * (HV_HMAX / 32);    // S: the ring
constexpr size_t HV_U_OFF = 0;                                             // G: D o X sigma of the band
constexpr size_t HV_GRING_OFF = 32768;                                     // G: the ring
constexpr size_t HV_RING_BYTES = (size_t)HV_STG * HV_STAGE + 8 * HV_STG;
static_assert((size_t)8 * HV_RB <= HV_GRING_OFF, "band vector");
static_assert(HV_SRING_OFF % 16 == 0 && HV_STAGE % 16 == 0, "ring alignment");
__host__ __device__ constexpr size_t hv_smem_bytes() {
    return (HV_SRING_OFF + HV_RING_BYTES) > (HV_GRING_OFF + HV_RING_BYTES) ? HV_SRING_OFF + HV_RING_BYTES
                                                                        : HV_GRING_OFF + HV_RING_BYTES;
}

// a chunk: entries [e0, e1) of a copy; its ns segments start at offsets[s0 .. s0 + ns] (absolute entry indices);
// base: first row (S; segment j is row base + j) or band (G; segment j is heavy column h0 + j)
struct HvChunk { int e0, e1, base, s0, ns, lg, h0, pad; };

// the heavy path's device state (Prm::hv)
struct HvPrm {
    int on;                 // built (m > SMALL_M, enough heavy nonzeros)
    int nh;                 // |H|
    int nb;                 // bands of the G copy
    int nts, ncg;           // S chunks, G chunks
    int mode;               // 0: per relaxation (nnz(A ∩ H) >= frac nnz(H)), 1: always, 2: never (ml_set_engine)
    double frac;
    long long nnzh;         // nonzeros of H
    const int* hid;         // [n] heavy id of column j, or -1
    const float* sval; const uint16_t* sidx; const int* soff; const HvChunk* schunk;   // S copy, row starts [m + 1]
    const float* gval; const uint16_t* gidx; const int* goff; const HvChunk* gchunk;   // G copy, starts [nb nh + 1]
    const uint16_t* sblk; const uint16_t* gblk;   // [chunks][256]: the segment (within its chunk) of each block's
                                                  // first entry
    double* sH;             // [HV_HMAX] the S coefficient of each heavy column of A this iteration (0 elsewhere)
    uint32_t* zH;           // [HV_HMAX / 32] its zeroing flags (the snap path's z = s on those columns)
    double* Xh; double* Xhz;   // [m] X_H s_H, X_H z_H
    double* hpart;          // [nh * nb] band partials of H sigma
    int* phid;              // [n] heavy id of free-set position p this relaxation (-1: light)
};

// The dynamic shared memory of the calling kernel (every extern __shared__ array names the same base): the ring and
// the ops' vectors are addressed through it, so that the out-of-line hv_stream still emits shared loads.
extern __shared__ __align__(16) unsigned char hv_dyn[];

// ------------------------------------------------------------------ one chunk: its segments, by groups of L lanes
// Both copies are stored swizzled in 16-entry blocks so that thread t, reading the 16 entries of block q = its
// global block index with 16-byte shared loads, hits distinct banks in every quarter warp: the values' 4-entry
// quarter j sits at quarter (j + (q >> 1)) & 3, the indices' 8-entry half j at half j ^ ((q >> 2) & 1).
__host__ __device__ __forceinline__ long long hv_phys_v(long long e) {
    return (e & ~15LL) | ((((e >> 2) + (e >> 5)) & 3) << 2) | (e & 3);
}
__host__ __device__ __forceinline__ long long hv_phys_i(long long e) {
    return (e & ~15LL) | ((((e >> 3) ^ (e >> 6)) & 1) << 3) | (e & 7);
}
// Per-thread ranges: thread t reduces the 16 entries of stage block t (the chunk's entries [v0, v1) of the stage,
// which starts at global entry eb = e0 & ~15).  Its products are summed per piece of segment, in entry order: a
// segment inside the range is written at once; a segment crossing ranges leaves its parts in shared slots (tail
// part tp of the thread where it starts, whole ranges wp, head part hp of the thread where it ends), which the
// ending thread adds in thread order after a barrier.
template <int NV> struct HvPart { double tp[NV][256]; double wp[NV][256]; };
template <int NV, class Op>
__device__ __forceinline__ void hv_ranges(const float* sv, const uint16_t* si, const int* so, const uint16_t* sbk,
                                          const HvChunk& ch, const Op& op, HvPart<NV>& pt) {
    const int t = threadIdx.x;
    const int eb = ch.e0 & ~15, v0 = ch.e0 - eb, v1 = ch.e1 - eb, ob = ch.s0 & 3;
    const int q = (eb >> 4) + t;
    const int lo = max(16 * t, v0), hi = min(16 * t + 16, v1);
    double p[16][NV];
    if (lo < hi) {
        float x[16];
        uint32_t ix[16];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float4 v = *reinterpret_cast<const float4*>(sv + 16 * t + 4 * ((j + (q >> 1)) & 3));
            x[4 * j] = v.x; x[4 * j + 1] = v.y; x[4 * j + 2] = v.z; x[4 * j + 3] = v.w;
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const uint4 v = *reinterpret_cast<const uint4*>(si + 16 * t + 8 * (j ^ ((q >> 2) & 1)));
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) { ix[8 * j + 2 * u] = w[u] & 0xFFFFu; ix[8 * j + 2 * u + 1] = w[u] >> 16; }
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) op.prod(ix[e], x[e], p[e]);
        for (int k = sbk[t]; k < ch.ns; ++k) {   // my segments, from the one holding my first entry
            const int sb = so[ob + k] - eb, se = so[ob + k + 1] - eb;
            if (sb >= hi) break;
            const int ps = max(sb, lo) - 16 * t, pe = min(se, hi) - 16 * t;
            double a[NV];
#pragma unroll
            for (int q2 = 0; q2 < NV; ++q2) a[q2] = 0.0;
#pragma unroll
            for (int e = 0; e < 16; ++e)
                if (e >= ps && e < pe) {
#pragma unroll
                    for (int q2 = 0; q2 < NV; ++q2) a[q2] += p[e][q2];
                }
            const bool before = sb < lo, after = se > hi;
            if (!before && !after) {
                if (se > sb) op.out(ch, k, a);
            } else if (before && after) {
#pragma unroll
                for (int q2 = 0; q2 < NV; ++q2) pt.wp[q2][t] = a[q2];
            } else if (after) {
#pragma unroll
                for (int q2 = 0; q2 < NV; ++q2) pt.tp[q2][t] = a[q2];
            } else {   // the head part of a segment that started in an earlier range: kept until after the barrier
#pragma unroll
                for (int q2 = 0; q2 < NV; ++q2) p[0][q2] = a[q2];   // (this is my first piece: p[0] is free again)
            }
        }
    }
    __syncthreads();
    if (lo < hi) {
        // the segment holding my first entry, if it started before me and ends in my range
        const int k = sbk[t];
        const int sb = so[ob + k] - eb, se = so[ob + k + 1] - eb;
        if (sb < lo && se <= hi) {
            const int ts = sb >> 4;   // the range where it starts
            double a[NV];
#pragma unroll
            for (int q2 = 0; q2 < NV; ++q2) a[q2] = pt.tp[q2][ts];
            for (int u = ts + 1; u < t; ++u) {
#pragma unroll
                for (int q2 = 0; q2 < NV; ++q2) a[q2] = a[q2] + pt.wp[q2][u];
            }
#pragma unroll
            for (int q2 = 0; q2 < NV; ++q2) a[q2] = a[q2] + p[0][q2];   // my part, kept in p[0]
            op.out(ch, k, a);
        }
    }
}
// sv/si: the stage's entries from e0 & ~15; so: its offsets from s0 & ~3 (absolute entry indices)
template <int NV, class Op>
__device__ __forceinline__ void hv_segments(const float* sv, const uint16_t* si, const int* so, const uint16_t* sbk,
                                            const HvChunk& ch, const Op& op, double* wsum, HvPart<NV>& pt) {
    const int eb = ch.e0 & ~15, ob = ch.s0 & 3;
    if (ch.lg == HV_LGBLK) {   // a few long segments: the whole block on each, in turn
        const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int k = 0; k < ch.ns; ++k) {
            const int b = so[ob + k] - eb, e = so[ob + k + 1] - eb;
            double acc[NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) acc[q] = 0.0;
            for (int i = b + (int)threadIdx.x; i < e; i += 2048) {   // 8 entries in flight, summed in order
                float x[8];
                uint32_t ix[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int t = i + 256 * u;
                    const bool ok = t < e;
                    x[u] = ok ? sv[hv_phys_v(eb + t) - eb] : 0.0f;
                    ix[u] = ok ? si[hv_phys_i(eb + t) - eb] : 0u;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (i + 256 * u < e) op.fma(ix[u], x[u], acc);
            }
#pragma unroll
            for (int q = 0; q < NV; ++q) acc[q] = warp_sum(acc[q]);
            double* ws = wsum + (k & 1) * NV * HV_W;   // (double-buffered: one barrier per segment)
            if (lane == 0) {
#pragma unroll
                for (int q = 0; q < NV; ++q) ws[q * HV_W + w] = acc[q];
            }
            __syncthreads();
            if (threadIdx.x == 0 && e > b) {
                double v[NV];
#pragma unroll
                for (int q = 0; q < NV; ++q) {
                    v[q] = ws[q * HV_W];
                    for (int u = 1; u < HV_W; ++u) v[q] = v[q] + ws[q * HV_W + u];
                }
                op.out(ch, k, v);
            }
        }
        return;
    }
    hv_ranges<NV>(sv, si, so, sbk, ch, op, pt);
}

// Stream chunks [c0, c1) through the block's TMA ring (thread 0 issues; every thread reduces).  on_chunk(ch) runs
// block-uniformly before a chunk is reduced (it may stage data, with its own barriers).
// (out of line: called once per sub-phase, so that its loop gets registers of its own instead of k_inner's spills)
template <int NV, class Op, class OnChunk>
__device__ __noinline__ void hv_stream(const HvChunk* chunks, int c0, int c1, const float* gv, const uint16_t* gi,
                                       const int* goff, const uint16_t* gblk, size_t ring_off, Op op, OnChunk on_chunk) {
    __shared__ double wsum[2 * NV * HV_W];
    __shared__ HvPart<NV> pt;
    unsigned char* ring = hv_dyn + ring_off;   // (a shared address the compiler can see)
    uint64_t* bar = reinterpret_cast<uint64_t*>(ring + (size_t)HV_STG * HV_STAGE);
    auto sval = [&](int st) { return reinterpret_cast<float*>(ring + (size_t)st * HV_STAGE); };
    auto sidx = [&](int st) { return reinterpret_cast<uint16_t*>(ring + (size_t)st * HV_STAGE + (size_t)HV_CAP * 4); };
    auto soff = [&](int st) { return reinterpret_cast<int*>(ring + (size_t)st * HV_STAGE + (size_t)HV_CAP * 6); };
    auto sblk = [&](int st) {
        return reinterpret_cast<uint16_t*>(ring + (size_t)st * HV_STAGE + (size_t)HV_CAP * 6 + (size_t)HV_OFFCAP * 4);
    };
    auto issue = [&](int c, int st) {
        const int e0 = __ldg(&chunks[c].e0), e1 = __ldg(&chunks[c].e1);
        const int s0 = __ldg(&chunks[c].s0), ns = __ldg(&chunks[c].ns);
        const int a0 = e0 & ~15, a1 = (e1 + 15) & ~15;
        const int o0 = s0 & ~3, o1 = (s0 + ns + 1 + 3) & ~3;
        const uint32_t n = (uint32_t)(a1 - a0), no = (uint32_t)(o1 - o0);
        mbar_arrive_expect_tx(bar + st, 6u * n + 4u * no + 512u);
        bulk_g2s(sval(st), gv + a0, 4u * n, bar + st);
        bulk_g2s(sidx(st), gi + a0, 2u * n, bar + st);
        bulk_g2s(soff(st), goff + o0, 4u * no, bar + st);
        bulk_g2s(sblk(st), gblk + (size_t)c * 256, 512u, bar + st);
    };
    if (threadIdx.x == 0) {
        for (int k = 0; k < HV_STG; ++k) mbar_init(bar + k, 1);
        fence_mbar_init();
        for (int k = 0; k < HV_STG && c0 + k < c1; ++k) issue(c0 + k, k);
    }
    __syncthreads();
    uint32_t phase = 0u;
    for (int c = c0, st = 0; c < c1; ++c, st = (st + 1) % HV_STG) {
        HvChunk ch;
        {
            const int4 a = __ldg(reinterpret_cast<const int4*>(chunks + c));
            const int4 b = __ldg(reinterpret_cast<const int4*>(chunks + c) + 1);
            ch = HvChunk{a.x, a.y, a.z, a.w, b.x, b.y, b.z, 0};
        }
        on_chunk(ch);
        mbar_wait(bar + st, (phase >> st) & 1u);
        phase ^= 1u << st;
        hv_segments<NV>(sval(st), sidx(st), soff(st), sblk(st), ch, op, wsum, pt);
        __syncthreads();   // stage st consumed
        if (threadIdx.x == 0 && c + HV_STG < c1) issue(c + HV_STG, st);
    }
    if (threadIdx.x == 0)
        for (int k = 0; k < HV_STG; ++k) mbar_inval(bar + k);
    __syncthreads();
}
// chunks [c0, c1) of block b: those starting in its share of the entries (balanced by nonzeros)
__device__ __forceinline__ int hv_chunk_lb(const HvChunk* chunks, int nch, long long target) {
    int lo = 0, hi = nch;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((long long)__ldg(&chunks[mid].e0) >= target) hi = mid; else lo = mid + 1;
    }
    return lo;
}
__device__ __forceinline__ int2 hv_my_chunks(const HvChunk* chunks, int nch) {
    if (nch == 0) return make_int2(0, 0);
    const long long e0 = __ldg(&chunks[0].e0), e1 = __ldg(&chunks[nch - 1].e1);
    const long long T = (e1 - e0 + gridDim.x - 1) / gridDim.x;
    const int c0 = hv_chunk_lb(chunks, nch, e0 + (long long)blockIdx.x * T);
    const int c1 = blockIdx.x + 1 == gridDim.x ? nch : hv_chunk_lb(chunks, nch, e0 + (long long)(blockIdx.x + 1) * T);
    return make_int2(c0, c1);
}

// S: row sums of the heavy entries times s_H (and z_H = s_H on the zeroing columns): Xh[row]
template <int NV> struct HvOpS {
    double* Xh; double* Xhz;
    __device__ __forceinline__ void prod(uint32_t h, float x, double (&p)[NV]) const {
        h &= HV_HMAX - 1;   // (entries outside the chunk hold stale indices; their products are discarded)
        const double v = (double)x * reinterpret_cast<const double*>(hv_dyn + HV_SH_OFF)[h];
        p[0] = v;
        if constexpr (NV == 2)
            p[1] = ((reinterpret_cast<const uint32_t*>(hv_dyn + HV_ZH_OFF)[h >> 5] >> (h & 31)) & 1u) ? v : 0.0;
    }
    __device__ __forceinline__ void fma(uint32_t h, float x, double (&a)[NV]) const {
        const double s = reinterpret_cast<const double*>(hv_dyn + HV_SH_OFF)[h];
        a[0] = ::fma((double)x, s, a[0]);
        if constexpr (NV == 2) {
            const bool z = (reinterpret_cast<const uint32_t*>(hv_dyn + HV_ZH_OFF)[h >> 5] >> (h & 31)) & 1u;
            a[1] = ::fma((double)x, z ? s : 0.0, a[1]);
        }
    }
    __device__ __forceinline__ void out(const HvChunk& ch, int k, const double (&v)[NV]) const {
        Xh[ch.base + k] = v[0];
        if constexpr (NV == 2) Xhz[ch.base + k] = v[1];
    }
};
// G: (band, h) sums of the heavy entries times u = D o X sigma of the band: hpart[h nb + band]
struct HvOpG {
    double* hpart;
    int nb;
    __device__ __forceinline__ void prod(uint32_t r, float x, double (&p)[1]) const {
        p[0] = (double)x * reinterpret_cast<const double*>(hv_dyn + HV_U_OFF)[r & 4095u];   // (as above)
    }
    __device__ __forceinline__ void fma(uint32_t r, float x, double (&a)[1]) const {
        a[0] = ::fma((double)x, reinterpret_cast<const double*>(hv_dyn + HV_U_OFF)[r], a[0]);
    }
    __device__ __forceinline__ void out(const HvChunk& ch, int k, const double (&v)[1]) const {
        hpart[(size_t)(ch.h0 + k) * nb + ch.base] = v[0];
    }
};

// ------------------------------------------------------------------ build kernels (ml_create; X is fixed)
// histogram of column lengths >= HV_MINLEN (clamped to 65535)
__global__ void k_hv_lenhist(const int* colptr, int n, unsigned* hist) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int L = colptr[j + 1] - colptr[j];
        if (L >= HV_MINLEN) atomicAdd(&hist[min(L, 65535)], 1u);
    }
}
__global__ void k_hv_flags(const int* colptr, int n, int T, int* flag) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        flag[j] = (colptr[j + 1] - colptr[j] >= T) ? 1 : 0;
}
// exclusive scan of int data in place (three launches; sums < 2^31): block-local scans of 1024, block sums,
// then the offsets
__global__ void k_scan_local(int* a, int n, int* bsum) {
    __shared__ int ws[32];
    const int base = blockIdx.x * 1024, t = threadIdx.x;   // 256 threads x 4 items
    int v[4], s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) { const int i = base + 4 * t + k; v[k] = i < n ? a[i] : 0; s += v[k]; }
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, incl, o); if ((t & 31) >= o) incl += y; }
    if ((t & 31) == 31) ws[t >> 5] = incl;
    __syncthreads();
    if (t < 32) {
        int x = t < 8 ? ws[t] : 0, xi = x;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, xi, o); if (t >= o) xi += y; }
        if (t < 8) ws[t] = xi - x;
        if (t == 7) bsum[blockIdx.x] = xi;
    }
    __syncthreads();
    int run = ws[t >> 5] + incl - s;
#pragma unroll
    for (int k = 0; k < 4; ++k) { const int i = base + 4 * t + k; if (i < n) a[i] = run; run += v[k]; }
}
__global__ void k_scan_bsum(int* bsum, int nb) {   // one block: exclusive scan of the block sums in place
    __shared__ int carry;
    __shared__ int ws[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int b0 = 0; b0 < nb; b0 += blockDim.x) {
        const int i = b0 + threadIdx.x;
        const int x = i < nb ? bsum[i] : 0;
        int incl = x;
        const int t = threadIdx.x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, incl, o); if ((t & 31) >= o) incl += y; }
        if ((t & 31) == 31) ws[t >> 5] = incl;
        __syncthreads();
        if (t < 32) {
            const int nw = blockDim.x >> 5;
            int y0 = t < nw ? ws[t] : 0, yi = y0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, yi, o); if (t >= o) yi += y; }
            if (t < nw) ws[t] = yi - y0;
        }
        __syncthreads();
        const int ex = carry + ws[t >> 5] + incl - x;
        if (i < nb) bsum[i] = ex;
        __syncthreads();
        if (t == blockDim.x - 1) carry = ex + x;
        __syncthreads();
    }
}
__global__ void k_scan_add(int* a, int n, const int* bsum) {
    const int base = blockIdx.x * 1024;
    const int add = bsum[blockIdx.x];
    for (int k = threadIdx.x; k < 1024; k += blockDim.x) { const int i = base + k; if (i < n) a[i] += add; }
}
// heavy columns in column order (pos = exclusive scan of the flags): hcols[pos] = j, lens[pos] = its length
__global__ void k_hv_cols(const int* colptr, int n, int T, const int* pos, int* hcols, int* lens) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int L = colptr[j + 1] - colptr[j];
        if (L >= T) { hcols[pos[j]] = j; lens[pos[j]] = L; }
    }
}
// hid[j] = -1, then the rank of each heavy column (by decreasing length: the host's order of hcols)
__global__ void k_hv_hid(int n, int* hid) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) hid[j] = -1;
}
__global__ void k_hv_hid_set(const int* hcols, int nh, int* hid) {
    for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < nh; h += gridDim.x * blockDim.x) hid[hcols[h]] = h;
}
// S copy: heavy entries per row (cnt), their maximum
__global__ void k_hv_rowcnt(const int* rowptr, const int* col, int m, const int* hid, int* cnt, int* maxcnt) {
    int mx = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        int c = 0;
        for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) c += __ldg(hid + col[k]) >= 0;
        cnt[i] = c;
        mx = max(mx, c);
    }
    mx = (int)__reduce_max_sync(0xffffffffu, (unsigned)mx);
    if ((threadIdx.x & 31) == 0) atomicMax(maxcnt, mx);
}
// S chunks: runs of whole rows with at most HV_CHMAX heavy entries and HV_SMAX rows (a chunk starts where hrp
// crosses a multiple of chp = HV_CHMAX - the longest row, or at a multiple of HV_SMAX rows); flag[r] = 1 at a chunk's
// first row (flag[m] = 0), exclusive-scanned in place to each row's chunk index
__device__ __forceinline__ int hv_tile_flag(const int* hrp, int r, int chp) {
    return r == 0 || hrp[r] / chp != hrp[r - 1] / chp || (r / HV_SMAX) != ((r - 1) / HV_SMAX);
}
__global__ void k_hv_tileflags(const int* hrp, int m, int chp, int* flag) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r <= m; r += gridDim.x * blockDim.x)
        flag[r] = r < m ? hv_tile_flag(hrp, r, chp) : 0;
}
// a chunk of segments longer than 512 entries on average is reduced by the whole block, segment by segment
// (HV_LGBLK); the others by per-thread ranges
__host__ __device__ __forceinline__ int hv_lg(int entries, int segs) {
    const int mean = segs > 0 ? entries / segs : 0;
    return mean > 512 ? HV_LGBLK : 0;
}
__global__ void k_hv_tiles(const int* hrp, int m, int chp, const int* tidx, HvChunk* sch) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) {
        if (!hv_tile_flag(hrp, r, chp)) continue;
        int r1 = r + 1;   // the next chunk's first row (or m)
        while (r1 < m && !hv_tile_flag(hrp, r1, chp)) ++r1;
        sch[tidx[r]] = HvChunk{hrp[r], hrp[r1], r, r, r1 - r, hv_lg(hrp[r1] - hrp[r], r1 - r), 0, 0};
    }
}
// the S copy's entries of each row (swizzled: hv_phys_v / hv_phys_i)
__global__ void k_hv_rowfill(const int* rowptr, const int* col, const float* val, int m, const int* hid, const int* hrp,
                             float* sval, uint16_t* sidx) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        long long o = hrp[i];
        for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) {
            const int h = __ldg(hid + col[k]);
            if (h >= 0) { sval[hv_phys_v(o)] = val[k]; sidx[hv_phys_i(o)] = (uint16_t)h; ++o; }
        }
    }
}
// per chunk and 16-entry block of its stage: the chunk's segment holding the block's first entry (a thread per
// block; blocks past the chunk get any valid index)
__global__ void k_hv_blocks(const HvChunk* ch, int nch, const int* off, uint16_t* blk) {
    const long long N = (long long)nch * 256;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
        const HvChunk c = ch[i >> 8];
        const int t = (int)(i & 255);
        const int eb = c.e0 & ~15;
        const int lo = max(eb + 16 * t, c.e0);
        int k = 0, kh = c.ns - 1;
        while (k < kh) {
            const int mid = (k + kh + 1) >> 1;
            if (off[c.s0 + mid] <= lo) k = mid; else kh = mid - 1;
        }
        blk[i] = (uint16_t)k;
    }
}
// G copy: segment (band k, heavy h) lengths by binary search in the column's ascending rows
__device__ __forceinline__ int hv_lower(const int* row, int b, int e, int x) {
    while (b < e) { const int mid = (b + e) >> 1; if (row[mid] >= x) e = mid; else b = mid + 1; }
    return b;
}
__global__ void k_hv_segcnt(const int* colptr, const int* row, const int* hcols, int nh, int nb, int m, int* cnt) {
    const long long N = (long long)nh * nb;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(t / nh), h = (int)(t % nh);
        const int j = hcols[h], b = colptr[j], e = colptr[j + 1];
        const int lo = hv_lower(row, b, e, k * HV_RB), hi = hv_lower(row, b, e, min(m, (k + 1) * HV_RB));
        cnt[t] = hi - lo;
    }
}
__global__ void k_hv_segfill(const int* colptr, const int* row, const float* val, const int* hcols, int nh, int nb,
                             const int* off, float* gval, uint16_t* gidx) {   // a warp per segment (swizzled copy)
    const long long N = (long long)nh * nb;
    const int lane = threadIdx.x & 31;
    for (long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < N;
         t += ((long long)gridDim.x * blockDim.x) >> 5) {
        const int o = off[t], L = off[t + 1] - o;
        if (L == 0) continue;
        const int k = (int)(t / nh), h = (int)(t % nh);
        const int j = hcols[h];
        const int lo = hv_lower(row, colptr[j], colptr[j + 1], k * HV_RB);
        for (int q = lane; q < L; q += 32) {
            gval[hv_phys_v((long long)o + q)] = val[lo + q];
            gidx[hv_phys_i((long long)o + q)] = (uint16_t)(row[lo + q] - k * HV_RB);
        }
    }
}
// G chunks: whole segments of one band, greedily packed up to HV_CHMAX entries and HV_SMAX heavy ids (a thread per
// band; a chunk's ids [h0, h1) start and end at non-empty segments).  Pass 0 counts each band's chunks, pass 1 writes
// them from choff[band].
__global__ void k_hv_chunks(const int* off, int nh, int nb, int pass, int* nch, const int* choff, HvChunk* gch) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nb; k += gridDim.x * blockDim.x) {
        const int* o = off + (size_t)k * nh;
        int cs = 0, cl = 0, h0 = -1, h1 = 0, nc = 0;
        int wc = pass ? choff[k] : 0;
        for (int h = 0; h < nh; ++h) {
            const int L = o[h + 1] - o[h];
            if (L == 0) continue;
            if (h0 >= 0 && (cl + L > HV_CHMAX || h + 1 - h0 > HV_SMAX)) {
                if (pass) gch[wc++] = HvChunk{cs, cs + cl, k, k * nh + h0, h1 - h0, hv_lg(cl, h1 - h0), h0, 0};
                ++nc;
                h0 = -1;
            }
            if (h0 < 0) { h0 = h; cs = o[h]; cl = 0; }
            cl += L;
            h1 = h + 1;
        }
        if (h0 >= 0) {
            if (pass) gch[wc++] = HvChunk{cs, cs + cl, k, k * nh + h0, h1 - h0, hv_lg(cl, h1 - h0), h0, 0};
            ++nc;
        }
        if (!pass) nch[k] = nc;
    }
}

}  // namespace ml
