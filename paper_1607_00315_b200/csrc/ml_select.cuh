// ml_select.cuh — A8: coarse-set selection (|C_1| from the free set P:602 via P:798).
//
// C_l = supp(w) U top-T_l candidates by (|g| desc, index asc) (DESIGN Q14), T_l = k_l - |supp|, l = 1..L.
// All L thresholds come from ONE MSD radix select over unique 96-bit keys  key = (bits(|g|) : ~index)  — 12 passes
// of 8-bit digits, each pass building one 256-bin histogram per level in shared memory (integer atomics only).
// Because keys are unique, the T_l-th largest key K_l splits the candidates exactly, and K_1 <= K_2 <= ...
// (T_l non-increasing), so a candidate's level is the number of thresholds it reaches.  The level lists are then
// emitted in ascending index order by a tile count / scan / write pass.
#pragma once
#include "ml_common.cuh"

namespace ml {

constexpr int SEL_LMAX = 32;
struct I64x32 { long long v[SEL_LMAX]; };

struct SelState {
    unsigned long long pre_hi[SEL_LMAX];
    unsigned pre_lo[SEL_LMAX];
    long long rank[SEL_LMAX];   // remaining 1-based rank inside the current prefix group
    long long target[SEL_LMAX]; // T_l
    unsigned ghist[SEL_LMAX][256];
    unsigned done;
    int L;
};

struct SelIn {
    const int* list;      // candidate positions -> column ids (nullptr: identity)
    const double* g;      // gradient value per position
    const int* count_dev; // number of positions (device) or
    int count_host;
    const double* w;      // iterate: w[col] != 0 -> support member (not a candidate)
    unsigned char* lev;   // [positions] level mark
};

__device__ __forceinline__ void sel_key(const SelIn& in, int p, unsigned long long& hi, unsigned& lo, int& col) {
    col = in.list ? in.list[p] : p;
    hi = (unsigned long long)__double_as_longlong(in.g[p]) & 0x7fffffffffffffffull;   // bits of |g|
    lo = ~(unsigned)col;                                                               // ties: smaller index first
}

// prefix match for the first d digits (d in 0..12)
__device__ __forceinline__ bool sel_match(unsigned long long hi, unsigned lo, int d, unsigned long long phi, unsigned plo) {
    if (d == 0) return true;
    if (d <= 8) return (hi >> (64 - 8 * d)) == phi;
    return hi == phi && (lo >> (32 - 8 * (d - 8))) == plo;
}
__device__ __forceinline__ unsigned sel_digit(unsigned long long hi, unsigned lo, int d) {
    if (d < 8) return (unsigned)(hi >> (56 - 8 * d)) & 255u;
    return (lo >> (24 - 8 * (d - 8))) & 255u;
}

// One digit pass for every level.  Levels whose prefixes coincide share one histogram (rep[l]); counting is
// warp-aggregated (__match_any_sync) to keep shared-memory atomics off the hot bins.
__global__ void __launch_bounds__(ML_NT) k_sel_pass(SelIn in, SelState* st, int d) {
    __shared__ unsigned h[SEL_LMAX][256];
    __shared__ unsigned long long s_hi[SEL_LMAX];
    __shared__ unsigned s_lo[SEL_LMAX];
    __shared__ int s_rep[SEL_LMAX];
    __shared__ bool s_last;
    const int L = st->L;
    const int lane = threadIdx.x & 31;
    for (int k = threadIdx.x; k < L * 256; k += ML_NT) h[k / 256][k % 256] = 0u;
    if (threadIdx.x < L) {
        s_hi[threadIdx.x] = st->pre_hi[threadIdx.x];
        s_lo[threadIdx.x] = st->pre_lo[threadIdx.x];
    }
    __syncthreads();
    if (threadIdx.x < L) {
        const int l = threadIdx.x;
        int rep = -1;
        if (st->target[l] > 0) {
            rep = l;
            for (int k = 0; k < l; ++k)
                if (st->target[k] > 0 && s_hi[k] == s_hi[l] && s_lo[k] == s_lo[l]) { rep = k; break; }
        }
        s_rep[l] = rep;
    }
    __syncthreads();
    const int n = in.count_dev ? *in.count_dev : in.count_host;
    const int stride = gridDim.x * ML_NT;
    for (int base = blockIdx.x * ML_NT + (threadIdx.x & ~31); base < n; base += stride) {
        const int p = base + lane;
        unsigned long long hi = 0ull;
        unsigned lo = 0u;
        int col = 0;
        bool cand = false;
        if (p < n) {
            sel_key(in, p, hi, lo, col);
            cand = (in.w[col] == 0.0);   // support members are not candidates
        }
        const unsigned dg = sel_digit(hi, lo, d);
        for (int l = 0; l < L; ++l) {
            if (s_rep[l] != l) continue;   // inactive or shares a histogram
            const bool mt = cand && sel_match(hi, lo, d, s_hi[l], s_lo[l]);
            const unsigned mm = __ballot_sync(0xffffffffu, mt);
            if (mt) {
                const unsigned grp = __match_any_sync(mm, dg);
                if (lane == __ffs(grp) - 1) atomicAdd(&h[l][dg], (unsigned)__popc(grp));
            }
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < L * 256; k += ML_NT)
        if (h[k / 256][k % 256]) atomicAdd(&st->ghist[k / 256][k % 256], h[k / 256][k % 256]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(&st->done, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x < L && s_rep[threadIdx.x] >= 0) {
        const int l = threadIdx.x, src = s_rep[l];
        long long r = st->rank[l];
        int b = 255;
        for (; b >= 0; --b) {
            const long long c = (long long)ld_cg(&st->ghist[src][b]);
            if (r <= c) break;
            r -= c;
        }
        if (b < 0) b = 0;   // (cannot happen when T_l <= #candidates)
        if (d < 8) st->pre_hi[l] = (st->pre_hi[l] << 8) | (unsigned long long)b;
        else st->pre_lo[l] = (st->pre_lo[l] << 8) | (unsigned)b;
        st->rank[l] = r;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < L * 256; k += ML_NT) st->ghist[k / 256][k % 256] = 0u;
    if (threadIdx.x == 0) st->done = 0u;
}

// level mark: 255 for support members, else the number of thresholds the key reaches (0 = not selected)
__global__ void __launch_bounds__(ML_NT) k_sel_mark(SelIn in, const SelState* st) {
    const int n = in.count_dev ? *in.count_dev : in.count_host;
    const int L = st->L;
    for (int p = blockIdx.x * ML_NT + threadIdx.x; p < n; p += gridDim.x * ML_NT) {
        unsigned long long hi;
        unsigned lo;
        int col;
        sel_key(in, p, hi, lo, col);
        unsigned char lv = 0;
        if (in.w[col] != 0.0) lv = 255;
        else
            for (int l = 0; l < L; ++l) {
                if (st->target[l] <= 0) break;
                const unsigned long long th = st->pre_hi[l];
                const unsigned tl = st->pre_lo[l];
                if (hi > th || (hi == th && lo >= tl)) lv = (unsigned char)(l + 1);
                else break;
            }
        in.lev[p] = lv;
    }
}

// emission: tile counts per level
__global__ void __launch_bounds__(ML_NT) k_emit_count(SelIn in, int L, int* cnt /*[ntiles][L]*/) {
    __shared__ int wc[ML_NW][SEL_LMAX];
    const int n = in.count_dev ? *in.count_dev : in.count_host;
    const int ntiles = (n + ML_NT - 1) / ML_NT;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int p = t * ML_NT + threadIdx.x;
        const int lv = (p < n) ? (int)in.lev[p] : 0;
        for (int l = 0; l < L; ++l) {
            const unsigned b = __ballot_sync(0xffffffffu, lv >= l + 1);
            if (lane == 0) wc[wid][l] = __popc(b);
        }
        __syncthreads();
        if (threadIdx.x < L) {
            int s = 0;
            for (int k = 0; k < ML_NW; ++k) s += wc[k][threadIdx.x];
            cnt[(size_t)t * L + threadIdx.x] = s;
        }
        __syncthreads();
    }
}
// one block per level: exclusive scan over tiles (in place)
__global__ void __launch_bounds__(ML_NT) k_emit_scan(SelIn in, int L, int* cnt) {
    __shared__ int part[ML_NT];
    const int l = blockIdx.x;
    const int n = in.count_dev ? *in.count_dev : in.count_host;
    const int ntiles = (n + ML_NT - 1) / ML_NT;
    const int per = (ntiles + ML_NT - 1) / ML_NT;
    const int t0 = threadIdx.x * per, t1 = min(ntiles, t0 + per);
    int s = 0;
    for (int t = t0; t < t1; ++t) s += cnt[(size_t)t * L + l];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int a = 0;
        for (int k = 0; k < ML_NT; ++k) { int v = part[k]; part[k] = a; a += v; }
    }
    __syncthreads();
    int a = part[threadIdx.x];
    for (int t = t0; t < t1; ++t) { int v = cnt[(size_t)t * L + l]; cnt[(size_t)t * L + l] = a; a += v; }
}
// by-value variants of the selection kernels' small arrays
__global__ void k_sel_init_v(SelState* st, int L, I64x32 T) {
    const int l = threadIdx.x;
    if (l == 0) { st->L = L; st->done = 0u; }
    if (l < SEL_LMAX) {
        st->pre_hi[l] = 0ull;
        st->pre_lo[l] = 0u;
        st->target[l] = (l < L) ? T.v[l] : 0;
        st->rank[l] = st->target[l];
    }
    for (int k = threadIdx.x; k < SEL_LMAX * 256; k += blockDim.x) st->ghist[k / 256][k % 256] = 0u;
}
__global__ void __launch_bounds__(ML_NT) k_emit_write_v(SelIn in, int L, const int* off, int* out, I64x32 O) {
    __shared__ int wc[ML_NW][SEL_LMAX];
    const int n = in.count_dev ? *in.count_dev : in.count_host;
    const int ntiles = (n + ML_NT - 1) / ML_NT;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int p = t * ML_NT + threadIdx.x;
        const int lv = (p < n) ? (int)in.lev[p] : 0;
        const int col = (p < n) ? (in.list ? in.list[p] : p) : 0;
        for (int l = 0; l < L; ++l) {
            const unsigned b = __ballot_sync(0xffffffffu, lv >= l + 1);
            if (lane == 0) wc[wid][l] = __popc(b);
        }
        __syncthreads();
        for (int l = 0; l < L; ++l) {
            const unsigned b = __ballot_sync(0xffffffffu, lv >= l + 1);
            if (lv >= l + 1) {
                int o = off[(size_t)t * L + l];
                for (int k = 0; k < wid; ++k) o += wc[k][l];
                o += __popc(b & ((1u << lane) - 1u));
                out[O.v[l] + o] = col;
            }
        }
        __syncthreads();
    }
}

}  // namespace ml
