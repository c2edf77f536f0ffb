// ml_select.cuh — A8: coarse-set selection (|C_1| from the free set P:602 via P:798).
//
// C_l = supp(w) U top-T_l candidates by (|g| desc, index asc) (DESIGN Q14), T_l = k_l - |supp|, l = 1..L.
// All L thresholds come from ONE MSD radix select over unique 96-bit keys  key = (bits(|g|) : ~index)  — 12 passes
// of 8-bit digits, each pass building one 256-bin histogram per level in shared memory (integer atomics only).
// Because keys are unique, the T_l-th largest key K_l splits the candidates exactly, and K_1 <= K_2 <= ...
// (T_l non-increasing), so a candidate's level is the number of thresholds it reaches.  The level lists are then
// emitted in ascending index order.  One cooperative launch (k_select_coop) does all of it.
#pragma once
#include "ml_common.cuh"

namespace ml {

constexpr int SEL_LMAX = 32;
struct I64x32 { long long v[SEL_LMAX]; };

struct SelState {   // global scratch of k_select_coop
    unsigned ghist3[3][SEL_LMAX][256];   // pass d uses buffer d % 3
    int ecnt[160][SEL_LMAX];              // per-block level counts (emission)
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

// All of A8 in one cooperative launch (grid <= 160 blocks; block b owns the contiguous candidates [b q, (b+1) q)):
// the 12 digit passes (block histograms in shared memory -> integer atomics into a triple-buffered global histogram
// -> one grid barrier -> every block derives the same digits, one warp per level), the level marks, and the in-order
// emission (per-block level counts -> barrier -> offsets in block order -> block-local ordered writes).  Same keys,
// digits and order as the k_sel_* / k_emit_* sequence.
__global__ void __launch_bounds__(ML_NT) k_select_coop(SelIn in, SelState* st, int L, I64x32 T, int* out, I64x32 O) {
    __shared__ unsigned h[SEL_LMAX][256];
    __shared__ unsigned long long s_hi[SEL_LMAX];
    __shared__ unsigned s_lo[SEL_LMAX];
    __shared__ long long s_rank[SEL_LMAX];
    __shared__ int s_rep[SEL_LMAX];
    __shared__ int wc[ML_NW][SEL_LMAX];
    __shared__ int s_base[SEL_LMAX];
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int G = gridDim.x;
    const int n = in.count_dev ? *in.count_dev : in.count_host;
    const int q = (n + G - 1) / G;
    const int p0 = min(n, (int)blockIdx.x * q), p1 = min(n, p0 + q);
    if (threadIdx.x < SEL_LMAX) {
        s_hi[threadIdx.x] = 0ull;
        s_lo[threadIdx.x] = 0u;
        s_rank[threadIdx.x] = threadIdx.x < L ? T.v[threadIdx.x] : 0;
    }
    if (blockIdx.x == 0)
        for (int k = threadIdx.x; k < 2 * SEL_LMAX * 256; k += blockDim.x) (&st->ghist3[0][0][0])[k] = 0u;
    __syncthreads();
    grid.sync();
    for (int d = 0; d < 12; ++d) {
        unsigned (*gh)[256] = st->ghist3[d % 3];
        if (blockIdx.x == 0 && d >= 1)   // buffer (d + 1) % 3: pass d - 2's, read by everyone before the last barrier
            for (int k = threadIdx.x; k < SEL_LMAX * 256; k += blockDim.x) (&st->ghist3[(d + 1) % 3][0][0])[k] = 0u;
        for (int k = threadIdx.x; k < L * 256; k += ML_NT) h[k / 256][k % 256] = 0u;
        if (threadIdx.x < L) {   // levels with equal prefixes share one histogram
            const int l = threadIdx.x;
            int rep = -1;
            if (T.v[l] > 0) {
                rep = l;
                for (int k = 0; k < l; ++k)
                    if (T.v[k] > 0 && s_hi[k] == s_hi[l] && s_lo[k] == s_lo[l]) { rep = k; break; }
            }
            s_rep[l] = rep;
        }
        __syncthreads();
        for (int base = p0 + (threadIdx.x & ~31); base < p1; base += ML_NT) {
            const int p = base + lane;
            unsigned long long hi = 0ull;
            unsigned lo = 0u;
            int col = 0;
            bool cand = false;
            if (p < p1) {
                sel_key(in, p, hi, lo, col);
                cand = (in.w[col] == 0.0);
            }
            const unsigned dg = sel_digit(hi, lo, d);
            for (int l = 0; l < L; ++l) {
                if (s_rep[l] != l) continue;
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
            if (h[k / 256][k % 256]) atomicAdd(&gh[k / 256][k % 256], h[k / 256][k % 256]);
        grid.sync();
        for (int l = wid; l < L; l += ML_NW) {   // the digit of the rank-th largest key (identical in every block)
            if (s_rep[l] < 0) continue;
            const int src = s_rep[l];
            const long long r = s_rank[l];
            unsigned c[8];
            long long tot = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) { c[k] = ld_cg(&gh[src][255 - (lane * 8 + k)]); tot += c[k]; }
            long long incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const long long before = incl - tot;
            int bsel = -1;
            long long rr = 0;
            if (before < r && r <= incl) {
                long long acc = before;
                for (int k = 0; k < 8; ++k) {
                    if (r <= acc + (long long)c[k]) { bsel = 255 - (lane * 8 + k); rr = r - acc; break; }
                    acc += c[k];
                }
            }
            const unsigned who = __ballot_sync(0xffffffffu, bsel >= 0);
            const int sl = who ? __ffs(who) - 1 : 0;
            const int b = max(0, __shfl_sync(0xffffffffu, bsel, sl));
            const long long rn = __shfl_sync(0xffffffffu, rr, sl);
            __syncwarp();
            if (lane == 0) {
                if (d < 8) s_hi[l] = (s_hi[l] << 8) | (unsigned long long)b;
                else s_lo[l] = (s_lo[l] << 8) | (unsigned)b;
                s_rank[l] = who ? rn : r;
            }
        }
        __syncthreads();
    }
    // level marks and per-block level counts
    for (int k = threadIdx.x; k < SEL_LMAX; k += ML_NT) s_base[k] = 0;
    __syncthreads();
    for (int base = p0; base < p1; base += ML_NT) {
        const int p = base + threadIdx.x;
        int lv = 0;
        if (p < p1) {
            unsigned long long hi;
            unsigned lo;
            int col;
            sel_key(in, p, hi, lo, col);
            if (in.w[col] != 0.0) lv = 255;
            else
                for (int l = 0; l < L; ++l) {
                    if (T.v[l] <= 0) break;
                    if (hi > s_hi[l] || (hi == s_hi[l] && lo >= s_lo[l])) lv = l + 1;
                    else break;
                }
            in.lev[p] = (unsigned char)lv;
        }
        for (int l = 0; l < L; ++l) {
            const unsigned b = __ballot_sync(0xffffffffu, p < p1 && lv >= l + 1);
            if (lane == 0 && b) atomicAdd(&s_base[l], __popc(b));
        }
    }
    __syncthreads();
    for (int l = threadIdx.x; l < L; l += ML_NT) st->ecnt[blockIdx.x][l] = s_base[l];
    grid.sync();
    for (int l = threadIdx.x; l < L; l += ML_NT) {   // my offset per level: the counts of the blocks before me
        int o = 0;
        for (int b = 0; b < (int)blockIdx.x; ++b) o += ld_cg(&st->ecnt[b][l]);
        s_base[l] = o;
    }
    __syncthreads();
    for (int base = p0; base < p1; base += ML_NT) {   // in-order writes
        const int p = base + threadIdx.x;
        const int lv = (p < p1) ? (int)in.lev[p] : 0;
        const int col = (p < p1) ? (in.list ? in.list[p] : p) : 0;
        for (int l = 0; l < L; ++l) {
            const unsigned b = __ballot_sync(0xffffffffu, lv >= l + 1);
            if (lane == 0) wc[wid][l] = __popc(b);
        }
        __syncthreads();
        for (int l = 0; l < L; ++l) {
            const unsigned b = __ballot_sync(0xffffffffu, lv >= l + 1);
            if (lv >= l + 1) {
                int o = s_base[l];
                for (int k = 0; k < wid; ++k) o += wc[k][l];
                o += __popc(b & ((1u << lane) - 1u));
                out[O.v[l] + o] = col;
            }
        }
        __syncthreads();
        for (int l = threadIdx.x; l < L; l += ML_NT) {
            int t = 0;
            for (int k = 0; k < ML_NW; ++k) t += wc[k][l];
            s_base[l] += t;
        }
        __syncthreads();
    }
}

}  // namespace ml
