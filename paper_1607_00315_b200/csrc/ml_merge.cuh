// ml_merge.cuh — merge-path column passes (sm_100a): out_p = sum_{k in column C[p]} term(X_k, row_k) for every
// position p of a column list (or of all columns), for the A2 gathers (g_j, h_j) and the X_A^T v half of
// the Hessian-vector product.
//
// Why: the Zipf designs mix 45 % empty columns, millions of 1-10-nonzero columns and columns holding most of X
// (SURVEY §8(d) D.2).  A schedule per column (a lane group per light column, a warp per 1024-nonzero unit of a heavy
// one) pays a fixed cost per column and per unit that the light columns never amortise.  Here every thread gets the
// same number of merge items -- a merge item is either one nonzero or one column end -- wherever the column
// boundaries fall (the merge-path split of Merrill & Garland's CSR SpMV, applied to the CSC).
//
// Tile = MP_NT threads x MP_IPT merge items.  Per tile:
//   1. its start and end coordinates (x = positions emitted, y = nonzeros consumed) come from k_mp_search;
//   2. the ends of its positions are staged in shared memory, each thread finds its own start by a binary search
//      there and records the CSC index of each nonzero it will consume;
//   3. the tile's nonzeros are loaded and gathered ELEMENT-interleaved (lane l takes elements l, l + 256, ...: a
//      dense column's rows are consecutive, so a warp's gathers share cache lines) and the products land in shared
//      memory;
//   4. each thread walks its items in order, summing products and emitting a position at each column end; the
//      partial sum of the column open at the end of its range is its carry.  A thread's first emitted column adds
//      the carries of the threads before it that carried the same column, in thread order; the column open at the
//      tile's end becomes the tile's carry-out, and k_mp_fixup adds the carry-outs of consecutive tiles, in tile
//      order, to the column's output.
// Every sum has a fixed order for a given launch shape: results are bitwise reproducible.
#pragma once

#include "ml_kernels.cuh"

namespace ml {

constexpr int MP_NT = 256;
constexpr int MP_IPT = 8;
constexpr int MP_TILE = MP_NT * MP_IPT;   // merge items per tile
constexpr int MP_TP = MP_TILE + MP_TILE / 8;   // padded per-element arrays: element e at e + e / 8, so that threads
__device__ __forceinline__ int mp_pad(int e) { return e + (e >> 3); }   // walking 8 consecutive elements do not collide

// the merge problem of one column list
struct MPList {
    const int* colptr;   // CSC column pointers [n + 1]
    const int* idx;      // CSC row indices
    const float* val;    // CSC values
    const int* list;     // positions -> columns (nullptr: all columns, position = column)
    const int* vptr;     // virtual start of each position's nonzeros, [nC + 1] (list == nullptr: colptr)
    const int* nC_dev;   // position count on the device (nullptr: nC_host)
    int nC_host;
    int2* tstart;        // [tiles + 1] merge coordinates of the tile starts
    double2* cv;         // [tiles] carry-out value of each tile
    int* cx;             // [tiles] carry-out position of each tile (nC: none)
};

__device__ __forceinline__ int mp_nC(const MPList& L) { return L.nC_dev ? *L.nC_dev : L.nC_host; }

// per-nonzero terms
struct TermGH {   // (X_ij r_i, X_ij^2 D_i): g_j and h_j
    const double2* rD;
    __device__ __forceinline__ double2 operator()(int i, float x) const {
        const double2 q = __ldg(rD + i);
        const double xd = (double)x;
        return make_double2(xd * q.x, (xd * xd) * q.y);
    }
};
struct TermV2 {   // (X_ij v_i, X_ij u_i) with (v, u) interleaved: X_A^T (D o Xs) and X_A^T (D o Xz) at once
    const double2* vu;
    __device__ __forceinline__ double2 operator()(int i, float x) const {
        const double2 q = __ldg(vu + i);
        const double xd = (double)x;
        return make_double2(xd * q.x, xd * q.y);
    }
};
struct TermV1 {   // (X_ij v_i, 0)
    const double* v;
    __device__ __forceinline__ double2 operator()(int i, float x) const {
        return make_double2((double)x * __ldg(v + i), 0.0);
    }
};

// merge-path search on a diagonal: the split (x, y), x + y = d, with x column ends and y nonzeros before it;
// ends[x] = vptr[x + 1] (global memory)
__device__ __forceinline__ int2 mp_search_global(long long d, const int* vptr, int nC, int T) {
    int lo = (int)max(0LL, d - (long long)T), hi = (int)min(d, (long long)nC);
    while (lo < hi) {
        const int pivot = (lo + hi) >> 1;
        if ((long long)__ldg(vptr + pivot + 1) <= d - pivot - 1) lo = pivot + 1;
        else hi = pivot;
    }
    return make_int2(lo, (int)(d - lo));
}

// tile starts: tstart[t] for t in [0, tiles], tiles = ceil((nC + T) / MP_TILE); also clears the carries
__global__ void k_mp_search(MPList L, int tiles_cap) {
    const int nC = mp_nC(L);
    const int T = L.vptr[nC] - L.vptr[0];
    const long long N = (long long)nC + T;
    const int tiles = (int)((N + MP_TILE - 1) / MP_TILE);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= tiles && t <= tiles_cap; t += gridDim.x * blockDim.x) {
        const long long d = min((long long)t * MP_TILE, N);
        L.tstart[t] = mp_search_global(d, L.vptr, nC, T);
        if (t < tiles) L.cx[t] = nC;
    }
}

// one merge-path pass.  out[p] (p in [0, nC)) gets every position's sum except the carry-outs of earlier tiles
// (k_mp_fixup adds those).  acc: streamed nonzeros / positions (pass accounting).
// dynamic shared memory of k_mp_pass (the list arrays only when the pass runs over a list)
__host__ __device__ constexpr size_t mp_smem_bytes(bool list) {
    return (size_t)16 * MP_TP + 16 * MP_NT + 4 * (MP_TILE + 1) + 4 * MP_NT + (list ? 4 * (MP_TILE + 1 + MP_TP) : 0);
}
template <class Term>
__global__ void __launch_bounds__(MP_NT) k_mp_pass(MPList L, Term term, double2* out, const int* skip, long long* acc) {
    if (skip && *skip) return;
    extern __shared__ __align__(16) unsigned char mp_sm[];
    double2* s_prod = reinterpret_cast<double2*>(mp_sm);        // [MP_TILE] the terms of the tile's nonzeros
    double2* s_cv = s_prod + MP_TP;                              // [MP_NT] carries
    int* s_end = reinterpret_cast<int*>(s_cv + MP_NT);           // [MP_TILE + 1] ends of the tile's positions
    int* s_cx = s_end + MP_TILE + 1;                             // [MP_NT]
    int* s_del = s_cx + MP_NT;                                   // list: [MP_TILE + 1] CSC start - virtual start
    int* s_act = s_del + MP_TILE + 1;                            // list: [MP_TILE] CSC index of each nonzero
    const int nC = mp_nC(L);
    const int base0 = L.vptr[0];
    const int T = L.vptr[nC] - base0;
    const long long N = (long long)nC + T;
    const int tiles = (int)((N + MP_TILE - 1) / MP_TILE);
    const int tid = threadIdx.x;
    long long streamed = 0, segs = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int2 c0 = L.tstart[t], c1 = L.tstart[t + 1];
        const int x0 = c0.x, y0 = c0.y, x1 = c1.x, y1 = c1.y;
        const int np = min(x1 + 1, nC) - x0;   // positions touched: x0 .. x1 (x1 only if < nC)
        for (int k = tid; k < np; k += MP_NT) {
            const int p = x0 + k;
            s_end[k] = __ldg(L.vptr + p + 1) - base0;
            if (L.list) s_del[k] = __ldg(L.colptr + __ldg(L.list + p)) - (__ldg(L.vptr + p) - base0);
        }
        __syncthreads();
        // my start on the tile's merge path (relative diagonal dd)
        const int nx = x1 - x0, ny = y1 - y0;
        const int dd = min(tid * MP_IPT, nx + ny);
        int lo = max(0, dd - ny), hi = min(dd, nx);
        while (lo < hi) {
            const int pivot = (lo + hi) >> 1;
            if (s_end[pivot] <= y0 + dd - pivot - 1) lo = pivot + 1;
            else hi = pivot;
        }
        const int xs = x0 + lo, ys = y0 + dd - lo;
        const int dend = min(dd + MP_IPT, nx + ny);
        // walk 1 (list only): the CSC index of each nonzero I will consume
        if (L.list) {
            int x = xs, y = ys;
            for (int d = dd; d < dend; ++d) {
                if (x < nC && y < s_end[x - x0]) { s_act[mp_pad(y - y0)] = y + s_del[x - x0]; ++y; }
                else ++x;
            }
        }
        __syncthreads();
        // gathers, element-interleaved; the products to shared memory
        {
            int ii[MP_IPT];
            float vv[MP_IPT];
#pragma unroll
            for (int u = 0; u < MP_IPT; ++u) {
                const int e = tid + u * MP_NT;
                ii[u] = -1;
                vv[u] = 0.f;
                if (e < ny) {
                    const int a = L.list ? s_act[mp_pad(e)] : y0 + e + base0;
                    ii[u] = __ldg(L.idx + a);
                    vv[u] = __ldg(L.val + a);
                }
            }
#pragma unroll
            for (int u = 0; u < MP_IPT; ++u)
                if (ii[u] >= 0) s_prod[mp_pad(tid + u * MP_NT)] = term(ii[u], vv[u]);
        }
        __syncthreads();
        // walk 2: sums and column ends
        int x = xs, y = ys, first_x = -1;
        double2 a = make_double2(0.0, 0.0), first_a = a;
        for (int d = dd; d < dend; ++d) {
            if (x < nC && y < s_end[x - x0]) {
                const double2 q = s_prod[mp_pad(y - y0)];
                a.x += q.x;
                a.y += q.y;
                ++y;
            } else {
                if (first_x < 0) { first_x = x; first_a = a; }   // (may have started in an earlier thread)
                else out[x] = a;
                a = make_double2(0.0, 0.0);
                ++x;
                ++segs;
            }
        }
        streamed += y - ys;
        // the carries: segmented inclusive scan of (x, a) over the threads (keys are non-decreasing in tid): within a
        // warp by shuffles, then the run that crosses each warp boundary from the warps before, in warp order
        {
            const int lane = tid & 31, wid = tid >> 5;
            int key = x;
            double2 v = a;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int ko = __shfl_up_sync(0xffffffffu, key, o);
                const double vx = __shfl_up_sync(0xffffffffu, v.x, o), vy = __shfl_up_sync(0xffffffffu, v.y, o);
                if (lane >= o && ko == key) { v.x = vx + v.x; v.y = vy + v.y; }
            }
            __shared__ int s_wk[MP_NT / 32];
            __shared__ double2 s_wv[MP_NT / 32], s_win[MP_NT / 32];
            __shared__ int s_wink[MP_NT / 32];
            if (lane == 31) { s_wk[wid] = key; s_wv[wid] = v; }
            __syncthreads();
            if (tid == 0) {   // carry into warp w: the run of warp w-1's last key, accumulated over the warps before
                int ck = -1;
                double2 cv = make_double2(0.0, 0.0);
                for (int w = 0; w < MP_NT / 32; ++w) {
                    s_wink[w] = ck;
                    s_win[w] = cv;
                    if (s_wk[w] == ck) { cv.x = cv.x + s_wv[w].x; cv.y = cv.y + s_wv[w].y; }
                    else cv = s_wv[w];
                    ck = s_wk[w];
                }
            }
            __syncthreads();
            if (key == s_wink[wid]) { v.x = s_win[wid].x + v.x; v.y = s_win[wid].y + v.y; }
            s_cx[tid] = key;
            s_cv[tid] = v;
        }
        __syncthreads();
        if (first_x >= 0) {   // the carries of earlier threads of this tile (their run ends at tid - 1), then my part
            double2 s = make_double2(0.0, 0.0);
            if (tid > 0 && s_cx[tid - 1] == first_x) s = s_cv[tid - 1];
            out[first_x] = make_double2(s.x + first_a.x, s.y + first_a.y);
        }
        if (tid == MP_NT - 1 && x1 < nC) {   // the tile's carry-out: the run of the column open at its end (x1)
            L.cv[t] = s_cv[MP_NT - 1];
            L.cx[t] = x1;
        }
        __syncthreads();
    }
    acc_add(acc, streamed, segs);
}

// carry-outs into the outputs: a warp per tile; the warp of the first tile of each run of tiles carrying the same
// position sums the run's carries (lane l takes tiles l, l + 32, ... of the run in order, then one fixed butterfly)
// and adds them to the output.  A top Zipf column spans ~1000 tiles: one lane walking the run would be ~1000
// dependent L2 round trips.
__global__ void k_mp_fixup(MPList L, double2* out, const int* skip) {
    if (skip && *skip) return;
    const int nC = mp_nC(L);
    const int T = L.vptr[nC] - L.vptr[0];
    const long long N = (long long)nC + T;
    const int tiles = (int)((N + MP_TILE - 1) / MP_TILE);
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < tiles; t += nw) {
        const int p = L.cx[t];
        if (p >= nC || (t > 0 && L.cx[t - 1] == p)) continue;   // (warp-uniform)
        double2 c = make_double2(0.0, 0.0);
        bool more = true;
        for (int u0 = t; more; u0 += 32) {
            const int u = u0 + lane;
            const bool in = u < tiles && L.cx[u] == p;
            if (in) { const double2 q = L.cv[u]; c.x += q.x; c.y += q.y; }
            more = __all_sync(0xffffffffu, in);
        }
        c.x = warp_sum(c.x);
        c.y = warp_sum(c.y);
        if (lane == 0) {
            const double2 s = out[p];   // the part written by the tile where p ends
            out[p] = make_double2(c.x + s.x, c.y + s.y);
        }
    }
}

// virtual offsets of a list: vptr[p] = sum_{q < p} len(C[q]) (exclusive scan), vptr[nC] = total.  Three launches:
// block sums of MP_SCAN positions, one block scans the block sums, each block rescans with its offset.
constexpr int MP_SCAN = 2048;
__global__ void k_vscan_sums(const int* colptr, const int* list, const int* nC_dev, int nC_host, int* bsum) {
    const int nC = nC_dev ? *nC_dev : nC_host;
    const int p0 = blockIdx.x * MP_SCAN;
    if (p0 >= nC && blockIdx.x > 0) return;
    int s = 0;
    for (int p = p0 + threadIdx.x; p < min(nC, p0 + MP_SCAN); p += blockDim.x) {
        const int j = list[p];
        s += colptr[j + 1] - colptr[j];
    }
    s = (int)block_sum_any((double)s);   // (exact: integer counts < 2^53)
    if (threadIdx.x == 0) bsum[blockIdx.x] = s;
}
__global__ void k_vscan_top(int* bsum, const int* nC_dev, int nC_host) {   // one block: exclusive scan of the block sums
    const int nC = nC_dev ? *nC_dev : nC_host;
    const int nb = max(1, (nC + MP_SCAN - 1) / MP_SCAN);
    __shared__ int s_w[32];
    __shared__ int s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    for (int b0 = 0; b0 < nb; b0 += blockDim.x) {
        const int b = b0 + threadIdx.x;
        const int v = b < nb ? bsum[b] : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int u = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += u; }
        if (lane == 31) s_w[wid] = incl;
        __syncthreads();
        int woff = 0, tot = 0;
        for (int k = 0; k < W; ++k) { if (k < wid) woff += s_w[k]; tot += s_w[k]; }
        if (b < nb) bsum[b] = s_carry + woff + incl - v;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) bsum[nb] = s_carry;
}
__global__ void k_vscan_apply(const int* colptr, const int* list, const int* nC_dev, int nC_host, const int* bsum,
                              int* vptr) {
    const int nC = nC_dev ? *nC_dev : nC_host;
    const int p0 = blockIdx.x * MP_SCAN;
    __shared__ int s_w[32];
    __shared__ int s_carry;
    if (p0 > nC) return;
    if (threadIdx.x == 0) s_carry = bsum[blockIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    for (int q0 = p0; q0 < min(nC, p0 + MP_SCAN); q0 += blockDim.x) {
        const int p = q0 + threadIdx.x;
        int v = 0;
        if (p < min(nC, p0 + MP_SCAN)) { const int j = list[p]; v = colptr[j + 1] - colptr[j]; }
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int u = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += u; }
        if (lane == 31) s_w[wid] = incl;
        __syncthreads();
        int woff = 0, tot = 0;
        for (int k = 0; k < W; ++k) { if (k < wid) woff += s_w[k]; tot += s_w[k]; }
        if (p < min(nC, p0 + MP_SCAN)) vptr[p] = s_carry + woff + incl - v;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += tot;
        __syncthreads();
    }
    if (p0 <= nC && nC <= p0 + MP_SCAN && threadIdx.x == 0) vptr[nC] = bsum[max(1, (nC + MP_SCAN - 1) / MP_SCAN)];
}

}  // namespace ml
