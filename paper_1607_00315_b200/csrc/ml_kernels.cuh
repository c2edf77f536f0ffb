// ml_kernels.cuh — sm_100a kernels of the multilevel proximal-Newton hot path.
//
// Every X pass goes through one "segment engine": a segment is a CSR row or a CSC column (restricted to an index
// list C).  Segments up to SPLIT nonzeros are reduced by a group of G lanes (G = 4..32, chosen per context from
// the mean segment length) streaming 128-bit vectors of indices and values; longer segments are cut into CHUNK-
// nonzero units, one warp each, whose partial sums are combined in unit order by the last-arriving warp of the
// segment (deterministic).  Epilogues (per-sample logistic quantities, free-set compaction with KKT, Hessian-vector
// outputs) run on the reduced values while they are in shared memory.
#pragma once
#include <cooperative_groups.h>

#include "ml_common.cuh"
#include "ml_heavy.cuh"

namespace cg = cooperative_groups;

namespace ml {

constexpr int CHUNK = 1024;      // nonzeros per heavy unit (one warp)
constexpr int SPLIT_MIN = 32;    // smallest heavy threshold (capacity bound); per-family threshold Seg::split = 8 G
constexpr int TILE = ML_NT;   // segments per tile

enum { OUT_UPDATED = 0, OUT_CONVERGED = 1, OUT_NOSTEP = 2, OUT_STAGNATION = 3 };

// ------------------------------------------------------------------ device control block
struct TraceRow { int level, outcome, inner_iters, nA; long long nC; double F_before, F_after, alpha; };

struct Ctl {
    // relaxation state
    int nA, skip, level_conv, outcome, ls_ok, nS, nAf, skipped, t_acc, nC, acc_steps, level;
    const int* Cptr;            // current restriction list (nullptr = all columns)
    double vmax, v1, l1, L, F, F_before;
    double alpha, Delta, gd;
    double l1diff_out[ML_MAXLS];
    // counters
    unsigned red_ctr[8];
    unsigned tile_ctr, done_ctr, epoch, gbar;   // gbar: k_inner's split grid barrier (top bit flips per barrier)
    unsigned long long vmax_bits;
    long long cls[2][16];         // per pass class: [0] nonzeros streamed, [1] segments (rows/columns) visited
    long long dsupp;
    long long idx_desc;           // k_check_index: index descents not at a segment start (0 for a valid X)
    int units_n[4], units_h[4];   // per unit slot: #units, #heavy segments
    int ntrace, trace_cap, bad_y, pad2;
    unsigned long long tph[16];  // persistent inner solver: ns spent per phase (block 0), diagnostics
    unsigned s_ctr, g_ctr;       // large-m inner solver: unit claim counters of the S and G streams
    unsigned hclaim, pad4;       // k_heavy: unit claim counter (zeroed before each launch)
    double xmax;                 // max |X_ij| (large m: the fixed-point scale of X_A s)
    int maxrow, pad5;            // longest row of X
    long long hv_relax;          // relaxations that ran the heavy-column path (diagnostics, ml_heavy_info)
    unsigned zcnt, pad6;         // heavy path: units of the zeroing heavy columns listed this iteration
};

// heavy-segment schedule for one segment list
struct Units {
    int4* u;          // {position p, chunk c, heavy ordinal, first unit of p}
    int* n;           // -> Ctl::units_n[slot]
    int* h;           // -> Ctl::units_h[slot]
    double2* part;    // per-unit partials
    int* hcnt;        // per-heavy-segment arrival counters (kept at 0 between launches)
    int cap;
    unsigned* claim;  // k_heavy: warps claim units four at a time from this counter (zeroed before the launch)
};

// a segment source: rows of CSR or columns of CSC restricted to a list
struct Seg {
    const int* ptr;   // rowptr / colptr
    const int* idx;   // col / row indices; nullptr: a dense X read by columns (index-free, ml.h), where the row of
                      // element k of a column starting at cb is k - cb
    const float* val;
    long long nnz;
    const int* list;  // positions -> segment ids (nullptr = identity)
    double2* hres;    // heavy results per position
    int split;        // segments longer than this take the heavy (split) path
    const int* rowtab;   // dense X: rowtab[t] = t (t < m), so that rowtab - cb stands in for a staged index chunk
};
// the index of element k of a segment starting at cb (dense X: computed, no load)
__device__ __forceinline__ int seg_idx(const Seg& S, long long k, int cb) { return S.idx ? __ldg(S.idx + k) : (int)(k - cb); }

// ------------------------------------------------------------------ per-element operations
// An operation is applied to a batch of elements in three phases, so that every gather of the batch is in flight
// before the first fused multiply-add waits for one (a gather behind a data-dependent branch or behind the previous
// element's multiply-add is one L2 round trip per element: measured 1.08 -> see profiles/r02_kernels.md):
//   pre(c, ok)     first-level lookup of the element with index c (OpMargin: its support-bitmap word)
//   fetch(c, q)    the gathered operand (predicated on q = pre's result)
//   fma(a0, a1, x, q, v)   accumulate in element order (skipped when !q)
struct OpMargin {     // z_i = sum_k X_ik w_k, gathers gated by the support bitmap
    const double* w; const uint32_t* bits;
    typedef double Val;
    __device__ __forceinline__ void prepare() {}
    __device__ __forceinline__ bool pre(int c, bool ok) const {
#ifdef ML_MARGIN_NOBITS   // (experiment: w gathered for every nonzero, no bitmap lookup)
        return ok;
#else
        const uint32_t wd = ok ? __ldg(bits + (c >> 5)) : 0u;
        return (wd >> (c & 31)) & 1u;
#endif
    }
    __device__ __forceinline__ Val fetch(int c, bool q) const { return q ? __ldg(w + c) : 0.0; }
    __device__ __forceinline__ void fma(double& a0, double&, float x, bool q, Val v) const {
        if (q) a0 += (double)x * v;
    }
};
struct OpGH {         // g_j = sum_i X_ij r_i ; h_j = sum_i X_ij^2 D_i
    const double2* rD;
    typedef double2 Val;
    __device__ __forceinline__ void prepare() {}
    __device__ __forceinline__ bool pre(int, bool ok) const { return ok; }
    __device__ __forceinline__ Val fetch(int r, bool q) const { return q ? __ldg(rD + r) : make_double2(0.0, 0.0); }
    __device__ __forceinline__ void fma(double& a0, double& a1, float v, bool q, Val t) const {
        if (q) {
            double x = (double)v;
            a0 += x * t.x;
            a1 += (x * x) * t.y;
        }
    }
};
struct OpDot {        // acc = sum_i X_ij v_i
    const double* v;
    typedef double Val;
    __device__ __forceinline__ void prepare() {}
    __device__ __forceinline__ bool pre(int, bool ok) const { return ok; }
    __device__ __forceinline__ Val fetch(int r, bool q) const { return q ? __ldg(v + r) : 0.0; }
    __device__ __forceinline__ void fma(double& a0, double&, float x, bool q, Val t) const {
        if (q) a0 += (double)x * t;
    }
};
// Reduce the elements [b, e) of one segment with G lanes (lane in [0, G)).  Each lane streams U 16-byte vectors of
// indices and U of values per iteration (all loads issued before use), peeling the unaligned ends; then, GB vectors
// at a time: the first-level lookups of their 4 GB elements, their gathers, their multiply-adds in element order.
// cb: the start of the segment's column / row (dense X: the index of element k is k - cb)
template <int G, int U = 2, int GB = 2, class Op>
__device__ __forceinline__ void seg_accum(const Seg& S, const Op& op, int b, int e, int lane, double& a0, double& a1,
                                          int cb) {
    static_assert(U % GB == 0, "gather batches");
    for (int k = (b & ~3) + 4 * lane; k < e; k += 4 * U * G) {
        int4 iv[U];
        float4 vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int ku = k + 4 * G * u;
            if (!S.idx) {   // dense X: values only
                iv[u] = make_int4(ku - cb, ku + 1 - cb, ku + 2 - cb, ku + 3 - cb);
                if (ku < e && ku + 4 <= S.nnz) vv[u] = ld_stream_f4(S.val + ku);
                else if (ku < e) {
                    vv[u].x = S.val[ku];
                    vv[u].y = (ku + 1 < S.nnz) ? S.val[ku + 1] : 0.f;
                    vv[u].z = (ku + 2 < S.nnz) ? S.val[ku + 2] : 0.f;
                    vv[u].w = 0.f;
                } else vv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (!(ku < e)) iv[u] = make_int4(0, 0, 0, 0);
            } else if (ku < e && ku + 4 <= S.nnz) { iv[u] = ld_stream_i4(S.idx + ku); vv[u] = ld_stream_f4(S.val + ku); }
            else if (ku < e) {
                iv[u].x = S.idx[ku]; vv[u].x = S.val[ku];
                iv[u].y = (ku + 1 < S.nnz) ? S.idx[ku + 1] : 0; vv[u].y = (ku + 1 < S.nnz) ? S.val[ku + 1] : 0.f;
                iv[u].z = (ku + 2 < S.nnz) ? S.idx[ku + 2] : 0; vv[u].z = (ku + 2 < S.nnz) ? S.val[ku + 2] : 0.f;
                iv[u].w = 0; vv[u].w = 0.f;
            } else { iv[u] = make_int4(0, 0, 0, 0); vv[u] = make_float4(0.f, 0.f, 0.f, 0.f); }
        }
#pragma unroll
        for (int u0 = 0; u0 < U; u0 += GB) {
            int ci[4 * GB];
            float xv[4 * GB];
            bool q[4 * GB];
            typename Op::Val gv[4 * GB];
#pragma unroll
            for (int u = 0; u < GB; ++u) {
                const int ku = k + 4 * G * (u0 + u);
                ci[4 * u + 0] = iv[u0 + u].x; ci[4 * u + 1] = iv[u0 + u].y;
                ci[4 * u + 2] = iv[u0 + u].z; ci[4 * u + 3] = iv[u0 + u].w;
                xv[4 * u + 0] = vv[u0 + u].x; xv[4 * u + 1] = vv[u0 + u].y;
                xv[4 * u + 2] = vv[u0 + u].z; xv[4 * u + 3] = vv[u0 + u].w;
#pragma unroll
                for (int t = 0; t < 4; ++t) q[4 * u + t] = (ku + t >= b) && (ku + t < e);
            }
#pragma unroll
            for (int t = 0; t < 4 * GB; ++t) q[t] = op.pre(ci[t], q[t]);
#pragma unroll
            for (int t = 0; t < 4 * GB; ++t) gv[t] = op.fetch(ci[t], q[t]);
#pragma unroll
            for (int t = 0; t < 4 * GB; ++t) op.fma(a0, a1, xv[t], q[t], gv[t]);
        }
    }
}

// One tile of TILE consecutive segment positions; results (a0, a1) land in res[slot] (shared memory).
// The tile's segment bounds are loaded once, in parallel (one thread per segment), so the G rounds only stream.
// Heavy segments (> S.split) are not streamed here: their results come from S.hres, written by k_heavy.
// TS (segments per tile, a multiple of ML_NT / G, at most TILE): smaller tiles spread a short segment list over more
// blocks (the coarse free-set gathers of the large-m path)
//
// G == 4 with whole tiles (segments of a few nonzeros on average: the columns of cfg 5, 45 % of them empty, 1.25
// nonzeros per column below the split): ONE THREAD PER SEGMENT, four elements per iteration (loads, lookups, gathers,
// then the multiply-adds in element order).  The groups-of-4 engine spent ~800 warp instructions per 32 columns on
// vector bookkeeping for ~40 nonzeros (measured: 12 G columns/s whatever the occupancy); adjacent threads' elements
// are adjacent in memory, so the scalar loads of a warp share sectors.  (Measured with R segments per group at once
// instead: slower, the registers cost a resident block.)
// thread-per-segment tiles: a thread reads back only the res slot it wrote, so the callers' block barriers around
// the tile are not needed (a tile then costs each warp its own longest segment, not the block's)
template <int G, int TS = TILE> __host__ __device__ constexpr bool seg_tile_private() { return G == 4 && TS == TILE; }
template <int G, int TS = TILE> __device__ __forceinline__ void seg_tile_sync() {
    if constexpr (!seg_tile_private<G, TS>()) __syncthreads();
}
template <int G, class Op, int TS = TILE>
__device__ __forceinline__ void seg_tile(const Seg& S, const Op& op, int nseg, int tile, double2* res, long long& streamed,
                                         long long& segs) {
    constexpr int NG = ML_NT / G;
    static_assert(TS % NG == 0 && TS <= TILE, "tile size");
    if constexpr (seg_tile_private<G, TS>()) {
        const int p = tile * TS + threadIdx.x;
        int b = 0, e = 0;
        bool heavy = false;
        if (p < nseg) {
            const int j = S.list ? __ldg(S.list + p) : p;
            b = __ldg(S.ptr + j);
            e = __ldg(S.ptr + j + 1);
            segs += 1;
            if (e - b > S.split) { heavy = true; e = b; }
            else streamed += e - b;
        }
        double a0 = 0.0, a1 = 0.0;
        const int cb = b;
        for (int k = b; k < e; k += 4) {
            int ci[4];
            float xv[4];
            bool q[4];
            typename Op::Val gv[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                q[t] = k + t < e;
                ci[t] = q[t] ? seg_idx(S, k + t, cb) : 0;
                xv[t] = q[t] ? __ldg(S.val + k + t) : 0.f;
            }
#pragma unroll
            for (int t = 0; t < 4; ++t) q[t] = op.pre(ci[t], q[t]);
#pragma unroll
            for (int t = 0; t < 4; ++t) gv[t] = op.fetch(ci[t], q[t]);
#pragma unroll
            for (int t = 0; t < 4; ++t) op.fma(a0, a1, xv[t], q[t], gv[t]);
        }
        if (p < nseg) res[threadIdx.x] = heavy ? ld_cg(S.hres + p) : make_double2(a0, a1);
        return;
    }
    __shared__ int sb[TILE], se[TILE];
    {
        const int p = tile * TS + threadIdx.x;
        int b = 0, e = 0;
        if (threadIdx.x < TS && p < nseg) {
            const int j = S.list ? __ldg(S.list + p) : p;
            b = __ldg(S.ptr + j);
            e = __ldg(S.ptr + j + 1);
            segs += 1;
            if (e - b > S.split) { res[threadIdx.x] = ld_cg(S.hres + p); b = 0; e = -1; }
            else streamed += e - b;
        }
        sb[threadIdx.x] = b;
        se[threadIdx.x] = e;
    }
    __syncthreads();
    const int grp = threadIdx.x / G, lane = threadIdx.x % G;
#pragma unroll 1
    for (int r = 0; r < TS / NG; ++r) {
        const int slot = r * NG + grp;
        const int b = sb[slot], e = se[slot];
        double a0 = 0.0, a1 = 0.0;
        seg_accum<G>(S, op, b, e, lane, a0, a1, b);
        a0 = group_sum<G>(a0);
        a1 = group_sum<G>(a1);
        if (lane == 0 && e >= 0) res[slot] = make_double2(a0, a1);
    }
}

// pass accounting: acc[0] += nonzeros streamed, acc[16] += segments visited (block-reduced, integer atomics)
__device__ __forceinline__ void acc_add(long long* acc, long long nnz, long long segs) {
    __shared__ long long s_acc[2][32];
    const int lane = threadIdx.x & 31;
    long long a = warp_sum_ll(nnz), b = warp_sum_ll(segs);
    if (lane == 0) { s_acc[0][threadIdx.x >> 5] = a; s_acc[1][threadIdx.x >> 5] = b; }
    __syncthreads();
    if (threadIdx.x == 0 && acc) {
        long long x = 0, y = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { x += s_acc[0][k]; y += s_acc[1][k]; }
        if (x) atomicAdd((unsigned long long*)acc, (unsigned long long)x);
        if (y) atomicAdd((unsigned long long*)(acc + 16), (unsigned long long)y);
    }
    __syncthreads();
}

// Block-wide sum / min for any blockDim (multiple of 32); every thread returns the block value.
__device__ __forceinline__ double block_sum_any(double v) {
    __shared__ double sh[32];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh[k];
    __syncthreads();
    return t;
}
// ------------------------------------------------------------------ heavy units
// Build the heavy-unit schedule of a segment list: every segment longer than SPLIT gets ceil(len/CHUNK) units.
// Unit order is arbitrary (atomics); results do not depend on it.
__global__ void k_units_build(const int* __restrict__ ptr, const int* __restrict__ list, const int* nseg_dev, int nseg_host,
                              Units U, int split) {
    const int nseg = nseg_dev ? *nseg_dev : nseg_host;
    for (int p = blockIdx.x * ML_NT + threadIdx.x; p < nseg; p += gridDim.x * ML_NT) {
        const int j = list ? list[p] : p;
        const int len = ptr[j + 1] - ptr[j];
        if (len > split) {
            const int nch = (len + CHUNK - 1) / CHUNK;
            const int hs = atomicAdd(U.h, 1);
            const int base = atomicAdd(U.n, nch);
            for (int c = 0; c < nch && base + c < U.cap; ++c) U.u[base + c] = make_int4(p, c, hs, base);
        }
    }
}

// One warp per heavy unit.  SCATTER: out[idx] += X * coef[p] (fp64 atomics), else partial sums + in-order
// combination by the segment's last-arriving warp into S.hres[p].
template <class Op, bool SCATTER>
__global__ void __launch_bounds__(ML_NT) k_heavy(Seg S, Units U, Op op, const double* coef, double* out,
                                                  const int* skip, const int* skip2, long long* nnz_acc) {
    if ((skip && *skip) || (skip2 && *skip2)) return;
    op.prepare();
    const int lane = threadIdx.x & 31;
    const int nunits = min(*U.n, U.cap);
    const int gw = (blockIdx.x * ML_NT + threadIdx.x) >> 5, nw = (gridDim.x * ML_NT) >> 5;
    long long streamed = 0;
    int uend = 0;
    for (int u = U.claim ? 0 : gw;; u = U.claim ? u + 1 : u + nw) {
        if (U.claim && u >= uend) {   // dynamic: the next four units
            int ub = 0;
            if (lane == 0) ub = (int)atomicAdd(U.claim, 4u);
            u = __shfl_sync(0xffffffffu, ub, 0);
            uend = u + 4;
        }
        if (u >= nunits) break;
        const int4 un = U.u[u];
        const int p = un.x;
        if (SCATTER && coef[p] == 0.0) continue;   // (z pass: most units have a zero coefficient)
        const int j = S.list ? __ldg(S.list + p) : p;
        const int b0 = __ldg(S.ptr + j), e0 = __ldg(S.ptr + j + 1);
        const int b = b0 + un.y * CHUNK;
        const int e = min(e0, b + CHUNK);
        if (SCATTER) {
            const double cf = coef[p];
            if (cf == 0.0) continue;
            if (lane == 0) streamed += e - b;
            int k = b + lane;
            for (; k + 96 < e; k += 128) {   // loads of 4 elements in flight before their reductions
                int r[4];
                float v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) { r[u] = seg_idx(S, k + 32 * u, b0); v[u] = __ldg(S.val + k + 32 * u); }
#pragma unroll
                for (int u = 0; u < 4; ++u) atomicAdd(out + r[u], (double)v[u] * cf);
            }
            for (; k < e; k += 32) atomicAdd(out + seg_idx(S, k, b0), (double)__ldg(S.val + k) * cf);
        } else {
            if (lane == 0) streamed += e - b;
            double a0 = 0.0, a1 = 0.0;
            seg_accum<32, 4>(S, op, b, e, lane, a0, a1, b0);
            a0 = warp_sum(a0);
            a1 = warp_sum(a1);
            int last = 0;
            if (lane == 0) {
                U.part[u] = make_double2(a0, a1);
                __threadfence();
                const int nch = (e0 - b0 + CHUNK - 1) / CHUNK;
                last = (atomicAdd(U.hcnt + un.z, 1) == nch - 1);
            }
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last) {
                __threadfence();
                const int nch = (e0 - b0 + CHUNK - 1) / CHUNK;
                double s0 = 0.0, s1 = 0.0;
                for (int c = lane; c < nch; c += 32) { double2 q = ld_cg(U.part + un.w + c); s0 += q.x; s1 += q.y; }
                s0 = warp_sum(s0);
                s1 = warp_sum(s1);
                if (lane == 0) { S.hres[p] = make_double2(s0, s1); U.hcnt[un.z] = 0; }
            }
        }
    }
    acc_add(nnz_acc, streamed, 0);
}
// ------------------------------------------------------------------ parameters shared by the relaxation kernels
struct Prm {
    int m, n;
    const int8_t* y;
    const double* b;   // squared loss (LASSO) targets; nullptr = logistic loss with labels y
    double lam, eps_h, sigma_in, sigma_out, beta_ls, tol, eta;
    int max_ls, inner_cg, pcd_snap, dyn;   // dyn: large-m streams claim units dynamically whatever their count
    double* w; uint32_t* wbits; double* z; double2* rD;
    double* Xd; double* Xs; double* sv; double* Xu;   // Xu: scatter target of the atomic path (kept zero between uses)
    double* Xz; double* svz; double* Xzu;             // snap path: X_A z, D o Xz; Xzu: atomic scatter target of z (kept zero)
    double2* sv2;                                     // large m, snap path: (D o Xs, D o Xz) per row, one 16-byte gather per nonzero
    double* parts; int nparts;                        // small-m scatter: per-block partials (+ group partials)
    double* irpart;                                   // persistent inner solver: slot-major block partials
    int2* uext; int* upos; double2* upart; int* ustart; int* uend; long long* unz;   // its column units (m > SMALL_M)
    Ctl* ctl;
    double* part;              // reduction partials
    double2* tilepart;         // per-tile partials of the compaction kernels
    unsigned long long* status;// look-back tile status
    TraceRow* trace;
    HvPrm hv;                  // the heavy-column path of the large-m inner solver (ml_heavy.cuh)
};
// free-set buffers of one relaxation (fine or coarse set)
struct ASet { int* A; double* gA; double* hA; double* wA; double* d; double* Hd; double* s; double* Hs; double* u; };


// ------------------------------------------------------------------ A1: margins (full CSR pass)
// z = Xw (CSR, support-bitmap-gated gathers of w), then per row: t, ell, r, D; L = sum ell.
template <int G>
__global__ void __launch_bounds__(ML_NT) k_margins(Prm P, Seg S, long long* acc) {
    __shared__ double2 res[TILE];
    __shared__ double sm[3 * ML_NW + 3];
    OpMargin op{P.w, P.wbits};
    const int ntiles = (P.m + TILE - 1) / TILE;
    double lsum = 0.0;
    long long streamed = 0, segs = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        seg_tile<G>(S, op, P.m, tile, res, streamed, segs);
        seg_tile_sync<G>();
        const int i = tile * TILE + threadIdx.x;
        if (i < P.m) {
            const double z = res[threadIdx.x].x;
            const RowState st = row_state_i(P.y, P.b, i, z);
            P.z[i] = z;
            P.rD[i] = make_double2(st.r, st.D);
            lsum += st.ell;
        }
        seg_tile_sync<G>();
    }
    acc_add(acc, streamed, segs);
    Red<1> r;
    r.s[0] = lsum;
    if (grid_reduce(r, P.part, &P.ctl->red_ctr[0], sm)) {
        if (threadIdx.x == 0) { P.ctl->L = r.s[0]; P.ctl->F = r.s[0] + P.lam * P.ctl->l1; }
    }
}

// ------------------------------------------------------------------ A2 + A3: gather over C with free-set compaction
// For each position p of C (j = C[p], or p when C is all columns): g_j, h_j; v_j (min-norm subgradient,
// P:248-256); free flag w_j != 0 or |g_j| > lam (P:459-461 via P:790).  Free columns are compacted IN ORDER into
// the ASet (A, gA, hA + eps_h, wA) with a decoupled look-back scan over dynamically claimed groups of SUP tiles
// (one look-back per group).  FINEST additionally computes ||w||_1 and sum |v| exactly.
// The last block to finish: nA, vmax, the convergence decision (R2), counters reset, epoch advance.
// MPOUT: the column sums were computed by the merge-path pass (ml_merge.cuh) into S.hres[p] (every position)
template <int G, bool FINEST, bool MPOUT = false>
__global__ void __launch_bounds__(ML_NT) k_gather_free(Prm P, Seg S, ASet AS, long long* acc) {
    // tiles per claim: one look-back per SUP tiles.  Coarse sets are small (tens of tiles): one tile per claim keeps
    // every tile's block busy (4 per claim left a 13 k-column coarse set on 13 blocks)
    constexpr int SUP = FINEST ? 4 : 1;
    constexpr int TS = FINEST ? TILE : 64;   // columns per tile (coarse: 64, so a 3.5 k-column set spans 55 blocks)
    __shared__ double2 res[TILE];
    __shared__ int s_tile, s_excl;
    __shared__ int s_wcnt[SUP][ML_NW];
    __shared__ double s_red[2 * ML_NW];
    __shared__ bool s_last;
    Ctl* ctl = P.ctl;
    if (ctl->skip) return;   // (not used at the finest level; coarse relaxations of a converged level)
    const int nC = S.list ? ctl->nC : P.n;
    const int ntiles = (nC + TS - 1) / TS;
    const int nsup = (ntiles + SUP - 1) / SUP;
    const unsigned epoch = ctl->epoch;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    OpGH op{P.rD};
    long long streamed = 0, segs = 0;
    double vmax_loc = 0.0;
    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&ctl->tile_ctr, 1u);
        __syncthreads();
        const int sup = s_tile;
        if (sup >= nsup) break;
        int jj[SUP], flag[SUP];
        double gg[SUP], hh[SUP], ww[SUP];
        double v1p = 0.0, l1p = 0.0;
        // the group's tiles: the sums (MPOUT: straight from S.hres, no shared memory, no barriers), then the bitmap
        // words of all SUP columns of a thread, then their w, then the flags (each a batch of independent loads)
        bool okc[SUP];
        uint32_t wb[SUP];
#pragma unroll
        for (int t = 0; t < SUP; ++t) {
            const int tile = sup * SUP + t;
            const int p = tile * TS + threadIdx.x;
            jj[t] = 0; flag[t] = 0; gg[t] = 0.0; hh[t] = 0.0; ww[t] = 0.0;
            okc[t] = tile < ntiles && threadIdx.x < TS && p < nC;
            if (MPOUT) {
                if (okc[t]) { const double2 q = S.hres[p]; gg[t] = q.x; hh[t] = q.y; }
            } else if (tile < ntiles) {   // (uniform over the block)
                seg_tile<G, OpGH, TS>(S, op, nC, tile, res, streamed, segs);
                seg_tile_sync<G, TS>();
                if (okc[t]) { gg[t] = res[threadIdx.x].x; hh[t] = res[threadIdx.x].y; }
                seg_tile_sync<G, TS>();
            }
        }
#pragma unroll
        for (int t = 0; t < SUP; ++t) {
            const int p = (sup * SUP + t) * TS + threadIdx.x;
            if (okc[t]) jj[t] = S.list ? S.list[p] : p;
            wb[t] = okc[t] ? P.wbits[jj[t] >> 5] : 0u;
        }
#pragma unroll
        for (int t = 0; t < SUP; ++t)
            if (okc[t] && ((wb[t] >> (jj[t] & 31)) & 1u)) ww[t] = P.w[jj[t]];
#pragma unroll
        for (int t = 0; t < SUP; ++t) {
            if (okc[t]) {
                const double v = (ww[t] != 0.0) ? gg[t] + P.lam * sgn(ww[t]) : soft(gg[t], P.lam);
                vmax_loc = fmax(vmax_loc, fabs(v));
                v1p += fabs(v);
                l1p += fabs(ww[t]);
                flag[t] = (ww[t] != 0.0) || (fabs(gg[t]) > P.lam);
            }
            const unsigned bal = __ballot_sync(0xffffffffu, flag[t]);
            if (lane == 0) s_wcnt[t][wid] = __popc(bal);
        }
        if (FINEST) {
            v1p = warp_sum(v1p);
            l1p = warp_sum(l1p);
            if (lane == 0) { s_red[wid] = v1p; s_red[ML_NW + wid] = l1p; }
        }
        __syncthreads();
        int total = 0;
        for (int t = 0; t < SUP; ++t)
            for (int k = 0; k < ML_NW; ++k) total += s_wcnt[t][k];
        if (wid == 0) {
            if (FINEST && lane == 0) {
                double a = 0.0, b = 0.0;
                for (int k = 0; k < ML_NW; ++k) { a += s_red[k]; b += s_red[ML_NW + k]; }
                P.tilepart[sup] = make_double2(a, b);
            }
            // publish and look back (epoch-tagged status words: epoch<<34 | flag<<32 | count; flag 1: this group's
            // count, flag 2: the inclusive prefix).  The look-back is warp-parallel: lane l reads predecessor
            // base - l, the nearest inclusive prefix ends it (one L2 round trip per 32 predecessors; one thread
            // walking them one by one made the prefix frontier the bottleneck of the pass: 0.74 ms of look-backs for
            // the 19.5 k groups of cfg 5's finest compaction).
            const unsigned long long e34 = (unsigned long long)epoch << 34;
            int excl = 0;
            if (lane == 0) {
                __threadfence();
                atomicExch(P.status + sup, e34 | ((sup == 0 ? 2ull : 1ull) << 32) | (unsigned)total);
            }
            if (sup > 0) {
                int wbase = sup - 1;
                while (true) {
                    const int pred = wbase - lane;
                    unsigned long long st = 0ull;
                    if (pred >= 0) {
                        do { st = *((volatile unsigned long long*)(P.status + pred)); }
                        while ((st >> 34) != epoch || ((st >> 32) & 3ull) == 0);
                    }
                    const bool incl = pred >= 0 && ((st >> 32) & 3ull) == 2;
                    const unsigned mi = __ballot_sync(0xffffffffu, incl);
                    const int first = mi ? __ffs(mi) - 1 : 32;   // the nearest predecessor with an inclusive prefix
                    int v = (pred >= 0 && lane <= first) ? (int)(st & 0xffffffffull) : 0;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    excl += v;
                    if (mi) break;   // (group 0 always publishes an inclusive prefix: the walk ends there at the latest)
                    wbase -= 32;
                }
                if (lane == 0) {
                    __threadfence();
                    atomicExch(P.status + sup, e34 | (2ull << 32) | (unsigned)(excl + total));
                }
            }
            if (lane == 0) s_excl = excl;
        }
        __syncthreads();
        int base = s_excl;
#pragma unroll
        for (int t = 0; t < SUP; ++t) {   // in order: tile t after the tiles before it, warps, lanes
            int woff = 0, ttot = 0;
            for (int k = 0; k < ML_NW; ++k) { if (k < wid) woff += s_wcnt[t][k]; ttot += s_wcnt[t][k]; }
            const unsigned bal = __ballot_sync(0xffffffffu, flag[t]);
            if (flag[t]) {
                const int o = base + woff + __popc(bal & ((1u << lane) - 1u));
                AS.A[o] = jj[t];
                AS.gA[o] = gg[t];
                AS.hA[o] = hh[t] + P.eps_h;
                AS.wA[o] = ww[t];
            }
            base += ttot;
        }
        __syncthreads();
    }
    acc_add(acc, streamed, segs);
    // block max -> global atomic max (order-independent)
    {
        double v = warp_max(vmax_loc);
        if (lane == 0) s_red[wid] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double mx = 0.0;
            for (int k = 0; k < ML_NW; ++k) mx = fmax(mx, s_red[k]);
            atomic_max_nonneg(reinterpret_cast<double*>(&ctl->vmax_bits), mx);
            __threadfence();
            s_last = (atomicAdd(&ctl->done_ctr, 1u) == gridDim.x - 1);
        }
        __syncthreads();
    }
    if (!s_last) return;
    __threadfence();
    if (FINEST) {   // exact sum |v| and ||w||_1 over all columns, in tile order
        double a = 0.0, b = 0.0;
        for (int t = threadIdx.x; t < nsup; t += ML_NT) { double2 q = ld_cg(P.tilepart + t); a += q.x; b += q.y; }
        Red<2> r;
        r.s[0] = a; r.s[1] = b;
        __shared__ double smr[2 * ML_NW + 2];
        block_reduce(r, smr);
        if (threadIdx.x == 0) { ctl->v1 = r.s[0]; ctl->l1 = r.s[1]; }
    }
    if (threadIdx.x == 0) {
        const unsigned long long st = nsup ? *((volatile unsigned long long*)(P.status + nsup - 1)) : 0ull;
        const int nA = nsup ? (int)(st & 0xffffffffull) : 0;
        ctl->nA = nA;
        const double vmax = __longlong_as_double((long long)ctl->vmax_bits);
        ctl->vmax = vmax;
        ctl->vmax_bits = 0ull;
        if (FINEST) { ctl->nAf = nA; ctl->F = ctl->L + P.lam * ctl->l1; }
        ctl->F_before = ctl->F;
        if (vmax / P.lam <= P.tol) { ctl->skip = 1; ctl->outcome = OUT_CONVERGED; ctl->level_conv = 1; }
        ctl->tile_ctr = 0u;
        ctl->done_ctr = 0u;
        ctl->epoch = (epoch + 1u) & 0x3fffffffu;
    }
}

// ------------------------------------------------------------------ plain gathers (API outputs / Hessian-vector)
// MODE 0: out0[p] = g, out1[p] = h (either may be null)      (ml_eval_f_grad, ml_diag_hess)
// MODE 1: out0[p] = sum X_ij v_i (+ eps_h * s[p] if s)       (Hs = X_A^T (D o Xs) + eps s, ml_hessvec)
// MODE 3: S.hres[p] = (g, h) for every position (the finest gather in two passes: k_gather_free<., ., true> then
//         compacts the free set from S.hres)
// MODE 2: PCD-CG epilogue: s_p = u_p + b s_prev_p, Hs_p = acc + eps s_p, first kink b_k = min_{x s < 0} -x/s,
//         last block: the CG step decision (R6')
template <int G, int MODE, class Op>
// (thread-per-column tiles, G == 4, are latency-bound: at most 32 registers, 8 resident blocks per SM)
__global__ void __launch_bounds__(ML_NT, (G == 4 ? 8 : 1)) k_gather_out(Seg S, Op op, const int* nseg_dev, int nseg_host, double* out0,
                                                      double* out1, long long* nnz_acc) {
    __shared__ double2 res[TILE];
    op.prepare();
    const int nseg = nseg_dev ? *nseg_dev : nseg_host;
    const int ntiles = (nseg + TILE - 1) / TILE;
    long long streamed = 0, segs = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        seg_tile<G>(S, op, nseg, tile, res, streamed, segs);
        seg_tile_sync<G>();
        const int p = tile * TILE + threadIdx.x;
        if (p < nseg) {
            const double2 q = res[threadIdx.x];
            if (MODE == 0) { if (out0) out0[p] = q.x; if (out1) out1[p] = q.y; }
            else if (MODE == 3) S.hres[p] = q;
            else out0[p] = q.x;
        }
        seg_tile_sync<G>();
    }
    acc_add(nnz_acc, streamed, segs);
}

// ------------------------------------------------------------------ A5: X_A s scatter (light segments)
template <int G>
__global__ void __launch_bounds__(ML_NT) k_scatter(Seg S, const int* nseg_dev, int nseg_host, const double* coef,
                                                   double* out, long long* nnz_acc) {
    const int nseg = nseg_dev ? *nseg_dev : nseg_host;
    const int grp = (blockIdx.x * ML_NT + threadIdx.x) / G, lane = threadIdx.x % G;
    const int ngrp = gridDim.x * (ML_NT / G);
    long long streamed = 0, segs = 0;
    for (int p = grp; p < nseg; p += ngrp) {
        const double cf = coef[p];
        if (cf == 0.0) continue;
        const int j = S.list ? __ldg(S.list + p) : p;
        const int b = __ldg(S.ptr + j), e = __ldg(S.ptr + j + 1);
        if (lane == 0) segs += 1;
        if (e - b > S.split) continue;   // heavy columns: k_heavy<SCATTER>
        if (lane == 0) streamed += e - b;
        for (int k = b + lane; k < e; k += G) atomicAdd(out + seg_idx(S, k, b), (double)__ldg(S.val + k) * cf);
    }
    acc_add(nnz_acc, streamed, segs);
}
// ------------------------------------------------------------------ A5 for small m: shared-memory passes
// When an m-vector fits in shared memory, the Hessian-vector passes over X_A stream whole columns per warp through
// a TMA-staged ring: one elected lane issues cp.async.bulk copies of SCH-element chunks of indices and values
// (mbarrier completion), NSTG chunks in flight per warp independently of occupancy; column metadata (coefficient,
// column pointers) is fetched 32 columns at a time, one per lane, and shuffled out, so no lane walks a dependent
// load chain per chunk.  Block b owns positions [b*q, (b+1)*q); warp w takes every W-th position of that range.
// SCH: elements per staged chunk (4*SCH bytes of indices + 4*SCH of values); NSTG: chunks in flight per warp.

// copy start, valid [vb, ve), copied to ce; cb: the start of the chunk's column (dense X: its row indices)
struct ChunkDesc { int a, vb, ve, ce; int p, last, cb, pad; double cf; };

// IND: the S phase of the large-m inner solver (coefficients by indirection, below); a plain stream does not carry
// (or test) those members, so that the long-lived G stream of k_inner keeps its registers
template <int SCH, int NSTG, bool IND = false>
struct ColStream {
    // warp-uniform producer state
    int p0, p1, W, wid, lane, nnz4;
    int batch, kk, noff;
    int mb, me;        // this lane's metadata for position p0 + wid + W * (batch * 32 + lane)
    double mcf;
    long long streamed, segs;
    const Seg* S;
    const double* coef;
    // coefficient by indirection (the large-m S phase: position p is a column unit, its coefficient coef[upos[p]] was
    // written by other blocks of this launch: L2 loads); zsrc: a second per-unit vector whose nonzero sets ChunkDesc::pad
    const int* upos = nullptr;
    const double* zsrc = nullptr;
    int mzf = 0;
    int* sidx; float* sval; uint64_t* bar; ChunkDesc* desc;
    const int2* ext; int ext_p0, ext_n;   // optional cached segment extents of positions [ext_p0, ext_p0 + ext_n)
    // dynamic schedule (claim != nullptr): the warp claims CLAIM_B positions of [p0, p1) at a time from a grid-wide
    // counter, so that no warp idles while another still holds a static share; its ring keeps streaming across claims
    static constexpr int CLAIM_B = 8;
    unsigned* claim = nullptr;
    int cb0 = 0, cbn = 0;

    __device__ void claim_next() {
        int base = 0;
        if (lane == 0) base = (int)atomicAdd(claim, (unsigned)CLAIM_B);
        base = __shfl_sync(0xffffffffu, base, 0);
        cb0 = base;
        cbn = max(0, min(CLAIM_B, p1 - base));
        load_batch();
    }
    __device__ void load_batch() {
        const int p = claim ? (lane < cbn ? cb0 + lane : p1) : p0 + wid + W * (batch * 32 + lane);
        mb = 0; me = 0; mcf = 0.0; mzf = 0;
        if (p < p1) {
            if constexpr (IND) {
                const int pu = __ldg(upos + p);
                mcf = ld_cg(coef + pu);
                if (zsrc && mcf != 0.0) mzf = ld_cg(zsrc + pu) != 0.0;
            } else mcf = coef ? coef[p] : 1.0;
            if (mcf != 0.0) {
                if (ext && p - ext_p0 < ext_n) {
                    const int2 x = ext[p - ext_p0];
                    mb = x.x;
                    me = x.y;
                } else {
                    const int j = S->list ? __ldg(S->list + p) : p;
                    mb = __ldg(S->ptr + j);
                    me = __ldg(S->ptr + j + 1);
                }
            }
        }
        kk = 0;
    }
    // next chunk descriptor (all lanes, uniform); false when the warp's range is exhausted
    __device__ bool next(ChunkDesc& d) {
        while (true) {
            int p;
            if (claim) {
                if (kk == cbn) {
                    claim_next();
                    if (cbn == 0) return false;
                }
                p = cb0 + kk;
            } else {
                if (kk == 32) { ++batch; load_batch(); }
                p = p0 + wid + W * (batch * 32 + kk);
                if (p >= p1) return false;
            }
            const int b = __shfl_sync(0xffffffffu, mb, kk), e = __shfl_sync(0xffffffffu, me, kk);
            const double cf = __shfl_sync(0xffffffffu, mcf, kk);
            if constexpr (IND) d.pad = __shfl_sync(0xffffffffu, mzf, kk);
            const int start = b + noff;
            if (cf == 0.0 || start >= e) {
                if (!coef && noff == 0 && cf != 0.0) {   // gather mode: an empty column still gets its (zero) output
                    d.a = b & ~3; d.vb = b; d.ve = b; d.ce = d.a; d.cf = 1.0; d.p = p; d.last = 1; d.cb = b;
                    ++kk;
                    return true;
                }
                ++kk; noff = 0; continue;
            }
            if (noff == 0 && lane == 0) { streamed += e - b; segs += 1; }
            d.a = start & ~3;
            d.vb = start;
            d.cb = b;
            d.ve = min(e, d.a + SCH);
            d.ce = min((d.ve + 3) & ~3, nnz4);
            if (d.ce < d.a) d.ce = d.a;
            d.cf = cf;
            d.p = p;
            d.last = (d.ve == e);
            if (d.last) { ++kk; noff = 0; } else noff = d.ve - b;
            return true;
        }
    }
    __device__ void issue(int st, const ChunkDesc& d) {   // lane 0 only
        const uint32_t bytes = 4u * (uint32_t)(d.ce - d.a);
        if (bytes) {
            fence_proxy_async();
            mbar_arrive_expect_tx(bar + st, S->idx ? 2 * bytes : bytes);   // (dense X: values only)
            if (S->idx) bulk_g2s(sidx + st * SCH, S->idx + d.a, bytes, bar + st);
            bulk_g2s(sval + st * SCH, S->val + d.a, bytes, bar + st);
        } else {
            mbar_arrive(bar + st);
        }
    }
};

// per-warp shared-memory layout: [idx NSTG*SCH int][val NSTG*SCH float][bars NSTG][desc NSTG][acc m double (scatter)]
template <int SCH, int NSTG>
__host__ __device__ inline size_t stream_warp_bytes(int m_acc) {
    const size_t b = (size_t)8 * NSTG * SCH + 8 * NSTG + NSTG * sizeof(ChunkDesc) + (size_t)8 * m_acc;
    return (b + 15) / 16 * 16;
}
constexpr int SC_SCH = 512, SC_NSTG = 2;   // scatter ring (the private m-vector shares the warp's shared memory)
constexpr int GA_SCH = 512, GA_NSTG = 3;   // gather ring
__host__ __device__ inline size_t scatter_smem_bytes(int W, int m) { return (size_t)W * stream_warp_bytes<SC_SCH, SC_NSTG>(m); }
__host__ __device__ inline size_t gather_smem_bytes(int W, int m) {
    return (size_t)W * stream_warp_bytes<GA_SCH, GA_NSTG>(0) + (size_t)8 * m;
}

template <int SCH, int NSTG>
__device__ __forceinline__ void stream_setup(ColStream<SCH, NSTG>& cs, unsigned char* base, const Seg& S, const double* coef, int nseg,
                                             int m_acc) {
    cs.ext = nullptr;
    cs.ext_n = 0;
    cs.W = blockDim.x >> 5;
    cs.wid = threadIdx.x >> 5;
    cs.lane = threadIdx.x & 31;
    const int q = (nseg + gridDim.x - 1) / gridDim.x;
    cs.p0 = blockIdx.x * q;
    cs.p1 = min(nseg, cs.p0 + q);
    cs.nnz4 = (int)(S.nnz & ~3LL);
    cs.batch = 0;
    cs.noff = 0;
    cs.streamed = 0;
    cs.segs = 0;
    cs.S = &S;
    cs.coef = coef;
    cs.sidx = reinterpret_cast<int*>(base);
    cs.sval = reinterpret_cast<float*>(base + 4 * NSTG * SCH);
    cs.bar = reinterpret_cast<uint64_t*>(base + 8 * NSTG * SCH);
    cs.desc = reinterpret_cast<ChunkDesc*>(cs.bar + NSTG);
    (void)m_acc;
    if (cs.lane == 0) {
        for (int k = 0; k < NSTG; ++k) mbar_init(cs.bar + k, 1);
        fence_mbar_init();
    }
    __syncwarp();
    cs.load_batch();
    // prologue: fill the ring
    for (int st = 0; st < NSTG; ++st) {
        ChunkDesc d;
        const bool ok = cs.next(d);
        if (cs.lane == 0) {
            if (ok) { cs.desc[st] = d; cs.issue(st, d); }
            else cs.desc[st].cf = 0.0;   // cf == 0 marks "no chunk"
        }
        if (!ok) {
            for (int s2 = st + 1; s2 < NSTG; ++s2) if (cs.lane == 0) cs.desc[s2].cf = 0.0;
            break;
        }
    }
    __syncwarp();
}

// X_A s into per-block partials (see above); every warp accumulates into its private shared m-vector: rows inside one
// column are distinct, so lanes never collide (plain LDS/STS, no atomics); warps and blocks are combined in fixed order.
// Cooperative launch.  After the per-block partials, one grid barrier; then every block combines its slice of rows
// over all partials (fixed order) and runs the m-side pass on it: mode 0 (API) out = X_A coef; mode 1 / 2 (PCD /
// PCD-CG relaxation step): pending Xd += beta Xs, Xs = Xu (+ b Xs_prev for CG), sv = D o Xs, and s^T H s summed in
// block order by the last block, which also takes the PCD decision.
__global__ void k_scatter_smem(Seg S, const int* nseg_dev, int nseg_host, const double* coef, double* parts,
                               int m, long long* acc, Prm P, double* out) {
    extern __shared__ __align__(16) unsigned char smraw[];
    constexpr int SCH = SC_SCH, NSTG = SC_NSTG;
    const size_t pw = stream_warp_bytes<SCH, NSTG>(m);
    unsigned char* base = smraw + (size_t)(threadIdx.x >> 5) * pw;
    double* mine = reinterpret_cast<double*>(base + stream_warp_bytes<SCH, NSTG>(0));
    for (int i = (threadIdx.x & 31); i < m; i += 32) mine[i] = 0.0;
    const int nseg = nseg_dev ? *nseg_dev : nseg_host;
    ColStream<SCH, NSTG> cs;
    stream_setup(cs, base, S, coef, nseg, m);
    uint32_t phase = 0u;
    int st = 0;
    while (true) {
        const ChunkDesc d = cs.desc[st];
        if (d.cf == 0.0) break;
        mbar_wait(cs.bar + st, (phase >> st) & 1u);
        phase ^= 1u << st;
        const int* ci = S.idx ? cs.sidx + st * SCH - d.a : S.rowtab - d.cb;
        const float* cv = cs.sval + st * SCH - d.a;
        const int kend = min(d.ve, d.ce);
        int k = d.vb + cs.lane;
        for (; k + 96 < kend; k += 128) {   // four independent read-modify-writes (distinct rows)
            const int r0 = ci[k], r1 = ci[k + 32], r2 = ci[k + 64], r3 = ci[k + 96];
            const double x0 = mine[r0], x1 = mine[r1], x2 = mine[r2], x3 = mine[r3];
            mine[r0] = fma((double)cv[k], d.cf, x0);
            mine[r1] = fma((double)cv[k + 32], d.cf, x1);
            mine[r2] = fma((double)cv[k + 64], d.cf, x2);
            mine[r3] = fma((double)cv[k + 96], d.cf, x3);
        }
        for (; k < kend; k += 32) { const int r = ci[k]; mine[r] = fma((double)cv[k], d.cf, mine[r]); }
        for (; k < d.ve; k += 32) {   // array tail not covered by 16-byte copies
            const int r = seg_idx(S, k, d.cb);
            mine[r] = fma((double)__ldg(S.val + k), d.cf, mine[r]);
        }
        __syncwarp();
        ChunkDesc nd;
        const bool ok = cs.next(nd);
        if (cs.lane == 0) {
            if (ok) { cs.desc[st] = nd; cs.issue(st, nd); }
            else cs.desc[st].cf = 0.0;
        }
        __syncwarp();
        st = (st + 1) % NSTG;
    }
    __syncthreads();
    const int W = blockDim.x >> 5;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        double t = 0.0;
        for (int w = 0; w < W; ++w)
            t += reinterpret_cast<const double*>(smraw + (size_t)w * pw + stream_warp_bytes<SCH, NSTG>(0))[i];
        parts[(size_t)blockIdx.x * m + i] = t;
    }
    acc_add(acc, cs.streamed, cs.segs);
    // all partials written -> grid barrier (cooperative launch: every block is resident)
    __threadfence();
    cg::this_grid().sync();
    // block b combines rows [b*R, b*R + R) over all partials: thread t sums the partials k = g, g + ng, ... of row
    // t % R (g = t / R); groups are combined in order -> deterministic
    const int R = (m + gridDim.x - 1) / gridDim.x;
    const int ng = max(1, (int)blockDim.x / max(R, 1));
    const int row0 = blockIdx.x * R, rr = threadIdx.x % max(R, 1), grp = threadIdx.x / max(R, 1);
    double* red = reinterpret_cast<double*>(smraw);   // the staging rings are no longer needed
    double t = 0.0;
    if (grp < ng && row0 + rr < m && rr < R)
        for (int k = grp; k < (int)gridDim.x; k += ng) t += ld_cg(parts + (size_t)k * m + row0 + rr);
    red[threadIdx.x] = t;
    __syncthreads();
    if ((int)threadIdx.x < R && row0 + (int)threadIdx.x < m) {
        double xu = 0.0;
        for (int g = 0; g < ng; ++g) xu += red[g * R + threadIdx.x];
        out[row0 + threadIdx.x] = xu;
    }
    // more rows per block than threads (a small grid, e.g. ml_set_sm_share): the remaining rows one thread each,
    // partials in block order
    for (int r = (int)blockDim.x + threadIdx.x; r < R && row0 + r < m; r += blockDim.x) {
        double xu = 0.0;
        for (int k = 0; k < (int)gridDim.x; ++k) xu += ld_cg(parts + (size_t)k * m + row0 + r);
        out[row0 + r] = xu;
    }
    (void)P;
}

// out_p = sum_i X_ij v_i over the positions of C (API Hessian-vector product), with v staged once per block in shared
// memory and the columns streamed through the TMA ring; one warp per column, lane partials reduced at its last chunk.
__global__ void k_gather_smem(Seg S, const int* nseg_dev, int nseg_host, const double* __restrict__ v, int m, double* out,
                              long long* acc) {
    extern __shared__ __align__(16) unsigned char smraw[];
    constexpr int SCH = GA_SCH, NSTG = GA_NSTG;
    const int W = blockDim.x >> 5;
    double* sv = reinterpret_cast<double*>(smraw + (size_t)W * stream_warp_bytes<SCH, NSTG>(0));
    for (int i = threadIdx.x; i < m; i += blockDim.x) sv[i] = v[i];
    __syncthreads();
    unsigned char* base = smraw + (size_t)(threadIdx.x >> 5) * stream_warp_bytes<SCH, NSTG>(0);
    const int nseg = nseg_dev ? *nseg_dev : nseg_host;
    ColStream<SCH, NSTG> cs;
    stream_setup(cs, base, S, nullptr, nseg, 0);
    uint32_t phase = 0u;
    int st = 0;
    double a = 0.0;
    while (true) {
        const ChunkDesc d = cs.desc[st];
        if (d.cf == 0.0) break;
        mbar_wait(cs.bar + st, (phase >> st) & 1u);
        phase ^= 1u << st;
        const int* ci = S.idx ? cs.sidx + st * SCH - d.a : S.rowtab - d.cb;
        const float* cv = cs.sval + st * SCH - d.a;
        const int kend = min(d.ve, d.ce);
        int k = d.vb + cs.lane;
        double a1 = 0.0, a2 = 0.0, a3 = 0.0;
        for (; k + 96 < kend; k += 128) {
            a = fma((double)cv[k], sv[ci[k]], a);
            a1 = fma((double)cv[k + 32], sv[ci[k + 32]], a1);
            a2 = fma((double)cv[k + 64], sv[ci[k + 64]], a2);
            a3 = fma((double)cv[k + 96], sv[ci[k + 96]], a3);
        }
        a += (a1 + a2) + a3;
        for (; k < kend; k += 32) a = fma((double)cv[k], sv[ci[k]], a);
        for (; k < d.ve; k += 32) a = fma((double)__ldg(S.val + k), sv[seg_idx(S, k, d.cb)], a);
        if (d.last) {
            const double t = warp_sum(a);
            if (cs.lane == 0) out[d.p] = t;
            a = 0.0;
        }
        __syncwarp();
        ChunkDesc nd;
        const bool ok = cs.next(nd);
        if (cs.lane == 0) {
            if (ok) { cs.desc[st] = nd; cs.issue(st, nd); }
            else cs.desc[st].cf = 0.0;
        }
        __syncwarp();
        st = (st + 1) % NSTG;
    }
    acc_add(acc, cs.streamed, cs.segs);
}

template <int SCH, int NSTG, bool IND>
__device__ __forceinline__ void stream_begin(ColStream<SCH, NSTG, IND>& cs, const Seg& S, const double* coef, int p0, int p1,
                                             unsigned char* base, const int2* ext = nullptr, int ext_n = 0) {
    cs.ext = ext;
    cs.ext_p0 = p0;
    cs.ext_n = ext_n;
    cs.W = blockDim.x >> 5;
    cs.wid = threadIdx.x >> 5;
    cs.lane = threadIdx.x & 31;
    cs.p0 = p0;
    cs.p1 = p1;
    cs.nnz4 = (int)(S.nnz & ~3LL);
    cs.batch = 0;
    cs.noff = 0;
    cs.S = &S;
    cs.coef = coef;
    cs.sidx = reinterpret_cast<int*>(base);
    cs.sval = reinterpret_cast<float*>(base + 4 * NSTG * SCH);
    cs.bar = reinterpret_cast<uint64_t*>(base + 8 * NSTG * SCH);
    cs.desc = reinterpret_cast<ChunkDesc*>(cs.bar + NSTG);
    if (cs.claim) { cs.cbn = 0; cs.kk = 0; }   // (the first next() claims)
    else cs.load_batch();
    for (int st = 0; st < NSTG; ++st) {
        ChunkDesc d;
        const bool ok = cs.next(d);
        if (cs.lane == 0) {
            if (ok) { cs.desc[st] = d; cs.issue(st, d); }
            else cs.desc[st].cf = 0.0;
        }
        if (!ok) {
            for (int s2 = st + 1; s2 < NSTG; ++s2) if (cs.lane == 0) cs.desc[s2].cf = 0.0;
            break;
        }
    }
    __syncwarp();
}


__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define PH_MARK(k)                                                                  \
    do {                                                                            \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                  \
            const unsigned long long t_ = gtimer();                                 \
            ph_acc[(k) + ph_off] += t_ - ph_t;                                      \
            ph_t = t_;                                                              \
        }                                                                           \
    } while (0)

#include "ml_inner.cuh"

// ------------------------------------------------------------------ relaxation bookkeeping
// Start of RELAX(C): reset per-relaxation flags; first == 1 starts a new level (clears level_conv).
__global__ void k_relax_begin(Prm P, int first_of_level, int level, const int* Cptr, int nC, int set_list) {
    Ctl* c = P.ctl;
    if (first_of_level) c->level_conv = 0;
    c->skip = c->level_conv;
    c->skipped = c->level_conv;
    c->outcome = c->level_conv ? OUT_CONVERGED : OUT_NOSTEP;
    c->ls_ok = 0;
    c->level = level;
    c->acc_steps = 0;
    if (set_list) { c->Cptr = Cptr; c->nC = nC; }
}

// R14-R16 for the API (ml_shrink_linesearch; the solver runs them inside k_inner): one batch of trials [t0, t0 + NT1)
// of the line search on F (Eq. 4; Armijo DESIGN Q7, Q26) for the step d = AS.d with Xd = P.Xd.  A-range
// blocks reduce the l1 trial differences sum(|w + a_t d| - |w|) of the batch (and, in the first batch, g^T d and
// max|d|); m-range blocks reduce sum_i dloss(t_i, a_t y_i Xd_i).  Last block: Delta, decision.  First batch
// {1, 1/2, 1/4, 1/8}; the second (rare) covers the remaining trials up to max_ls.
template <int NT1>
__global__ void __launch_bounds__(ML_NT) k_outer_ls(Prm P, ASet AS, int t0, int nblkA) {
    constexpr int NS = 1 + 2 * NT1;
    __shared__ double sm[(NS + 1) * ML_NW + NS + 1];
    Ctl* c = P.ctl;
    if (c->skip) return;
    if (t0 == 0) {
        if (c->acc_steps == 0) {   // R14: d = 0
            if (blockIdx.x == 0 && threadIdx.x == 0) { c->skip = 1; c->outcome = OUT_NOSTEP; }
            return;
        }
    } else if (c->ls_ok) return;
    const int T1 = min(P.max_ls, t0 + NT1);
    Red<NS, 1> r;
    r.zero();
    double at[NT1];
    {
        double a = 1.0;
        for (int t = 0; t < t0; ++t) a *= P.beta_ls;
#pragma unroll
        for (int k = 0; k < NT1; ++k) { at[k] = a; a *= P.beta_ls; }
    }
    if ((int)blockIdx.x < nblkA) {
        const int nA = c->nA;
        for (int p = blockIdx.x * ML_NT + threadIdx.x; p < nA; p += nblkA * ML_NT) {
            const double d = AS.d[p];
            const double w = AS.wA[p], aw = fabs(w);
            if (t0 == 0) {
                r.s[0] += AS.gA[p] * d;
                r.mx[0] = fmax(r.mx[0], fabs(d));
            }
#pragma unroll
            for (int k = 0; k < NT1; ++k) r.s[1 + k] += fabs(w + at[k] * d) - aw;
        }
    } else {
        const int nb = gridDim.x - nblkA;
        for (int i = (blockIdx.x - nblkA) * ML_NT + threadIdx.x; i < P.m; i += nb * ML_NT) {
            const double xd = P.Xd[i], zi = P.z[i];
#pragma unroll
            for (int k = 0; k < NT1; ++k)
                if (t0 + k < T1) r.s[1 + NT1 + k] += dloss_i(P.y, P.b, i, zi, at[k] * xd);
        }
    }
    if (grid_reduce(r, P.part, &c->red_ctr[5], sm)) {
        if (threadIdx.x == 0) {
            if (t0 == 0) {
                c->gd = r.s[0];
                c->Delta = r.s[0] + P.lam * r.s[1];
                if (r.mx[0] == 0.0) { c->skip = 1; c->outcome = OUT_NOSTEP; return; }
            }
            for (int k = 0; k < NT1 && t0 + k < T1; ++k) c->l1diff_out[t0 + k] = r.s[1 + k];
            const double Delta = c->Delta;
            for (int k = 0; k < NT1 && t0 + k < T1; ++k) {
                const double dF = r.s[1 + NT1 + k] + P.lam * r.s[1 + k];
                if (dF <= P.sigma_out * at[k] * Delta) { c->ls_ok = 1; c->alpha = at[k]; c->t_acc = t0 + k; break; }
            }
            if (!c->ls_ok && T1 >= P.max_ls) { c->skip = 1; c->outcome = OUT_STAGNATION; c->alpha = 0.0; }
        }
    }
}

// R18: w_A += a d (bitmap and |supp| maintained), ||w||_1 += l1 diff of the accepted trial; z += a Xd and the
// per-sample refresh (A1 incremental); L, F; trace row.
__global__ void __launch_bounds__(ML_NT) k_update(Prm P, ASet AS, int nblkA) {
    __shared__ double sm[2 * ML_NW + 2];
    __shared__ long long sml[ML_NW];
    Ctl* c = P.ctl;
    if (c->skip || !c->ls_ok) return;
    const double a = c->alpha;
    Red<1> r;
    r.zero();
    long long ds = 0;
    if ((int)blockIdx.x < nblkA) {
        const int nA = c->nA;
        for (int p = blockIdx.x * ML_NT + threadIdx.x; p < nA; p += nblkA * ML_NT) {
            const double w0 = AS.wA[p];
            const double w1 = w0 + a * AS.d[p];
            const int j = AS.A[p];
            P.w[j] = w1;
            AS.wA[p] = w1;
            const int nz0 = (w0 != 0.0), nz1 = (w1 != 0.0);
            if (nz0 != nz1) { atomicXor(P.wbits + (j >> 5), 1u << (j & 31)); ds += nz1 - nz0; }
        }
    } else {
        const int nb = gridDim.x - nblkA;
        for (int i = (blockIdx.x - nblkA) * ML_NT + threadIdx.x; i < P.m; i += nb * ML_NT) {
            const double z = P.z[i] + a * P.Xd[i];
            P.z[i] = z;
            const RowState st = row_state_i(P.y, P.b, i, z);
            P.rD[i] = make_double2(st.r, st.D);
            r.s[0] += st.ell;
        }
    }
    {
        long long t = warp_sum_ll(ds);
        if ((threadIdx.x & 31) == 0) sml[threadIdx.x >> 5] = t;
        __syncthreads();
        if (threadIdx.x == 0) {
            long long s = 0;
            for (int k = 0; k < ML_NW; ++k) s += sml[k];
            if (s) atomicAdd((unsigned long long*)&c->dsupp, (unsigned long long)s);
        }
    }
    if ((int)blockIdx.x < nblkA) r.s[0] = 0.0;
    if (grid_reduce(r, P.part, &c->red_ctr[6], sm)) {
        if (threadIdx.x == 0) {
            __threadfence();
            c->nS += (int)c->dsupp;
            c->dsupp = 0;
            c->L = r.s[0];
            c->l1 += c->l1diff_out[c->t_acc];
            const double Fb = c->F;
            c->F = c->L + P.lam * c->l1;
            c->outcome = OUT_UPDATED;
            if (c->ntrace < c->trace_cap) {
                TraceRow tr{c->level, OUT_UPDATED, c->acc_steps, c->nA, (long long)c->nC, Fb, c->F, a};
                P.trace[c->ntrace] = tr;
            }
            c->ntrace += 1;
        }
    }
}

}  // namespace ml
