// Persistent small-m inner solver (A4-A6 for m <= SMALL_M).
//
// One cooperative launch per relaxation runs all K inner iterations (R4-R12) on the free set A.
// Block b owns the contiguous free-set positions [b q, (b+1) q) and the contiguous rows [b R, (b+1) R).  Per inner
// iteration, two grid barriers:
//   D   my positions: direction (PCD Eq. 5 with the zeroing part z of Q27, or the PCD-CG residual u of Q9b), block
//       partial sums;
//   S   X_A coef over my columns into ONE shared m-vector per block: the block stages one column chunk at a time
//       (TMA bulk copies, a 4-stage ring) and every warp takes a slice of it -- rows are distinct within a column, so
//       there are no conflicts and no per-warp copies; zeroing columns also go to a second m-vector (X_A z);
//       the m-vector(s) are written as this block's partials                                      -> barrier B1
//   R   every block sums the direction partials (identical in every block: fixed order); my rows: X_A s = sum of the
//       block partials in block order (PCD-CG: X_A u + b X s_prev), X_A z, D-weighted squares; PCD-CG: s = u + b s_prev
//       and the first kink on my positions                                                         -> barrier B2
//   G   totals; the step decision (model Armijo with the snap path, or the CG step truncated at the first kink) in
//       every block; my rows Xd += X sigma; sv = D o X sigma for all rows into shared memory; my positions:
//       H sigma = X_A^T sv + eps sigma through per-warp TMA rings (prefetched across B2), d += sigma, Hd += H sigma.
// Partials are slot-major (part[slot * G + block]): a warp sums one slot with coalesced loads in a fixed order, so
// every block takes bitwise identical decisions, and results are reproducible run to run.
#pragma once

constexpr int IR_W = 8;          // warps per block (launch with 256 threads)
constexpr int IR_GMAX = 160;     // grid <= 160 blocks (5 partials per lane in the totals)
constexpr int IR_NT0 = 4;        // l1 trial differences computed with the direction; the rest only if Armijo needs them
constexpr int IR_SCH = 2048;               // S phase: block-shared ring of IR_SCH-element chunks, sst(GSCH) stages
#ifndef IR_RL
#define IR_RL 12   // R phase: partial loads in flight per thread (m = 2000, G = 148: one round)
#endif
#ifndef IR_GU
#define IR_GU 8   // BIG G phase: L2 gathers in flight per lane (multiple of 4)
#endif
#ifndef IR_GUZ
#define IR_GUZ IR_GU   // the same on the snap path (16-byte gathers of (D o Xs, D o Xz)); even (8: G 430 us, 4: 435)
#endif
#ifndef IR_RB
#define IR_RB 4   // BIG R phase: rows in flight per thread
#endif
constexpr int IR_QC = 1024;               // column extents of up to IR_QC own positions cached in shared memory
// phase timers (block 0, thread 0): 8 phases for small |A| and 8 for large |A|.  Debug builds: IR_PHDBG puts
// sub-phases of the small-|A| iteration in slots 8..15 (large |A| relaxations are then not timed) and the kernel time
// and iterations run in the trace rows (F_before, alpha); GS_PHDBG puts k_gather_small's phases in slots 8..15
#if defined(IR_PHDBG) || defined(GS_PHDBG)
constexpr int IR_PHN = 32;
#else
constexpr int IR_PHN = 16;
#endif
#ifdef IR_PHDBG
#define PH_SUB(k) PH_MARK(8 + (k))
#define IR_FB(x) ((double)(gtimer() - ph_k0))
#define IR_AL(x) ((double)ph_its)
#else
#define PH_SUB(k) do {} while (0)
#define IR_FB(x) (x)
#define IR_AL(x) (x)
#endif
#ifdef GS_PHDBG
#define GS_MARK(k) PH_MARK(8 + (k))
#else
#define GS_MARK(k) do {} while (0)
#endif
constexpr int IN_GST = 2;                  // G phase: per-warp rings of GSCH-element chunks (template)
// partial slots: D (PCD) 0 ps, 1 ss, 2 pz, 3 Z1, 4 zz, 5 #zeroing, 6..9 l1 trials 0..3, 10 max|s|, 11 vq
//                D (CG)  0 rz, 1 gx.u, 2 gx.s_prev, 3 u.u, 4 u.s_prev, 5 s_prev.s_prev, 11 vq
//                R       12 D Xs^2, 13 D Xs Xz, 14 D Xz^2, 15 first kink (min);  lazy l1 trials 16 ..
enum { IR_SD = 0, IR_SR = 12, IR_SL1 = 16 };
// outer line search + update (R14-R18): 0 g.d, 1 max|d|, 2..5 l1 trials 0..3, 6..9 loss trials 0..3; the rest:
// 10.. l1 trials 4.., then loss trials 4..; update: 0 L, 1 support change
constexpr int IR_NLS = ML_MAXLS - 4;
enum { IR_SO = 0, IR_SO2 = 10, IR_SU = 10 + 2 * IR_NLS, IR_SO3 = IR_SU + 5, IR_NSLOT = IR_SO3 + 6 };
// IR_SU .. +4: unit counts, nnz; the same without the heavy columns; nnz of A's heavy columns (BIG); IR_SO3: trials 1/2, 1/4, 1/8 of a large-m outer line search (l1, loss) when
// alpha = 1 failed
// the heavy-path instantiation's column rings (elements per chunk, stages per warp): build knobs for measurement
#ifndef IR_HSCH
#define IR_HSCH 1024
#endif
#ifndef IR_HST
#define IR_HST IN_GST
#endif
#ifndef IR_UNIT_V
#define IR_UNIT_V 2048
#endif
constexpr int IR_UNIT = IR_UNIT_V;
#ifndef IR_DYN_V
#define IR_DYN_V 32
#endif
constexpr int IR_DYN = IR_DYN_V;   // BIG: the S and G streams claim units dynamically when there are >= IR_DYN per warp   // BIG: columns are streamed in units of at most IR_UNIT nonzeros
#ifndef IR_UCOST_V
#define IR_UCOST_V 1024
#endif
constexpr int IR_UCOST = IR_UCOST_V;   // BIG: a unit's fixed cost in nonzeros (TMA issue, barrier wait) for the balance
constexpr unsigned IR_DMAX = (1u << 10) | (1u << 11);

// my positions' state, indexed by p - p0: shared memory when q <= IR_QS, else the ASet arrays (offset by p0)
constexpr int IR_QS = 160, IR_RS = 64;   // cached positions / rows per block (rows: m <= IR_RS * G)
struct PosState { const double* wA; const double* gA; const double* hA; double* d; double* Hd; double* s; double* u; };
struct SChunk { int p, a, vb, ve, ce, ok, cb, pad; };   // copy [a, ce) of column p (starting at cb), valid [vb, ve);
                                                       // ok = 0: no chunk

__host__ __device__ constexpr int ir_sst(int gsch) { return gsch >= 1024 ? 8 : 4; }   // the S ring fits the G rings
__host__ __device__ inline size_t ir_sring_bytes(int sst) {
    return (size_t)8 * sst * IR_SCH + 8 * sst + sizeof(SChunk) * sst;
}
template <int GSCH, int GST = IN_GST>
__host__ __device__ inline size_t ir_ring_bytes() {
    const size_t g = (size_t)IR_W * stream_warp_bytes<GSCH, GST>(0), s = ir_sring_bytes(ir_sst(GSCH));
    return ((g > s ? g : s) + 15) / 16 * 16;
}
static_assert(sizeof(SChunk) == 32, "SChunk layout");
// dynamic shared memory: the rings (S ring and G rings alias), then two m-vectors (X_A s | sv, X_A z); BIG: rings only
template <int GSCH>
__host__ __device__ inline size_t inner_smem_bytes(int m) { return ir_ring_bytes<GSCH>() + (size_t)16 * m; }
template <int GSCH, int GST>
__host__ __device__ inline size_t inner_big_smem_bytes() { return ir_ring_bytes<GSCH, GST>(); }
constexpr size_t IR_SMEM_MAX = 196 * 1024;   // dynamic shared memory budget (the static part is ~30 KB)

// The transposed warp butterfly: NP (a power of 2, <= 32) values per lane are reduced across the warp with
// NP - 1 + (5 - log2 NP) shuffles instead of 5 NP (the shuffle pipe, not latency, bounds the plain form).  At each
// offset a lane keeps one half of its slots and sends the other half to its partner, so every slot is combined in
// the same tree as warp_sum / warp_max: the results are bitwise those of the per-slot butterflies.  On return a[0]
// holds slot (lane >> (5 - log2 NP)).
template <int NP>
__device__ __forceinline__ void warp_reduce_slots(double (&a)[NP], unsigned maxmask, unsigned minmask) {
    const int lane = threadIdx.x & 31;
    int base = 0;
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        const int o = 16 >> s;
        const int c = NP >> s;   // slots still held (compile time after unrolling)
        if (c >= 2) {
            const int h = c >> 1;
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < h; ++i) {
                const double send = up ? a[i] : a[i + h];
                const double keep = up ? a[i + h] : a[i];
                const double recv = __shfl_xor_sync(0xffffffffu, send, o);
                const int slot = base + (up ? h : 0) + i;
                a[i] = ((maxmask >> slot) & 1u) ? fmax(keep, recv) : ((minmask >> slot) & 1u) ? fmin(keep, recv) : keep + recv;
            }
            if (up) base += h;
        } else {
            const double recv = __shfl_xor_sync(0xffffffffu, a[0], o);
            a[0] = ((maxmask >> base) & 1u) ? fmax(a[0], recv) : ((minmask >> base) & 1u) ? fmin(a[0], recv) : a[0] + recv;
        }
    }
}
template <int N> struct SlotPad { static constexpr int NP = N <= 1 ? 1 : N <= 2 ? 2 : N <= 4 ? 4 : N <= 8 ? 8 : N <= 16 ? 16 : 32;
                                  static constexpr int SH = NP == 1 ? 5 : NP == 2 ? 4 : NP == 4 ? 3 : NP == 8 ? 2 : NP == 16 ? 1 : 0; };

// N values per thread -> per-block totals in part[(slot0 + k) * G + block] (sum, or max / min per mask bit); the
// block's own totals stay in sh_w[IR_W * N + k].  Launch with IR_W warps.
template <int N>
__device__ __forceinline__ void ir_block_partials(const double (&v)[N], unsigned maxmask, unsigned minmask,
                                                  double* sh_w, double* part, int slot0) {
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if constexpr (N <= 32) {
        constexpr int NP = SlotPad<N>::NP, SH = SlotPad<N>::SH;
        double a[NP];
#pragma unroll
        for (int k = 0; k < NP; ++k) a[k] = k < N ? v[k] : 0.0;
        warp_reduce_slots<NP>(a, maxmask, minmask);
        const int slot = lane >> SH;
        if ((lane & ((1 << SH) - 1)) == 0 && slot < N) sh_w[wid * N + slot] = a[0];
    } else {   // (cold paths: the lazy line-search trials)
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const double t = ((maxmask >> k) & 1u) ? warp_max(v[k]) : ((minmask >> k) & 1u) ? warp_min(v[k]) : warp_sum(v[k]);
            if (lane == 0) sh_w[wid * N + k] = t;
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        double x[IR_W];
#pragma unroll
        for (int w = 0; w < IR_W; ++w) x[w] = sh_w[w * N + k];   // all loads first, then the sums in warp order
        double t = x[0];
#pragma unroll
        for (int w = 1; w < IR_W; ++w) t = ((maxmask >> k) & 1u) ? fmax(t, x[w]) : ((minmask >> k) & 1u) ? fmin(t, x[w]) : t + x[w];
        part[(size_t)(slot0 + k) * gridDim.x + blockIdx.x] = t;
        sh_w[IR_W * N + k] = t;
    }
    __syncthreads();
}
// slots [s0, s0 + n) -> out[0 .. n) in shared memory, every block identically; a warp loads its (up to 2) slots
// before reducing them (one transposed butterfly for both), so the totals cost one round trip for n <= 2 W
__device__ __forceinline__ void ir_totals(const double* part, int s0, int n, unsigned maxmask, unsigned minmask,
                                          double* out) {
    const int W = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31, G = gridDim.x;
    for (int k0 = wid; k0 < n; k0 += 2 * W) {
        double v[2][5];
        int op[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k = k0 + h * W;
            op[h] = k >= n ? 0 : ((maxmask >> k) & 1u) ? 1 : ((minmask >> k) & 1u) ? 2 : 0;
            const double idn = op[h] == 2 ? __longlong_as_double(0x7ff0000000000000LL) : 0.0;
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                const int b = lane + 32 * j;
                v[h][j] = (k < n && b < G) ? ld_cg(part + (size_t)(s0 + k) * G + b) : idn;
            }
        }
        double a[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double t = v[h][0];
#pragma unroll
            for (int j = 1; j < 5; ++j) t = op[h] == 0 ? t + v[h][j] : op[h] == 1 ? fmax(t, v[h][j]) : fmin(t, v[h][j]);
            a[h] = t;
        }
        warp_reduce_slots<2>(a, (op[0] == 1 ? 1u : 0u) | (op[1] == 1 ? 2u : 0u), (op[0] == 2 ? 1u : 0u) | (op[1] == 2 ? 2u : 0u));
        const int k = k0 + (lane >> 4) * W;
        if ((lane & 15) == 0 && k < n) out[k] = a[0];
    }
    __syncthreads();
}

// Split grid barrier (the cooperative-groups algorithm with the arrival and the wait apart, so that block-local work
// overlaps the wait): block 0 adds 2^31 - (G - 1), every other block 1, so the counter's top bit flips exactly when the
// last block arrives; its low 31 bits return to their value (0) after every barrier.  Release fence before the
// arrival, acquire load in the wait, the block barrier on both sides.
__device__ __forceinline__ unsigned gbar_arrive(unsigned* ctr) {
    __syncthreads();
    unsigned old = 0u;
    if (threadIdx.x == 0) {
        __threadfence();
        old = atomicAdd(ctr, blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1u) : 1u);
    }
    return old;   // (thread 0)
}
__device__ __forceinline__ void gbar_wait(const unsigned* ctr, unsigned old) {
    if (threadIdx.x == 0) {
        unsigned v;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (((v ^ old) & 0x80000000u) == 0u);
    }
    __syncthreads();
}

// S phase producer (thread 0): the next chunk of my columns; with coef, columns with a zero coefficient are skipped
// (the first SST chunks are issued before the direction exists, without skipping)
struct SProducer {
    int p, p0, p1, noff, nnz4;
    const int2* ext;   // cached column extents of positions [p0, p0 + IR_QC)
    __device__ bool next(const Seg& S, const double* coef, SChunk& d) {
        while (p < p1) {
            int b, e;
            if (ext && p - p0 < IR_QC) { const int2 x = ext[p - p0]; b = x.x; e = x.y; }
            else { const int j = __ldg(S.list + p); b = __ldg(S.ptr + j); e = __ldg(S.ptr + j + 1); }
            const int start = b + noff;
            if ((coef && noff == 0 && coef[p - p0] == 0.0) || start >= e) { ++p; noff = 0; continue; }
            d.p = p;
            d.a = start & ~3;
            d.vb = start;
            d.cb = b;
            d.ve = min(e, d.a + IR_SCH);
            d.ce = max(d.a, min((d.ve + 3) & ~3, nnz4));
            d.ok = 1;
            if (d.ve == e) { ++p; noff = 0; } else noff = d.ve - b;
            return true;
        }
        return false;
    }
    __device__ void issue(const Seg& S, const SChunk& d, int st, int* s_idx, float* s_val, uint64_t* s_bar) const {
        fence_proxy_async();
        mbar_arrive_expect_tx(s_bar + st, (S.idx ? 8u : 4u) * (uint32_t)(d.ce - d.a));   // (dense X: values only)
        if (d.ce > d.a) {
            if (S.idx) bulk_g2s(s_idx + st * IR_SCH, S.idx + d.a, 4u * (uint32_t)(d.ce - d.a), s_bar + st);
            bulk_g2s(s_val + st * IR_SCH, S.val + d.a, 4u * (uint32_t)(d.ce - d.a), s_bar + st);
        }
    }
    // the first sst chunks of my columns (no skipping: issued before the direction exists)
    __device__ void prefetch(const Seg& S, int sst, SChunk* s_desc, int* s_idx, float* s_val, uint64_t* s_bar) {
        p = p0;
        noff = 0;
        for (int k = 0; k < sst; ++k) mbar_init(s_bar + k, 1);
        fence_mbar_init();
        for (int k = 0; k < sst; ++k) {
            SChunk d;
            if (next(S, nullptr, d)) { s_desc[k] = d; issue(S, d, k, s_idx, s_val, s_bar); }
            else s_desc[k].ok = 0;
        }
    }
};

// l1 trial differences for trials IR_NT0 .. ML_MAXLS - 1 on my positions -> block partials (rare: Armijo past 1/8)
__device__ __noinline__ void ir_lazy_l1(const Prm& P, const PosState& X, int q0, double b_last, double* sh_w,
                                        double* part) {
    double v[ML_MAXLS - IR_NT0];
#pragma unroll
    for (int k = 0; k < ML_MAXLS - IR_NT0; ++k) v[k] = 0.0;
    for (int k0 = threadIdx.x; k0 < q0; k0 += blockDim.x) {
        const double x = X.wA[k0] + X.d[k0], sp = X.s[k0], ax = fabs(x);
        double b = b_last;
#pragma unroll
        for (int k = 0; k < ML_MAXLS - IR_NT0; ++k) {
            b *= P.beta_ls;
            v[k] += fabs(x + b * sp) - ax;
        }
    }
    ir_block_partials<ML_MAXLS - IR_NT0>(v, 0u, 0u, sh_w, part, IR_SL1);
}

// R14-R18 second batch: l1 and loss differences of trials 4 .. max_ls - 1 (rare) -> block partials
__device__ __noinline__ void ir_outer_batch2(const Prm& P, const PosState& X, int q0, int r0, int r1, const double* xd_r,
                                             double* sh_w, double* part) {
    double v[2 * IR_NLS];
#pragma unroll
    for (int k = 0; k < 2 * IR_NLS; ++k) v[k] = 0.0;
    double a4 = 1.0;
    for (int t = 0; t < 4; ++t) a4 *= P.beta_ls;
    for (int k0 = threadIdx.x; k0 < q0; k0 += blockDim.x) {
        const double d = X.d[k0], w = X.wA[k0], aw = fabs(w);
        double a = a4;
#pragma unroll
        for (int k = 0; k < IR_NLS; ++k) { v[k] += fabs(w + a * d) - aw; a *= P.beta_ls; }
    }
    for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        const double zi = P.z[i], xd = xd_r[i - r0];
        double a = a4;
#pragma unroll
        for (int k = 0; k < IR_NLS; ++k) { v[IR_NLS + k] += dloss_i(P.y, P.b, i, zi, a * xd); a *= P.beta_ls; }
    }
    ir_block_partials<2 * IR_NLS>(v, 0u, 0u, sh_w, part, IR_SO2);
}
__device__ __forceinline__ void ir_trace(const Prm& P, Ctl* c, int outcome, int steps, double Fb, double Fa, double a) {
    if (c->ntrace < c->trace_cap) {
        TraceRow tr{c->level, outcome, steps, c->nA, (long long)c->nC, Fb, Fa, a};
        P.trace[c->ntrace] = tr;
    }
    c->ntrace += 1;
}

// BIG (m > SMALL_M): the m-vectors live in global memory: S scatters with 64-bit fixed-point reductions (integer
// addition: order-independent, so bitwise reproducible; scale from max |X| x max |coef| x the longest row) into Xu (Xzu) through
// per-warp TMA column rings, R takes my rows of Xu directly (and clears them), G gathers D o Xs (D o Xz) from L2 and
// applies beta at each column end.  The iteration structure, barriers, decisions and the tail are the same.
template <int GSCH, int GST, bool BIG, bool HVP = false>   // HVP: with the heavy-column path (ml_heavy.cuh)
__global__ void __launch_bounds__(256, 1) k_inner(Prm P, ASet AS, Seg S, int K, int inner_cg, long long* acc_sc,
                                                  long long* acc_hs) {
    unsigned long long ph_t = gtimer(), ph_acc[IR_PHN] = {};
    const unsigned long long ph_k0 = ph_t;
    int ph_its = 0;
    (void)ph_k0;
#ifdef IR_BLKDBG
    unsigned long long bd_t0 = 0, bd_s = 0, bd_g = 0;   // this block's S and G work (BIG), before the barriers
#endif
    extern __shared__ __align__(16) unsigned char smraw[];
    __shared__ double sh_w[IR_W * 2 * IR_NLS + 2 * IR_NLS];   // >= IR_W * N + N for every ir_block_partials<N>
    __shared__ double sh_t[12], sh_r[4], sh_l1[2 * IR_NLS];
    __shared__ int2 col_ext[IR_QC];
    __shared__ double pos_sh[7][IR_QS];   // wA gA hA d Hd s u of my positions (q <= IR_QS)
    __shared__ double row_sh[4][IR_RS];   // D, X s, X z, X d of my rows
    __shared__ int s_res;                 // small m: all my column chunks stay in the S ring for the whole launch
    constexpr int SST = ir_sst(GSCH);
    cg::grid_group grid = cg::this_grid();
    Ctl* c = P.ctl;
    if (c->skip) {   // grid-uniform: converged at R2 (or a converged level): the relaxation's trace row
        if (blockIdx.x == 0 && threadIdx.x == 0 && !c->skipped)
            ir_trace(P, c, c->outcome, 0, c->F, c->F, 0.0);
        return;
    }
    const int m = P.m, G = gridDim.x;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nA = c->nA;
    const int ph_off = nA < 2048 ? 0 : IR_PHN / 2;
    // balanced contiguous position ranges: nA / G each, one more for the first nA % G blocks (the coarse free sets
    // are written interleaved by k_gather_small, so that a block's range holds every G-th column of the level)
    const int qb = nA / G, rb = nA % G;
    const int p0 = (int)blockIdx.x * qb + min((int)blockIdx.x, rb), p1 = p0 + qb + ((int)blockIdx.x < rb ? 1 : 0);
    const int R = (m + G - 1) / G;
    const int r0 = min(m, (int)blockIdx.x * R), r1 = min(m, r0 + R);
    double* part = P.irpart;
    double* xs_sh = reinterpret_cast<double*>(smraw + ir_ring_bytes<GSCH, GST>());   // X_A s of my columns, later sv
    double* xz_sh = xs_sh + m;                                                 // X_A z of my columns
    double* parts = P.parts;                                              // [G][m] block partials of X_A s
    double* zparts = P.parts + (size_t)G * m;                             // [G][m] block partials of X_A z
    // S ring (block-shared)
    int* s_idx = reinterpret_cast<int*>(smraw);
    float* s_val = reinterpret_cast<float*>(smraw + (size_t)4 * SST * IR_SCH);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smraw + (size_t)8 * SST * IR_SCH);
    SChunk* s_desc = reinterpret_cast<SChunk*>(s_bar + SST);
    // G rings (per warp; alias the S ring, used after it)
    unsigned char* gbase = smraw + (size_t)wid * stream_warp_bytes<GSCH, GST>(0);
    uint64_t* g_bar = reinterpret_cast<uint64_t*>(gbase + 8 * GST * GSCH);
    uint32_t g_phase = 0u;
    long long nsc = 0, nhs = 0;

    const int q0 = p1 - p0;
    PosState X;
    if (!BIG && q0 <= IR_QS) {
        X = PosState{pos_sh[0], pos_sh[1], pos_sh[2], pos_sh[3], pos_sh[4], pos_sh[5], pos_sh[6]};
        for (int k = threadIdx.x; k < q0; k += blockDim.x) {
            pos_sh[0][k] = AS.wA[p0 + k];
            pos_sh[1][k] = AS.gA[p0 + k];
            pos_sh[2][k] = AS.hA[p0 + k];
        }
    } else {
        X = PosState{AS.wA + p0, AS.gA + p0, AS.hA + p0, AS.d + p0, AS.Hd + p0, AS.s + p0, AS.u + p0};
    }
    for (int k = threadIdx.x; k < q0; k += blockDim.x) { X.d[k] = 0.0; X.Hd[k] = 0.0; }
    double* rD_r = row_sh[0];   // (not used when BIG: D from P.rD)
    double* xs_r = BIG ? P.Xs + r0 : row_sh[1];
    double* xz_r = BIG ? P.Xz + r0 : row_sh[2];
    double* xd_r = BIG ? P.Xd + r0 : row_sh[3];
    for (int k = threadIdx.x; k < r1 - r0; k += blockDim.x) {
        if (!BIG) rD_r[k] = P.rD[r0 + k].y;
        xs_r[k] = 0.0;
        xz_r[k] = 0.0;
        xd_r[k] = 0.0;
    }

    int next_pcd = 1, cg_restart = 1, acc_steps = 0, stop = 0, pcd = 1, zs = 0, ksnap = 0;   // R6: PCD first
    double fq = 1.0, fqi = 1.0;   // BIG: this iteration's fixed-point scale of X_A s (and its inverse)
    double beta = 0.0, bk = 0.0, bq = 0.0, bcg = 0.0, rz = 0.0, rz_prev = 0.0, slope = 0.0, ss = 0.0, ps = 0.0;
    double sHs = 0.0, vq = 0.0;
    const double vmax_C = c->vmax;
    double bt[IR_NT0];
    bt[0] = 1.0;
#pragma unroll
    for (int t = 1; t < IR_NT0; ++t) bt[t] = bt[t - 1] * P.beta_ls;
    for (int p = p0 + threadIdx.x; p < min(p1, p0 + IR_QC); p += blockDim.x) {
        const int j = __ldg(S.list + p);
        col_ext[p - p0] = make_int2(__ldg(S.ptr + j), __ldg(S.ptr + j + 1));
    }
    __syncthreads();
    SProducer pr{p0, p0, p1, 0, (int)(S.nnz & ~3LL), col_ext};   // the S-ring producer's state
    int u0 = 0, u1 = 0;   // BIG: my range of column units (balanced by nonzeros across blocks)
    int nU = 0;           // BIG: all units (the S and G streams claim them dynamically, Ctl::s_ctr / g_ctr)
    int nUS = 0, us0 = 0, us1 = 0;   // BIG: the units of the X_A s stream (heavy mode: the light columns' only)
    // BIG, heavy-column path (ml_heavy.cuh): on for this relaxation when A holds enough of H's nonzeros; then the
    // X_A s products of A's heavy columns come from the S copy (their column units are skipped by the S stream)
    bool hvm = false;
    long long hv_nz = 0;     // nonzeros of A's heavy columns (the algorithmic count of the heavy pass)
    if constexpr (BIG) {
        const bool hvb = HVP && P.hv.on != 0;
        int nu_loc = 0, nz_loc = 0, nu_l = 0, nz_l = 0;
        double nzh = 0.0;
        for (int k = threadIdx.x; k < q0; k += blockDim.x) {
            int b, e, j;
            if (k < IR_QC) { b = col_ext[k].x; e = col_ext[k].y; j = hvb ? __ldg(S.list + p0 + k) : 0; }
            else { j = __ldg(S.list + p0 + k); b = __ldg(S.ptr + j); e = __ldg(S.ptr + j + 1); }
            const int nu1 = max(1, (e - b + IR_UNIT - 1) / IR_UNIT);
            nu_loc += nu1;
            nz_loc += e - b + IR_UCOST * nu1;
            const int h = hvb ? __ldg(P.hv.hid + j) : -1;
            if (hvb) P.hv.phid[p0 + k] = h;
            if (h < 0) { nu_l += nu1; nz_l += e - b + IR_UCOST * nu1; }
            else nzh += (double)(e - b);
        }
        if (hvb) {   // no heavy column of A has a coefficient yet (D writes those of A's)
            for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < HV_HMAX; i += G * blockDim.x) P.hv.sH[i] = 0.0;
        }
        {
            const double v[5] = {(double)nu_loc, (double)nz_loc, (double)nu_l, (double)nz_l, nzh};
            ir_block_partials<5>(v, 0u, 0u, sh_w, part, IR_SU);
        }
        grid.sync();
        // unit sequence: the light columns' units first, then (heavy mode) the heavy columns' (the X_A s stream
        // covers only the first part; the H sigma stream all); each part in position order
        __shared__ long long s_uoff[10];
        if (wid == 0) {   // the heavy decision; my offsets in both parts of the unit and cost sequences, their totals
            double hz = 0.0;
            for (int b = lane; b < G; b += 32) hz += ld_cg(part + (size_t)(IR_SU + 4) * G + b);
            hz = warp_sum(hz);   // (integers below 2^53: exact in any order)
            const bool on = hvb && (P.hv.mode == 1 || (P.hv.mode == 0 && hz >= P.hv.frac * (double)P.hv.nnzh)) && hz > 0.0;
            long long off[2] = {0, 0}, tot[2] = {0, 0}, zoff[2] = {0, 0}, ztot[2] = {0, 0};
            for (int b0 = 0; b0 < G; b0 += 32) {
                const int b = b0 + lane;
                const long long xa = b < G ? (long long)ld_cg(part + (size_t)IR_SU * G + b) : 0;
                const long long za = b < G ? (long long)ld_cg(part + (size_t)(IR_SU + 1) * G + b) : 0;
                const long long xl = !on ? xa : b < G ? (long long)ld_cg(part + (size_t)(IR_SU + 2) * G + b) : 0;
                const long long zl = !on ? za : b < G ? (long long)ld_cg(part + (size_t)(IR_SU + 3) * G + b) : 0;
                const long long x[2] = {xl, xa - xl}, z[2] = {zl, za - zl};
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    off[h] += warp_sum_ll(b < (int)blockIdx.x ? x[h] : 0);
                    tot[h] += warp_sum_ll(x[h]);
                    zoff[h] += warp_sum_ll(b < (int)blockIdx.x ? z[h] : 0);
                    ztot[h] += warp_sum_ll(z[h]);
                }
            }
            if (lane == 0) {
#pragma unroll
                for (int h = 0; h < 2; ++h) { s_uoff[4 * h] = off[h]; s_uoff[4 * h + 1] = tot[h]; s_uoff[4 * h + 2] = zoff[h]; s_uoff[4 * h + 3] = ztot[h]; }
                s_uoff[8] = on ? (long long)hz : -1;
            }
        }
        __syncthreads();
        hvm = s_uoff[8] >= 0;
        hv_nz = hvm ? s_uoff[8] : 0;
        if (hvm && blockIdx.x == 0 && threadIdx.x == 0) c->hv_relax += 1;
        const int NUL = (int)s_uoff[1];                 // units of the first (light) part
        const long long NZL = s_uoff[3];
        const int NU = NUL + (int)s_uoff[5];
        const long long NZ = NZL + s_uoff[7];
        int base[2] = {(int)s_uoff[0], NUL + (int)s_uoff[4]};
        long long zbase[2] = {s_uoff[2], NZL + s_uoff[6]};
        for (int k00 = 0; k00 < q0; k00 += blockDim.x) {   // my positions in order: their units
            const int k = k00 + threadIdx.x;
            int b = 0, e = 0, nu = 0, hp = 0;
            if (k < q0) {
                if (k < IR_QC) { b = col_ext[k].x; e = col_ext[k].y; }
                else { const int j = __ldg(S.list + p0 + k); b = __ldg(S.ptr + j); e = __ldg(S.ptr + j + 1); }
                nu = max(1, (e - b + IR_UNIT - 1) / IR_UNIT);
                hp = (hvm && P.hv.phid[p0 + k] >= 0) ? 1 : 0;
            }
            const long long cost = (long long)(e - b) + (long long)IR_UCOST * nu;
            int incl[2] = {hp ? 0 : nu, hp ? nu : 0};
            long long zincl[2] = {hp ? 0 : cost, hp ? cost : 0};
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int t = __shfl_up_sync(0xffffffffu, incl[h], o);
                    const long long tz = __shfl_up_sync(0xffffffffu, zincl[h], o);
                    if (lane >= o) { incl[h] += t; zincl[h] += tz; }
                }
            }
            __shared__ int s_wsum[2][IR_W];
            __shared__ long long s_zsum[2][IR_W];
            if (lane == 31) {
#pragma unroll
                for (int h = 0; h < 2; ++h) { s_wsum[h][wid] = incl[h]; s_zsum[h][wid] = zincl[h]; }
            }
            __syncthreads();
            int woff[2] = {0, 0}, wtot[2] = {0, 0};
            long long zwoff[2] = {0, 0}, zwtot[2] = {0, 0};
            for (int w = 0; w < IR_W; ++w) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (w < wid) { woff[h] += s_wsum[h][w]; zwoff[h] += s_zsum[h][w]; }
                    wtot[h] += s_wsum[h][w];
                    zwtot[h] += s_zsum[h][w];
                }
            }
            if (k < q0) {
                const int us = base[hp] + woff[hp] + incl[hp] - nu;
                const long long zs0 = zbase[hp] + zwoff[hp] + zincl[hp] - cost;
                P.ustart[p0 + k] = us;
                P.uend[p0 + k] = us + nu;
                for (int c2 = 0; c2 < nu; ++c2) {
                    P.uext[us + c2] = make_int2(b + c2 * IR_UNIT, min(e, b + (c2 + 1) * IR_UNIT));
                    P.upos[us + c2] = p0 + k;
                    P.unz[us + c2] = zs0 + (long long)c2 * (IR_UNIT + IR_UCOST);   // weighted cost before this unit
                }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) { base[h] += wtot[h]; zbase[h] += zwtot[h]; }
            __syncthreads();
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) { P.unz[NU] = NZ; c->s_ctr = 0u; c->g_ctr = 0u; c->zcnt = 0u; }
        grid.sync();
        nU = NU;
        nUS = NUL;
        if (threadIdx.x == 0) {   // my units: those starting in my share [b T, (b+1) T) of the costs (S: of the first part)
            for (int q = 0; q < 2; ++q) {
                const int n_ = q ? NUL : NU;
                const long long T = ((q ? NZL : NZ) + G - 1) / G;
                for (int h = 0; h < 2; ++h) {
                    const long long target = (long long)(blockIdx.x + h) * T;
                    int lo = 0, hi = n_;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (ld_cg(P.unz + mid) >= target) hi = mid; else lo = mid + 1;
                    }
                    s_uoff[2 * q + h] = (blockIdx.x + h == G) ? n_ : lo;
                }
            }
        }
        __syncthreads();
        u0 = (int)s_uoff[0];
        u1 = (int)s_uoff[1];
        us0 = (int)s_uoff[2];
        us1 = (int)s_uoff[3];
    }
    for (int it = 0; it < K; ++it) {
        pcd = next_pcd;
        ColStream<GSCH, GST> csG;   // the G rings: prefetched during B1 (small m) or B2 (BIG)
        const bool need_hs = it < K - 1;
        ph_its += 1;
        const bool producer = threadIdx.x == blockDim.x - 32;   // lane 0 of the last warp (idle in D for small q)
        // small m: the first S-ring prefetch decides residency -- if it holds all my column chunks, S and G read
        // them from shared memory for the whole relaxation (no TMA, no ring refills, G block-cooperative)
        if (!BIG && producer && (it == 0 || !s_res)) {
            pr.prefetch(S, SST, s_desc, s_idx, s_val, s_bar);   // overlaps the direction
            if (it == 0) s_res = pr.p >= p1;
        }
        PH_SUB(0);
        // ------------------------------------------------ D: direction on my positions
        int my_z = 0;
        {
            double v[12];
#pragma unroll
            for (int k = 0; k < 12; ++k) v[k] = 0.0;
            for (int k = threadIdx.x; k < q0; k += blockDim.x) {
                const double x = X.wA[k] + X.d[k], pj = X.gA[k] + X.Hd[k], hh = X.hA[k];
                if (pcd) {   // R6 (Eq. 5, D = diag H + eps) + the zeroing part z (Q27)
                    const double sp = soft(x - pj / hh, P.lam / hh) - x;
                    X.s[k] = sp;
                    const double zp = (P.pcd_snap && x != 0.0 && x + sp == 0.0) ? sp : 0.0;
                    X.u[k] = zp;
                    const double vv = (x != 0.0) ? pj + P.lam * sgn(x) : soft(pj, P.lam);
                    v[0] += pj * sp;
                    v[1] += sp * sp;
                    v[2] += pj * zp;
                    v[3] += fabs(zp);
                    v[4] += zp * zp;
                    v[5] += (zp != 0.0) ? 1.0 : 0.0;
                    const double ax = fabs(x);
#pragma unroll
                    for (int t = 0; t < IR_NT0; ++t) v[6 + t] += fabs(x + bt[t] * sp) - ax;
                    v[10] = fmax(v[10], fabs(sp));
                    v[11] = fmax(v[11], fabs(vv));
                } else {     // R6' (Q9b): orthant residual, preconditioned by diag H + eps
                    const double gx = (x != 0.0) ? pj + P.lam * sgn(x) : 0.0;
                    const double u = (x != 0.0) ? -gx / hh : 0.0;
                    X.u[k] = u;
                    const double sp = X.s[k];
                    const double vv = (x != 0.0) ? gx : soft(pj, P.lam);
                    v[0] += hh * u * u;
                    v[1] += gx * u;
                    v[2] += gx * sp;
                    v[3] += u * u;
                    v[4] += u * sp;
                    v[5] += sp * sp;
                    v[10] = fmax(v[10], fabs(u));   // (max |coef| of the X_A u pass: its fixed-point scale)
                    v[11] = fmax(v[11], fabs(vv));
                }
                if (BIG && hvm) {   // a heavy column of A: its S coefficient for the S copy; a zeroing one's units for
                    const int h = P.hv.phid[p0 + k];      // the z pass (X_A z through the units: z is rare)
                    if (h >= 0) {
                        P.hv.sH[h] = pcd ? X.s[k] : X.u[k];
                        if (pcd && X.u[k] != 0.0) {
                            const int ua = P.ustart[p0 + k], ub = P.uend[p0 + k];
                            const unsigned zb = atomicAdd(&c->zcnt, (unsigned)(ub - ua));
                            for (int u = ua; u < ub; ++u) P.hv.zunits[zb + (unsigned)(u - ua)] = u;
                        }
                    }
                }
            }
            PH_SUB(1);
            ir_block_partials<12>(v, IR_DMAX, 0u, sh_w, part, IR_SD);
            my_z = pcd && sh_w[IR_W * 12 + 5] > 0.0;
        }
        const bool resident = !BIG && s_res;   // (block-uniform; s_res is visible after the partials' barriers)
        PH_MARK(0);
        if (BIG) grid.sync();   // the units of my stream may belong to other blocks' positions
        if (BIG) {   // X_A s in fixed point: |(X_A coef)_i| <= maxrow * max|X| * max|coef| < 2^62 q (every block alike)
            __shared__ double s_q[2];
            if (wid == 0) {
                double cm = 0.0;
                for (int b = lane; b < G; b += 32) cm = fmax(cm, ld_cg(part + (size_t)(IR_SD + 10) * G + b));
                cm = warp_max(cm);
                if (lane == 0) {
                    const double bound = (double)c->maxrow * c->xmax * cm;
                    int ex = 0;
                    frexp(bound, &ex);
                    const bool ok = bound > 0.0 && isfinite(bound);
                    s_q[0] = ok ? ldexp(1.0, 62 - ex) : 1.0;
                    s_q[1] = ok ? ldexp(1.0, ex - 62) : 1.0;
                }
            }
            __syncthreads();
            fq = s_q[0];
            fqi = s_q[1];
        }
#ifdef IR_BLKDBG
        __syncthreads();
        bd_t0 = gtimer();
#endif
        // ------------------------------------------------ S: X_A coef (and X_A z) over my columns
        if constexpr (BIG) {   // per-warp rings, fixed-point reductions into Xu / Xzu (kept zero between uses)
            const double* coef = pcd ? AS.s : AS.u;
            if constexpr (HVP) if (hvm) {   // heavy columns first: s_H in shared memory, the S copy's row sums
                double* sHs = reinterpret_cast<double*>(smraw + HV_SH_OFF);
                for (int i = threadIdx.x; i < P.hv.nh; i += blockDim.x) sHs[i] = ld_cg(P.hv.sH + i);
                __syncthreads();
#ifdef IR_HVDBG
                const unsigned long long hv_t0 = gtimer();
#endif
                hv_sweep(P.hv, c->tph + 2);
                // X_A z of the zeroing heavy columns (the snap path's z = s there): their units, a warp each, with the
                // same fixed-point reductions as the column stream (order-independent)
                const unsigned nzu = ld_cg(&c->zcnt);
                for (unsigned k = (unsigned)(blockIdx.x * IR_W + wid); k < nzu; k += (unsigned)(G * IR_W)) {
                    const int u = ld_cg(P.hv.zunits + k);
                    const int2 ex = ld_cg(P.uext + u);
                    const double cf = ld_cg(coef + ld_cg(P.upos + u));
                    int e = ex.x + lane;
                    for (; e + 96 < ex.y; e += 128) {   // four elements per lane in flight (ncu: 2 % of a snap-path
                                                        // launch waited here on one dependent load at a time)
                        int r[4];
                        double xv[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) { r[u] = __ldg(S.idx + e + 32 * u); xv[u] = (double)__ldg(S.val + e + 32 * u) * cf; }
#pragma unroll
                        for (int u = 0; u < 4; ++u) red_add_fixed(P.Xzu + r[u], xv[u], fq);
                    }
                    for (; e < ex.y; e += 32)
                        red_add_fixed(P.Xzu + __ldg(S.idx + e), (double)__ldg(S.val + e) * cf, fq);
                }
                __syncthreads();   // (the rings' shared memory is reused by the column stream below)
                if (blockIdx.x == 0 && threadIdx.x == 0) nsc += hv_nz;
#ifdef IR_HVDBG   // (block 0's heavy S time in slot 0, heavy G time in slot 1: the small-|A| D / S slots)
                if (blockIdx.x == 0 && threadIdx.x == 0) ph_acc[0] += gtimer() - hv_t0;
#endif
            }
            if (lane == 0) {
                for (int k = 0; k < GST; ++k) mbar_init(g_bar + k, 1);
                fence_mbar_init();
            }
            __syncwarp();
            g_phase = 0u;   // fresh barriers
            ColStream<GSCH, GST, true> cs;
            cs.streamed = 0;
            cs.segs = 0;
            // a unit's coefficient and zeroing flag come with its descriptor (loaded for a whole batch of units at once:
            // two dependent L2 round trips per batch, not per chunk of a few hundred nonzeros); zero-coefficient units
            // are not streamed at all
            cs.upos = P.upos;
            cs.zsrc = (pcd && P.pcd_snap) ? AS.u : nullptr;
            if (nUS >= IR_DYN * G * IR_W || P.dyn) {   // many units per warp: dynamic claims (no block waits on another
                                                        // at B1)
                cs.claim = &c->s_ctr;
                stream_begin(cs, S, coef, 0, nUS, gbase, P.uext, nUS);
            } else {
                stream_begin(cs, S, coef, us0, us1, gbase, P.uext + us0, us1 - us0);
            }
            int stg = 0;
            while (true) {
                const ChunkDesc dsc = cs.desc[stg];
                if (dsc.cf == 0.0) break;
                mbar_wait(cs.bar + stg, (g_phase >> stg) & 1u);
                g_phase ^= 1u << stg;
                const double cf = dsc.cf;
                if (cf != 0.0) {
                    const int zf = dsc.pad;   // z_p = s_p on a zeroing column (pcd && pcd_snap && u_p != 0)
                    const int* ci = S.idx ? cs.sidx + stg * GSCH - dsc.a : S.rowtab - dsc.cb;
                    const float* cv = cs.sval + stg * GSCH - dsc.a;
                    const int kend = min(dsc.ve, dsc.ce);
                    int k = dsc.vb + lane;
                    for (; k + 96 < kend; k += 128) {   // 4 reductions per lane issued back to back
                        int r[4];
                        double xv[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) { r[u] = ci[k + 32 * u]; xv[u] = (double)cv[k + 32 * u] * cf; }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            red_add_fixed(P.Xu + r[u], xv[u], fq);
                            if (zf) red_add_fixed(P.Xzu + r[u], xv[u], fq);
                        }
                    }
                    for (; k < kend; k += 32) {
                        const int r = ci[k];
                        const double xv = (double)cv[k] * cf;
                        red_add_fixed(P.Xu + r, xv, fq);
                        if (zf) red_add_fixed(P.Xzu + r, xv, fq);
                    }
                    for (; k < dsc.ve; k += 32) {
                        const int r = seg_idx(S, k, dsc.cb);
                        const double xv = (double)__ldg(S.val + k) * cf;
                        red_add_fixed(P.Xu + r, xv, fq);
                        if (zf) red_add_fixed(P.Xzu + r, xv, fq);
                    }
                }
                __syncwarp();
                ChunkDesc nd;
                const bool ok = cs.next(nd);
                if (lane == 0) {
                    if (ok) { cs.desc[stg] = nd; cs.issue(stg, nd); }
                    else cs.desc[stg].cf = 0.0;
                }
                __syncwarp();
                stg = (stg + 1) % GST;
            }
            nsc += cs.streamed;
            __syncwarp();
            if (lane == 0)
                for (int k = 0; k < GST; ++k) mbar_inval(g_bar + k);
        } else {
            const double* coef = pcd ? X.s : X.u;
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                xs_sh[i] = 0.0;
                if (my_z) xz_sh[i] = 0.0;
            }
            __syncthreads();
            PH_SUB(2);
            uint32_t s_phase = 0u;
            for (int st = 0, used = 0;; st = (st + 1) % SST, ++used) {
                if (resident && used == SST) break;   // (a resident ring is read once per pass, never refilled)
                const SChunk d = s_desc[st];
                if (!d.ok) break;
                PH_SUB(3);
                mbar_wait(s_bar + st, (s_phase >> st) & 1u);
                PH_SUB(7);
                s_phase ^= 1u << st;
                const double cf = coef[d.p - p0];
                if (cf != 0.0) {
                    const int zf = my_z && X.u[d.p - p0] != 0.0;   // z_p = s_p on a zeroing column
                    const int* ci = S.idx ? s_idx + st * IR_SCH - d.a : S.rowtab - d.cb;
                    const float* cv = s_val + st * IR_SCH - d.a;
                    const int kend = min(d.ve, d.ce);
                    // rows are distinct within a column: all loads of a batch are issued before its stores.  The
                    // staged part [vb, kend) has branch-free (predicated) loads; the global tail past the last
                    // 16-byte boundary of X (at most 3 nonzeros) is a separate loop
                    constexpr int UB = IR_SCH / 256;
                    for (int k0 = d.vb + threadIdx.x; k0 < kend; k0 += UB * (int)blockDim.x) {
                        int r[UB];
                        double xv[UB], a[UB];
#pragma unroll
                        for (int u = 0; u < UB; ++u) {
                            const int k = k0 + u * blockDim.x;
                            r[u] = -1;
                            xv[u] = 0.0;
                            if (k < kend) { r[u] = ci[k]; xv[u] = (double)cv[k]; }
                        }
#pragma unroll
                        for (int u = 0; u < UB; ++u) a[u] = r[u] >= 0 ? xs_sh[r[u]] : 0.0;
#pragma unroll
                        for (int u = 0; u < UB; ++u)
                            if (r[u] >= 0) xs_sh[r[u]] = fma(xv[u], cf, a[u]);
                        if (zf) {
#pragma unroll
                            for (int u = 0; u < UB; ++u) a[u] = r[u] >= 0 ? xz_sh[r[u]] : 0.0;
#pragma unroll
                            for (int u = 0; u < UB; ++u)
                                if (r[u] >= 0) xz_sh[r[u]] = fma(xv[u], cf, a[u]);
                        }
                    }
                    for (int k = max(kend, d.vb) + threadIdx.x; k < d.ve; k += blockDim.x) {   // (a chunk may start past kend)
                        const int r = seg_idx(S, k, d.cb);
                        const double xv = (double)__ldg(S.val + k);
                        xs_sh[r] = fma(xv, cf, xs_sh[r]);
                        if (zf) xz_sh[r] = fma(xv, cf, xz_sh[r]);
                    }
                    if (threadIdx.x == 0) nsc += d.ve - d.vb;
                }
                PH_SUB(4);
                __syncthreads();   // stage st consumed by every warp
                PH_SUB(5);
                if (producer && !resident) {
                    SChunk nd;
                    if (pr.next(S, coef, nd)) { s_desc[st] = nd; pr.issue(S, nd, st, s_idx, s_val, s_bar); }
                    else s_desc[st].ok = 0;
                }
                PH_SUB(6);
            }
            __syncthreads();
            PH_SUB(3);
            if (producer && !resident)
                for (int k = 0; k < SST; ++k) mbar_inval(s_bar + k);
            // my block partials (a block without zeroing columns writes zeros for X_A z)
            const int zpart = pcd && P.pcd_snap;
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                parts[(size_t)blockIdx.x * m + i] = xs_sh[i];
                if (zpart) zparts[(size_t)blockIdx.x * m + i] = my_z ? xz_sh[i] : 0.0;
            }
        }
#ifdef IR_BLKDBG
        if (BIG) { __syncthreads(); bd_s += gtimer() - bd_t0; }
#endif
        PH_MARK(1);
        if constexpr (BIG) {
            grid.sync();   // B1
            if (blockIdx.x == 0 && threadIdx.x == 0) { c->s_ctr = 0u; c->zcnt = 0u; }   // (S claims and z units done)
        }
        else {   // B1, split: the G rings (aliasing the consumed S ring) are set up and issued while it completes
            const unsigned bar_old = gbar_arrive(&c->gbar);
            if (need_hs && !resident) {
                if (lane == 0) {
                    for (int k = 0; k < GST; ++k) mbar_init(g_bar + k, 1);
                    fence_mbar_init();
                }
                __syncwarp();
                g_phase = 0u;
                csG.streamed = 0;
                csG.segs = 0;
                stream_begin(csG, S, nullptr, p0, p1, gbase, col_ext, IR_QC);
            }
            gbar_wait(&c->gbar, bar_old);
        }
        ir_totals(part, IR_SD, 12, IR_DMAX, 0u, sh_t);
        PH_MARK(2);
        int nzero = 0;
        double pz = 0.0, Z1 = 0.0, zz = 0.0;
        if (pcd) {
            ps = sh_t[0]; ss = sh_t[1]; pz = sh_t[2]; Z1 = sh_t[3]; zz = sh_t[4]; nzero = (int)sh_t[5]; vq = sh_t[11];
            stop = (it > 0 && P.eta > 0.0 && vq <= P.eta * vmax_C) || sh_t[10] == 0.0;   // R13, R7
            bcg = 0.0;
        } else {
            rz = sh_t[0]; vq = sh_t[11];
            stop = (it > 0 && P.eta > 0.0 && vq <= P.eta * vmax_C) || rz == 0.0;
            if (!stop) {
                bcg = cg_restart ? 0.0 : rz / rz_prev;
                slope = sh_t[1] + bcg * sh_t[2];
                ss = sh_t[3] + 2.0 * bcg * sh_t[4] + bcg * bcg * sh_t[5];
            }
        }
        if (stop) {
            if (BIG)   // the scatter of this iteration is complete (B1): clear my rows for the next relaxation
                for (int k = threadIdx.x; k < r1 - r0; k += blockDim.x) { P.Xu[r0 + k] = 0.0; P.Xzu[r0 + k] = 0.0; }
            else if (need_hs && !resident) {   // drain the prefetched G rings
                for (int stg2 = 0; stg2 < GST; ++stg2)
                    if (csG.desc[stg2].cf != 0.0) { mbar_wait(csG.bar + stg2, (g_phase >> stg2) & 1u); g_phase ^= 1u << stg2; }
                __syncwarp();
                if (lane == 0)
                    for (int k = 0; k < GST; ++k) mbar_inval(g_bar + k);
            }
            break;
        }
        const int dual = pcd && nzero > 0;
        // ------------------------------------------------ R: my rows; PCD-CG: s and the first kink on my positions
        {
            double a_ss = 0.0, a_sz = 0.0, a_zz = 0.0;
            const int nr = r1 - r0;
            if (BIG) {   // my rows of Xu (Xzu), cleared for the next scatter; sv = D o Xs, svz = D o Xz for the G phase
                for (int k0 = threadIdx.x; k0 < nr; k0 += IR_RB * blockDim.x) {
                    double xu[IR_RB], xzu[IR_RB], xo[IR_RB], dd[IR_RB];
#pragma unroll
                    for (int u = 0; u < IR_RB; ++u) {
                        const int k = k0 + u * blockDim.x;
                        const bool in = k < nr;
                        xu[u] = in ? ld_fixed(P.Xu + r0 + k, fqi) + (hvm ? ld_cg(P.hv.Xh + r0 + k) : 0.0) : 0.0;
                        xzu[u] = (in && dual) ? ld_fixed(P.Xzu + r0 + k, fqi) : 0.0;
                        xo[u] = (in && !pcd) ? xs_r[k] : 0.0;
                        dd[u] = in ? P.rD[r0 + k].y : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < IR_RB; ++u) {
                        const int k = k0 + u * blockDim.x;
                        if (k >= nr) break;
                        const double xs = pcd ? xu[u] : xu[u] + bcg * xo[u];
                        P.Xu[r0 + k] = 0.0;
                        xs_r[k] = xs;
                        P.sv[r0 + k] = dd[u] * xs;
                        if (dual) {   // (D o Xs, D o Xz) side by side: the snap path's G phase gathers both with one sector
                            P.Xzu[r0 + k] = 0.0;
                            xz_r[k] = xzu[u];
                            P.sv2[r0 + k] = make_double2(dd[u] * xs, dd[u] * xzu[u]);
                        }
                        a_ss += dd[u] * xs * xs;
                        a_sz += dd[u] * xs * xzu[u];
                        a_zz += dd[u] * xzu[u] * xzu[u];
                    }
                }
            } else if (nr > 0) {   // thread (group g, row rr) sums blocks g, g + ng, ...; then the groups in order
                const int ng = max(1, (int)blockDim.x / nr);
                const int g = threadIdx.x / nr, rr = threadIdx.x % nr;
                double t = 0.0, tz = 0.0;
                if (g < ng) {
                    const double* src = parts + r0 + rr;
                    const double* srz = zparts + r0 + rr;
                    for (int b0 = g; b0 < G; b0 += IR_RL * ng) {   // IR_RL loads in flight, summed in block order
                        double x[IR_RL], z[IR_RL];
#pragma unroll
                        for (int u = 0; u < IR_RL; ++u) {
                            const int b = b0 + u * ng;
                            x[u] = b < G ? ld_cg(src + (size_t)b * m) : 0.0;
                            z[u] = (dual && b < G) ? ld_cg(srz + (size_t)b * m) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < IR_RL; ++u) { t += x[u]; tz += z[u]; }
                    }
                    sh_w[threadIdx.x] = t;   // sh_w holds >= 2 * 256 doubles
                    sh_w[blockDim.x + threadIdx.x] = tz;
                }
                __syncthreads();
                for (int rr2 = threadIdx.x; rr2 < nr; rr2 += blockDim.x) {
                    double xs = 0.0, xz = 0.0;
                    for (int g2 = 0; g2 < ng; ++g2) {
                        xs += sh_w[g2 * nr + rr2];
                        xz += sh_w[blockDim.x + g2 * nr + rr2];
                    }
                    const int i = r0 + rr2;
                    if (!pcd) xs += bcg * xs_r[rr2];
                    xs_r[rr2] = xs;
                    P.Xs[i] = xs;
                    if (dual) { xz_r[rr2] = xz; P.Xz[i] = xz; }
                    const double D = rD_r[rr2];
                    a_ss += D * xs * xs;
                    a_sz += D * xs * xz;
                    a_zz += D * xz * xz;
                }
                __syncthreads();   // group sums read before sh_w is reused by the block partials
            }
            double kmin = __longlong_as_double(0x7ff0000000000000LL);
            if (!pcd)
                for (int k = threadIdx.x; k < q0; k += blockDim.x) {
                    const double sp = X.u[k] + bcg * X.s[k];
                    X.s[k] = sp;
                    const double x = X.wA[k] + X.d[k];
                    if (x * sp < 0.0) kmin = fmin(kmin, -x / sp);
                }
            const double v[4] = {a_ss, a_sz, a_zz, kmin};
            ir_block_partials<4>(v, 0u, 1u << 3, sh_w, part, IR_SR);
        }
        // BIG: prefetch the G rings (X_A's columns do not depend on the step) across the barrier
        if (BIG && need_hs) {
            if (lane == 0) {
                for (int k = 0; k < GST; ++k) mbar_init(g_bar + k, 1);
                fence_mbar_init();
            }
            __syncwarp();
            g_phase = 0u;
            csG.streamed = 0;
            csG.segs = 0;
            if (nU >= IR_DYN * G * IR_W || P.dyn) {
                csG.claim = &c->g_ctr;
                stream_begin(csG, S, nullptr, 0, nU, gbase, P.uext, nU);
            } else {
                stream_begin(csG, S, nullptr, u0, u1, gbase, P.uext + u0, u1 - u0);
            }
        }
        PH_MARK(3);
        grid.sync();   // B2
        ir_totals(part, IR_SR, 4, 0u, 1u << 3, sh_r);
        // ------------------------------------------------ step decision, identical in every block
        int have_l1 = 0;
        auto l1 = [&](int t) -> double {   // sum_p |x + beta^t s| - |x| (trials >= IR_NT0 on demand: one more barrier)
            if (t < IR_NT0) return sh_t[6 + t];
            if (!have_l1) {
                ir_lazy_l1(P, X, q0, bt[IR_NT0 - 1], sh_w, part);
                grid.sync();
                ir_totals(part, IR_SL1, ML_MAXLS - IR_NT0, 0u, 0u, sh_l1);
                have_l1 = 1;
            }
            return sh_l1[t - IR_NT0];
        };
        zs = 0;
        ksnap = 0;
        if (pcd) {   // R10: model Armijo, snap path first (Q27), then the plain path
            sHs = sh_r[0] + P.eps_h * ss;
            const double zHs = sh_r[1] + P.eps_h * zz, zHz = sh_r[2] + P.eps_h * zz;
            const double delta = ps + P.lam * sh_t[6];
            double b = 1.0;
            int ok = 0;
            if (dual) {
                const double snHsn = sHs - 2.0 * zHs + zHz, snHz = zHs - zHz;
                for (int t = 0; t < P.max_ls; ++t, b *= P.beta_ls) {
                    const double dq = b * (ps - pz) + pz + 0.5 * (b * b * snHsn + 2.0 * b * snHz + zHz) +
                                      P.lam * (l1(t) - (1.0 - b) * Z1);
                    if (dq <= P.sigma_in * b * delta) { ok = 1; zs = 1; break; }
                }
            }
            if (!ok) {
                b = 1.0;
                for (int t = 0; t < P.max_ls; ++t, b *= P.beta_ls) {
                    const double dq = b * ps + 0.5 * b * b * sHs + P.lam * l1(t);
                    if (dq <= P.sigma_in * b * delta) { ok = 1; break; }
                }
            }
            cg_restart = 1;
            next_pcd = (inner_cg == 0);
            if (!ok) stop = 1;
            else beta = b;
        } else {     // R6': exact model step along s, truncated at the first kink
            sHs = sh_r[0] + P.eps_h * ss;
            bk = sh_r[3];
            if (!(slope < 0.0) || !(sHs > 0.0)) stop = 1;
            else {
                bq = -slope / sHs;
                beta = bq < bk ? bq : bk;
                ksnap = (bk <= bq);
                cg_restart = ksnap;
                next_pcd = (inner_cg == 2) && ksnap;
                rz_prev = rz;
            }
        }
        PH_MARK(4);
        if (stop) {
            if (need_hs && !resident) {   // drain the prefetched rings
                for (int stg2 = 0; stg2 < GST; ++stg2)
                    if (csG.desc[stg2].cf != 0.0) { mbar_wait(csG.bar + stg2, (g_phase >> stg2) & 1u); g_phase ^= 1u << stg2; }
                __syncwarp();
                if (lane == 0)
                    for (int k = 0; k < GST; ++k) mbar_inval(g_bar + k);
            }
            break;
        }
        acc_steps += 1;
        // R12, m side: Xd += X sigma on my rows (sigma = beta s, or beta s + (1 - beta) z on the snap path)
        if (BIG) {   // (thousands of rows per block in global memory: 8 rows in flight per thread)
            for (int k0 = threadIdx.x; k0 < r1 - r0; k0 += 8 * blockDim.x) {
                double xd[8], xs[8], xz[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int k = k0 + u * blockDim.x;
                    const bool in = k < r1 - r0;
                    xd[u] = in ? xd_r[k] : 0.0;
                    xs[u] = in ? xs_r[k] : 0.0;
                    xz[u] = (in && zs) ? xz_r[k] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int k = k0 + u * blockDim.x;
                    if (k < r1 - r0) xd_r[k] = xd[u] + (beta * xs[u] + (zs ? (1.0 - beta) * xz[u] : 0.0));
                }
            }
        } else {
            for (int k = threadIdx.x; k < r1 - r0; k += blockDim.x)
                xd_r[k] += beta * xs_r[k] + (zs ? (1.0 - beta) * xz_r[k] : 0.0);
        }
        if (BIG && need_hs) {   // G from L2: Hsigma = beta X^T (D o Xs) (+ (1 - beta) X^T (D o Xz)) + eps sigma
            __syncthreads();
            PH_MARK(5);
#ifdef IR_BLKDBG
            bd_t0 = gtimer();
#endif
            ColStream<GSCH, GST>& cs = csG;
            int stg = 0;
            double a = 0.0, az = 0.0;
            while (true) {
                const ChunkDesc dsc = cs.desc[stg];
                if (dsc.cf == 0.0) break;
                mbar_wait(cs.bar + stg, (g_phase >> stg) & 1u);
                g_phase ^= 1u << stg;
                const int* ci = S.idx ? cs.sidx + stg * GSCH - dsc.a : S.rowtab - dsc.cb;
                const float* cv = cs.sval + stg * GSCH - dsc.a;
                const int kend = min(dsc.ve, dsc.ce);
                int k = dsc.vb + lane;
                // the L2 gathers of D o X sigma are latency-bound: IR_GU gathers in flight per lane
                if (zs) {
                    double a1 = 0.0, az1 = 0.0;
                    for (; k + 32 * (IR_GUZ) - 32 < kend; k += 32 * (IR_GUZ)) {
                        int q[IR_GUZ];
                        double2 sq[IR_GUZ];   // (D o Xs, D o Xz) of a row share a sector: one gather per nonzero, not
                                                 // two (the chip serves a fixed number of random sectors per second)
#pragma unroll
                        for (int u = 0; u < IR_GUZ; ++u) q[u] = ci[k + 32 * u];
#pragma unroll
                        for (int u = 0; u < IR_GUZ; ++u) sq[u] = ld_cg(P.sv2 + q[u]);
#pragma unroll
                        for (int u = 0; u < IR_GUZ; u += 2) {
                            a = fma((double)cv[k + 32 * u], sq[u].x, a);
                            az = fma((double)cv[k + 32 * u], sq[u].y, az);
                            a1 = fma((double)cv[k + 32 * u + 32], sq[u + 1].x, a1);
                            az1 = fma((double)cv[k + 32 * u + 32], sq[u + 1].y, az1);
                        }
                    }
                    a += a1;
                    az += az1;
                    for (; k < kend; k += 32) {
                        const int r = ci[k];
                        const double xv = (double)cv[k];
                        const double2 sq = ld_cg(P.sv2 + r);
                        a = fma(xv, sq.x, a);
                        az = fma(xv, sq.y, az);
                    }
                } else {
                    double a1 = 0.0, a2 = 0.0, a3 = 0.0;
                    for (; k + 32 * IR_GU - 32 < kend; k += 32 * IR_GU) {
                        int q[IR_GU];
                        double sa[IR_GU];
#pragma unroll
                        for (int u = 0; u < IR_GU; ++u) q[u] = ci[k + 32 * u];
#pragma unroll
                        for (int u = 0; u < IR_GU; ++u) sa[u] = ld_cg(P.sv + q[u]);
#pragma unroll
                        for (int u = 0; u < IR_GU; u += 4) {
                            a = fma((double)cv[k + 32 * u], sa[u], a);
                            a1 = fma((double)cv[k + 32 * u + 32], sa[u + 1], a1);
                            a2 = fma((double)cv[k + 32 * u + 64], sa[u + 2], a2);
                            a3 = fma((double)cv[k + 32 * u + 96], sa[u + 3], a3);
                        }
                    }
                    for (; k + 96 < kend; k += 128) {
                        const int q0r = ci[k], q1r = ci[k + 32], q2r = ci[k + 64], q3r = ci[k + 96];
                        const double s0 = ld_cg(P.sv + q0r), s1 = ld_cg(P.sv + q1r), s2 = ld_cg(P.sv + q2r),
                                     s3 = ld_cg(P.sv + q3r);
                        a = fma((double)cv[k], s0, a);
                        a1 = fma((double)cv[k + 32], s1, a1);
                        a2 = fma((double)cv[k + 64], s2, a2);
                        a3 = fma((double)cv[k + 96], s3, a3);
                    }
                    a += (a1 + a2) + a3;
                    for (; k < kend; k += 32) a = fma((double)cv[k], ld_cg(P.sv + ci[k]), a);
                }
                for (; k < dsc.ve; k += 32) {
                    const int r = seg_idx(S, k, dsc.cb);
                    const double xv = (double)__ldg(S.val + k);
                    if (zs) {
                        const double2 sq = ld_cg(P.sv2 + r);
                        a = fma(xv, sq.x, a);
                        az = fma(xv, sq.y, az);
                    } else a = fma(xv, ld_cg(P.sv + r), a);
                }
                if (dsc.last) {   // unit end: its partial (combined per column after the barrier)
                    const double t = warp_sum(a), tz = zs ? warp_sum(az) : 0.0;
                    if (lane == 0) P.upart[dsc.p] = make_double2(t, tz);
                    a = 0.0;
                    az = 0.0;
                }
                __syncwarp();
                ChunkDesc nd;
                const bool ok = cs.next(nd);
                if (lane == 0) {
                    if (ok) { cs.desc[stg] = nd; cs.issue(stg, nd); }
                    else cs.desc[stg].cf = 0.0;
                }
                __syncwarp();
                stg = (stg + 1) % GST;
            }
            nhs += cs.streamed;
            __syncwarp();
            if (lane == 0)
                for (int k = 0; k < GST; ++k) mbar_inval(g_bar + k);
#ifdef IR_BLKDBG
            __syncthreads();
            bd_g += gtimer() - bd_t0;
#endif
            grid.sync();   // every unit's partial
            if (blockIdx.x == 0 && threadIdx.x == 0) c->g_ctr = 0u;
            for (int k = threadIdx.x; k < q0; k += blockDim.x) {   // my columns: partials in unit order, the step
                const int p = p0 + k;
                const int ua = ld_cg(P.ustart + p), ub = ld_cg(P.uend + p);
                double t = 0.0, tz = 0.0;
                for (int u = ua; u < ub; ++u) { const double2 q2 = ld_cg(P.upart + u); t += q2.x; tz += q2.y; }
                const double sp = X.s[k], zp = zs ? X.u[k] : 0.0;
                const double x = X.wA[k] + X.d[k];
                const bool kink = ksnap && x * sp < 0.0 && -x / sp == bk;
                X.Hd[k] += beta * t + (zs ? (1.0 - beta) * tz : 0.0) + P.eps_h * ((zp != 0.0) ? zp : beta * sp);
                X.d[k] = (zp != 0.0 || kink) ? -X.wA[k] : X.d[k] + beta * sp;
            }
            PH_MARK(6);
        } else if (need_hs && resident) {   // G from the resident chunks: each column's dot over the whole block
            double* sv_sh = xs_sh;
            for (int i0 = threadIdx.x; i0 < m; i0 += 8 * blockDim.x) {   // 8 rows in flight per thread
                double xs[8], xz[8], dd[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = i0 + u * blockDim.x;
                    xs[u] = i < m ? ld_cg(P.Xs + i) : 0.0;
                    xz[u] = (zs && i < m) ? ld_cg(P.Xz + i) : 0.0;
                    dd[u] = i < m ? P.rD[i].y : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = i0 + u * blockDim.x;
                    if (i < m) sv_sh[i] = dd[u] * (beta * xs[u] + (zs ? (1.0 - beta) * xz[u] : 0.0));
                }
            }
            __syncthreads();
            PH_MARK(5);
            constexpr int NPG = SlotPad<SST>::NP;   // (the butterfly takes a power of two of slots)
            double acc[NPG];
#pragma unroll
            for (int st = SST; st < NPG; ++st) acc[st] = 0.0;
#pragma unroll
            for (int st = 0; st < SST; ++st) {   // chunk st: my elements k = vb + t + 256 u, in order
                acc[st] = 0.0;
                const SChunk d = s_desc[st];
                if (d.ok) {
                    const int* ci = S.idx ? s_idx + st * IR_SCH - d.a : S.rowtab - d.cb;
                    const float* cv = s_val + st * IR_SCH - d.a;
                    const int kend = min(d.ve, d.ce);
                    double a = 0.0;
#pragma unroll
                    for (int u = 0; u < IR_SCH / 256; ++u) {
                        const int k = d.vb + threadIdx.x + 256 * u;
                        const bool in = k < kend;
                        const double x = in ? (double)cv[k] : 0.0;
                        const double sv = in ? sv_sh[ci[k]] : 0.0;
                        a = fma(x, sv, a);
                    }
                    const int kt = max(kend, d.vb) + (int)threadIdx.x;   // the global tail past X's last 16-byte
                    if (kt < d.ve)                                          // boundary (a chunk may start past kend)
                        a = fma((double)__ldg(S.val + kt), sv_sh[seg_idx(S, kt, d.cb)], a);
                    acc[st] = a;
                    if (threadIdx.x == 0) nhs += d.ve - d.vb;
                }
            }
            warp_reduce_slots<NPG>(acc, 0u, 0u);
            constexpr int SH = SlotPad<NPG>::SH;
            if ((lane & ((1 << SH) - 1)) == 0) sh_w[wid * NPG + (lane >> SH)] = acc[0];
            __syncthreads();
            double* ctot = sh_w + IR_W * NPG;
            if (threadIdx.x < SST) {   // chunk totals, warps in order
                double t = sh_w[threadIdx.x];
#pragma unroll
                for (int w = 1; w < IR_W; ++w) t += sh_w[w * NPG + threadIdx.x];
                ctot[threadIdx.x] = t;
            }
            __syncthreads();
            for (int k = threadIdx.x; k < q0; k += blockDim.x) {   // my positions: their chunks in order, the step
                double t = 0.0;
#pragma unroll
                for (int st = 0; st < SST; ++st)
                    if (s_desc[st].ok && s_desc[st].p == p0 + k) t += ctot[st];
                const double sp = X.s[k], zp = zs ? X.u[k] : 0.0;
                const double x = X.wA[k] + X.d[k];
                const bool kink = ksnap && x * sp < 0.0 && -x / sp == bk;
                X.Hd[k] += t + P.eps_h * ((zp != 0.0) ? zp : beta * sp);
                X.d[k] = (zp != 0.0 || kink) ? -X.wA[k] : X.d[k] + beta * sp;   // snapped coordinates become 0
            }
            PH_MARK(6);
        } else if (need_hs) {   // G: H sigma on my positions, then d += sigma, Hd += H sigma
            double* sv_sh = xs_sh;
            for (int i0 = threadIdx.x; i0 < m; i0 += 8 * blockDim.x) {   // 8 rows in flight per thread
                double xs[8], xz[8], dd[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = i0 + u * blockDim.x;
                    xs[u] = i < m ? ld_cg(P.Xs + i) : 0.0;
                    xz[u] = (zs && i < m) ? ld_cg(P.Xz + i) : 0.0;
                    dd[u] = i < m ? P.rD[i].y : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = i0 + u * blockDim.x;
                    if (i < m) sv_sh[i] = dd[u] * (beta * xs[u] + (zs ? (1.0 - beta) * xz[u] : 0.0));
                }
            }
            __syncthreads();
            PH_MARK(5);
            ColStream<GSCH, GST>& cs = csG;
            int stg = 0;
            double a = 0.0;
            while (true) {
                const ChunkDesc dsc = cs.desc[stg];
                if (dsc.cf == 0.0) break;
                mbar_wait(cs.bar + stg, (g_phase >> stg) & 1u);
                g_phase ^= 1u << stg;
                const int* ci = S.idx ? cs.sidx + stg * GSCH - dsc.a : S.rowtab - dsc.cb;
                const float* cv = cs.sval + stg * GSCH - dsc.a;
                const int kend = min(dsc.ve, dsc.ce);
                int k = dsc.vb + lane;
                double a1 = 0.0, a2 = 0.0, a3 = 0.0;
                for (; k + 96 < kend; k += 128) {
                    a = fma((double)cv[k], sv_sh[ci[k]], a);
                    a1 = fma((double)cv[k + 32], sv_sh[ci[k + 32]], a1);
                    a2 = fma((double)cv[k + 64], sv_sh[ci[k + 64]], a2);
                    a3 = fma((double)cv[k + 96], sv_sh[ci[k + 96]], a3);
                }
                a += (a1 + a2) + a3;
                for (; k < kend; k += 32) a = fma((double)cv[k], sv_sh[ci[k]], a);
                for (; k < dsc.ve; k += 32) a = fma((double)__ldg(S.val + k), sv_sh[seg_idx(S, k, dsc.cb)], a);
                if (dsc.last) {
                    const double t = warp_sum(a);
                    if (lane == 0) {
                        const int k = dsc.p - p0;
                        const double sp = X.s[k], zp = zs ? X.u[k] : 0.0;
                        const double x = X.wA[k] + X.d[k];
                        const bool kink = ksnap && x * sp < 0.0 && -x / sp == bk;
                        X.Hd[k] += t + P.eps_h * ((zp != 0.0) ? zp : beta * sp);
                        X.d[k] = (zp != 0.0 || kink) ? -X.wA[k] : X.d[k] + beta * sp;   // snapped coordinates become 0
                    }
                    a = 0.0;
                }
                __syncwarp();
                ChunkDesc nd;
                const bool ok = cs.next(nd);
                if (lane == 0) {
                    if (ok) { cs.desc[stg] = nd; cs.issue(stg, nd); }
                    else cs.desc[stg].cf = 0.0;
                }
                __syncwarp();
                stg = (stg + 1) % GST;
            }
            nhs += cs.streamed;
            __syncwarp();
            if (lane == 0)
                for (int k = 0; k < GST; ++k) mbar_inval(g_bar + k);
            PH_MARK(6);
        } else {   // last iteration: d only
            for (int k = threadIdx.x; k < q0; k += blockDim.x) {
                const double sp = X.s[k], zp = zs ? X.u[k] : 0.0;
                const double x = X.wA[k] + X.d[k];
                const bool kink = ksnap && x * sp < 0.0 && -x / sp == bk;
                X.d[k] = (zp != 0.0 || kink) ? -X.wA[k] : X.d[k] + beta * sp;
            }
        }
        __syncthreads();   // my positions' d, Hd and the shared rings before the next direction
    }
#ifdef IR_BLKDBG
    if (BIG && threadIdx.x == 0) {   // tph[0..2]: sum / max / (2^62 - min) of S work over blocks; [3..5] the same for G
        atomicAdd(&c->tph[0], bd_s); atomicMax(&c->tph[1], bd_s); atomicMax(&c->tph[2], (1ull << 62) - bd_s);
        atomicAdd(&c->tph[3], bd_g); atomicMax(&c->tph[4], bd_g); atomicMax(&c->tph[5], (1ull << 62) - bd_g);
    }
#endif
    if (!BIG && s_res && threadIdx.x == blockDim.x - 32)   // the resident ring's barriers
        for (int k = 0; k < SST; ++k) mbar_inval(s_bar + k);
    // accounting: X_A s scatters, Hs gathers
    {
        const long long s1 = warp_sum_ll(lane == 0 ? nsc : 0), s2 = warp_sum_ll(lane == 0 ? nhs : 0);
        if (lane == 0) {
            if (s1) atomicAdd((unsigned long long*)acc_sc, (unsigned long long)s1);
            if (s2) atomicAdd((unsigned long long*)acc_hs, (unsigned long long)s2);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) c->acc_steps = acc_steps;
    (void)bq; (void)vq; (void)sHs;
    // ------------------------------------------------ R14-R18: outer line search on F and the update
    PH_MARK(7);
    const double F0 = c->F;
    if (acc_steps == 0) {   // R14: d = 0
        if (blockIdx.x == 0 && threadIdx.x == 0) { c->skip = 1; c->outcome = OUT_NOSTEP; ir_trace(P, c, OUT_NOSTEP, 0, IR_FB(F0), F0, IR_AL(0.0)); }
        return;
    }
    double at[4];
    at[0] = 1.0;
#pragma unroll
    for (int k = 1; k < 4; ++k) at[k] = at[k - 1] * P.beta_ls;
    // first batch {1, 1/2, 1/4, 1/8} (Eq. 4; Armijo Q7; term-by-term differences Q26).  Large m: alpha = 1
    // alone first -- it is the common outcome, and each trial costs an exp / expm1 / log1p per row (thousands of rows
    // per block) -- then {1/2, 1/4, 1/8} only if it fails
    constexpr int NT1 = BIG ? 1 : 4;
    {
        double v[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) v[k] = 0.0;
        for (int k0 = threadIdx.x; k0 < q0; k0 += blockDim.x) {
            const double d = X.d[k0], w = X.wA[k0], aw = fabs(w);
            v[0] += X.gA[k0] * d;
            v[1] = fmax(v[1], fabs(d));
#pragma unroll
            for (int k = 0; k < NT1; ++k) v[2 + k] += fabs(w + at[k] * d) - aw;
        }
        if (BIG) {   // (four rows' loads in flight per thread; the sums in the same order)
            for (int i0 = r0 + threadIdx.x; i0 < r1; i0 += 4 * blockDim.x) {
                double zz[4], xd[4], yb[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = i0 + u * blockDim.x;
                    const bool in = i < r1;
                    zz[u] = in ? P.z[i] : 0.0;
                    xd[u] = in ? xd_r[i - r0] : 0.0;
                    yb[u] = in ? (P.b ? P.b[i] : (double)P.y[i]) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (i0 + u * (int)blockDim.x < r1) {
#pragma unroll
                        for (int k = 0; k < NT1; ++k) {
                            const double dz = at[k] * xd[u];
                            if (P.b) { const double r = zz[u] - yb[u]; v[6 + k] += dz * (r + 0.5 * dz); }
                            else v[6 + k] += dloss(yb[u] * zz[u], yb[u] * dz);
                        }
                    }
                }
            }
        } else {
            for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
                const double zi = P.z[i], xd = xd_r[i - r0];
#pragma unroll
                for (int k = 0; k < NT1; ++k) v[6 + k] += dloss_i(P.y, P.b, i, zi, at[k] * xd);
            }
        }
        ir_block_partials<10>(v, 1u << 1, 0u, sh_w, part, IR_SO);
    }
    grid.sync();
    ir_totals(part, IR_SO, 10, 1u << 1, 0u, sh_t);
    if (BIG && sh_t[1] != 0.0 && P.max_ls > 1 &&
        !(sh_t[6] + P.lam * sh_t[2] <= P.sigma_out * (sh_t[0] + P.lam * sh_t[2]))) {   // alpha = 1 failed
        double v[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) v[k] = 0.0;
        for (int k0 = threadIdx.x; k0 < q0; k0 += blockDim.x) {
            const double d = X.d[k0], w = X.wA[k0], aw = fabs(w);
#pragma unroll
            for (int k = 1; k < 4; ++k) v[k - 1] += fabs(w + at[k] * d) - aw;
        }
        for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
            const double zi = P.z[i], xd = xd_r[i - r0];
#pragma unroll
            for (int k = 1; k < 4; ++k) v[2 + k] += dloss_i(P.y, P.b, i, zi, at[k] * xd);
        }
        ir_block_partials<6>(v, 0u, 0u, sh_w, part, IR_SO3);
        grid.sync();
        __shared__ double sh_t3[6];
        ir_totals(part, IR_SO3, 6, 0u, 0u, sh_t3);
        if (threadIdx.x < 3) { sh_t[3 + threadIdx.x] = sh_t3[threadIdx.x]; sh_t[7 + threadIdx.x] = sh_t3[3 + threadIdx.x]; }
        __syncthreads();
    }
    const double Delta = sh_t[0] + P.lam * sh_t[2];
    if (sh_t[1] == 0.0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) { c->skip = 1; c->outcome = OUT_NOSTEP; ir_trace(P, c, OUT_NOSTEP, acc_steps, IR_FB(F0), F0, IR_AL(0.0)); }
        return;
    }
    int t_acc = -1;
    double alpha = 0.0, l1d = 0.0;
    for (int k = 0; k < 4 && k < P.max_ls; ++k)
        if (sh_t[6 + k] + P.lam * sh_t[2 + k] <= P.sigma_out * at[k] * Delta) { t_acc = k; alpha = at[k]; l1d = sh_t[2 + k]; break; }
    if (t_acc < 0 && P.max_ls > 4) {   // rare: the remaining trials
        ir_outer_batch2(P, X, q0, r0, r1, xd_r, sh_w, part);
        grid.sync();
        ir_totals(part, IR_SO2, 2 * IR_NLS, 0u, 0u, sh_l1);
        double a = at[3];
        for (int k = 0; k + 4 < P.max_ls; ++k) {
            a *= P.beta_ls;
            if (sh_l1[IR_NLS + k] + P.lam * sh_l1[k] <= P.sigma_out * a * Delta) { t_acc = 4 + k; alpha = a; l1d = sh_l1[k]; break; }
        }
    }
    if (t_acc < 0) {   // R17
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            c->skip = 1; c->outcome = OUT_STAGNATION; c->alpha = 0.0;
            ir_trace(P, c, OUT_STAGNATION, acc_steps, IR_FB(F0), F0, IR_AL(0.0));
        }
        return;
    }
    {   // R18: w_A += a d (bitmap, support count), z += a Xd with the per-sample refresh, L, F
        double v[2] = {0.0, 0.0};
        for (int k0 = threadIdx.x; k0 < q0; k0 += blockDim.x) {
            const double w0 = X.wA[k0], w1 = w0 + alpha * X.d[k0];
            const int j = AS.A[p0 + k0];
            P.w[j] = w1;
            const int nz0 = (w0 != 0.0), nz1 = (w1 != 0.0);
            if (nz0 != nz1) { atomicXor(P.wbits + (j >> 5), 1u << (j & 31)); v[1] += nz1 - nz0; }
        }
        if (BIG) {   // (thousands of rows per block: four rows' loads in flight per thread; same order of the sums)
            for (int i0 = r0 + threadIdx.x; i0 < r1; i0 += 4 * blockDim.x) {
                double zz[4], xd[4], yb[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = i0 + u * blockDim.x;
                    const bool in = i < r1;
                    zz[u] = in ? P.z[i] : 0.0;
                    xd[u] = in ? xd_r[i - r0] : 0.0;
                    yb[u] = in ? (P.b ? P.b[i] : (double)P.y[i]) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = i0 + u * blockDim.x;
                    if (i < r1) {
                        const double z = zz[u] + alpha * xd[u];
                        P.z[i] = z;
                        RowState st;
                        if (P.b) { const double r = z - yb[u]; st = RowState{r, 1.0, 0.5 * r * r}; }
                        else st = row_state(z, yb[u]);
                        P.rD[i] = make_double2(st.r, st.D);
                        v[0] += st.ell;
                    }
                }
            }
        } else {
            for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
                const double z = P.z[i] + alpha * xd_r[i - r0];
                P.z[i] = z;
                const RowState st = row_state_i(P.y, P.b, i, z);
                P.rD[i] = make_double2(st.r, st.D);
                v[0] += st.ell;
            }
        }
        ir_block_partials<2>(v, 0u, 0u, sh_w, part, IR_SO);
    }
    grid.sync();
    PH_MARK(7);
    if (blockIdx.x == 0) {
        if (threadIdx.x == 0)
            for (int q2 = 0; q2 < 16; ++q2) atomicAdd(&c->tph[q2], ph_acc[q2]);
        ir_totals(part, IR_SO, 2, 0u, 0u, sh_t);
        if (threadIdx.x == 0) {
            c->nS += (int)sh_t[1];
            c->L = sh_t[0];
            c->l1 += l1d;
            c->alpha = alpha;
            c->t_acc = t_acc;
            c->ls_ok = 1;
            c->F = c->L + P.lam * c->l1;
            c->outcome = OUT_UPDATED;
            ir_trace(P, c, OUT_UPDATED, acc_steps, IR_FB(F0), c->F, IR_AL(alpha));
        }
    }
}

// ------------------------------------------------------------------ A2 + A3 for small m: cooperative free-set gather
// Block b owns the contiguous positions [b q, (b+1) q) of C (or of all columns at the finest level).  (r, D) of all rows
// is staged in shared memory; each warp streams its columns through a TMA ring (as in k_inner's Hs phase):
// g_j = sum_i X_ij r_i, h_j = sum_i X_ij^2 D_i into AS.s / AS.Hs (scratch, by position).  Then my
// positions in order: v_j, free flag w_j != 0 or |g_j| > lam; block counts and partial sums -> one grid
// barrier -> every block: its offset (counts of the blocks before it, in order), the totals; my free columns are
// written IN ORDER into the ASet.  Block 0 takes the last-block decisions of k_gather_free (nA, vmax, F, R2).
template <int GSCH>
__host__ __device__ inline size_t gather_small_smem_bytes(int m) {
    return (size_t)IR_W * stream_warp_bytes<GSCH, IN_GST>(0) + (size_t)16 * m;
}
template <int GSCH, bool FINEST>
// It also starts the relaxation (what k_relax_begin does on the large-m path): a relaxation of a level that already
// converged is skipped; block 0 resets the per-relaxation flags.
__global__ void __launch_bounds__(256, 1) k_gather_small(Prm P, Seg S, ASet AS, long long* acc, int first_of_level,
                                                         int level, int nC_list) {
    extern __shared__ __align__(16) unsigned char smraw[];
    __shared__ double sh_w[2 * 256 + 8];
    __shared__ double sh_t[4];
    __shared__ int sh_cnt[IR_W + 1];
    cg::grid_group grid = cg::this_grid();
    Ctl* ctl = P.ctl;
    const int conv = first_of_level ? 0 : ctl->level_conv;   // (only written at the end of this kernel, by block 0)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (first_of_level) ctl->level_conv = 0;
        ctl->skip = conv;
        ctl->skipped = conv;
        ctl->outcome = conv ? OUT_CONVERGED : OUT_NOSTEP;
        ctl->ls_ok = 0;
        ctl->level = level;
        ctl->acc_steps = 0;
        if (S.list) { ctl->Cptr = S.list; ctl->nC = nC_list; }
    }
    if (conv) return;   // grid-uniform (coarse relaxations of a converged level)
#ifdef GS_PHDBG
    unsigned long long ph_t = gtimer(), ph_acc[IR_PHN] = {};
    const int ph_off = FINEST ? 16 : 0;   // coarse-level launches only
#endif
    const int m = P.m, G = gridDim.x;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nC = S.list ? nC_list : P.n;
    const int q = (nC + G - 1) / G;
    const int p0 = min(nC, (int)blockIdx.x * q), p1 = min(nC, p0 + q);
    double2* rd_sh = reinterpret_cast<double2*>(smraw + (size_t)IR_W * stream_warp_bytes<GSCH, IN_GST>(0));
    unsigned char* gbase = smraw + (size_t)wid * stream_warp_bytes<GSCH, IN_GST>(0);
    uint64_t* g_bar = reinterpret_cast<uint64_t*>(gbase + 8 * IN_GST * GSCH);
    if (lane == 0) {
        for (int k = 0; k < IN_GST; ++k) mbar_init(g_bar + k, 1);
        fence_mbar_init();
    }
    __syncwarp();
    ColStream<GSCH, IN_GST> cs;
    cs.streamed = 0;
    cs.segs = 0;
    stream_begin(cs, S, nullptr, p0, p1, gbase);   // X first: its latency overlaps the (r, D) staging
    for (int i0 = threadIdx.x; i0 < m; i0 += 8 * blockDim.x) {   // 8 loads in flight per thread
        double2 t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * blockDim.x;
            t[u] = i < m ? P.rD[i] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * blockDim.x;
            if (i < m) rd_sh[i] = t[u];
        }
    }
    __syncthreads();
    GS_MARK(0);
    {
        uint32_t phase = 0u;
        int stg = 0;
        double a = 0.0, b = 0.0;
        while (true) {
            const ChunkDesc dsc = cs.desc[stg];
            if (dsc.cf == 0.0) break;
            GS_MARK(1);
            mbar_wait(cs.bar + stg, (phase >> stg) & 1u);
            GS_MARK(6);
            phase ^= 1u << stg;
            const int* ci = S.idx ? cs.sidx + stg * GSCH - dsc.a : S.rowtab - dsc.cb;
            const float* cv = cs.sval + stg * GSCH - dsc.a;
            const int kend = min(dsc.ve, dsc.ce);
            int k = dsc.vb + lane;
            double a1 = 0.0, b1 = 0.0;
            for (; k + 32 < kend; k += 64) {
                const double2 q0 = rd_sh[ci[k]], q1 = rd_sh[ci[k + 32]];
                const double x0 = (double)cv[k], x1 = (double)cv[k + 32];
                a = fma(x0, q0.x, a);
                b = fma(x0 * x0, q0.y, b);
                a1 = fma(x1, q1.x, a1);
                b1 = fma(x1 * x1, q1.y, b1);
            }
            a += a1;
            b += b1;
            for (; k < kend; k += 32) {
                const double2 q0 = rd_sh[ci[k]];
                const double x0 = (double)cv[k];
                a = fma(x0, q0.x, a);
                b = fma(x0 * x0, q0.y, b);
            }
            for (; k < dsc.ve; k += 32) {
                const double2 q0 = rd_sh[seg_idx(S, k, dsc.cb)];
                const double x0 = (double)__ldg(S.val + k);
                a = fma(x0, q0.x, a);
                b = fma(x0 * x0, q0.y, b);
            }
            if (dsc.last) {
                const double g = warp_sum(a), h = warp_sum(b);
                if (lane == 0) { AS.s[dsc.p] = g; AS.Hs[dsc.p] = h; }
                a = 0.0;
                b = 0.0;
            }
            __syncwarp();
            ChunkDesc nd;
            const bool ok = cs.next(nd);
            if (lane == 0) {
                if (ok) { cs.desc[stg] = nd; cs.issue(stg, nd); }
                else cs.desc[stg].cf = 0.0;
            }
            __syncwarp();
            stg = (stg + 1) % IN_GST;
        }
        __syncwarp();
        if (lane == 0)
            for (int k = 0; k < IN_GST; ++k) mbar_inval(g_bar + k);
    }
    GS_MARK(1);
    acc_add(acc, cs.streamed, cs.segs);   // (synchronises the block: g, h of my positions are visible)
    // my positions in order: flags, block count, partial sums
    double v1p = 0.0, l1p = 0.0, vmx = 0.0;
    int cnt = 0;
    const bool one_pass = p1 - p0 <= (int)blockDim.x;   // then my position's (j, g, w_j) stay in registers
    int j1 = 0;
    double g1 = 0.0, w1 = 0.0, h1 = 0.0;
    for (int p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
        const int j = S.list ? __ldg(S.list + p) : p;
        const double g = AS.s[p];
        h1 = AS.Hs[p];
        double wj = 0.0;
        if ((P.wbits[j >> 5] >> (j & 31)) & 1u) wj = P.w[j];
        const double v = (wj != 0.0) ? g + P.lam * sgn(wj) : soft(g, P.lam);
        vmx = fmax(vmx, fabs(v));
        v1p += fabs(v);
        l1p += fabs(wj);
        cnt += (wj != 0.0) || (fabs(g) > P.lam);
        j1 = j; g1 = g; w1 = wj;
    }
    {
        const double v[4] = {v1p, l1p, vmx, (double)cnt};
        ir_block_partials<4>(v, 1u << 2, 0u, sh_w, P.irpart, 0);
    }
    GS_MARK(2);
    grid.sync();
    GS_MARK(3);
    // totals (identical in every block) and my offset: the counts of the blocks before me, in order
    ir_totals(P.irpart, 0, 3, 1u << 2, 0u, sh_t);
    if (wid == 0) {
        int off = 0, tot = 0;
        for (int b0 = 0; b0 < G; b0 += 32) {
            const int b = b0 + lane;
            const int c = b < G ? (int)ld_cg(P.irpart + (size_t)3 * G + b) : 0;
            const int before = (b < (int)blockIdx.x) ? c : 0;
            off += __reduce_add_sync(0xffffffffu, before);
            tot += __reduce_add_sync(0xffffffffu, c);
        }
        if (lane == 0) { sh_cnt[IR_W] = off; sh_cnt[0] = tot; }
    }
    __syncthreads();
    const int my_off = sh_cnt[IR_W], nA = sh_cnt[0];
    __syncthreads();
    GS_MARK(4);
    // my free columns, in position order
    int base = my_off;
    for (int p00 = p0; p00 < p1; p00 += blockDim.x) {
        const int p = p00 + threadIdx.x;
        int j = 0, flag = 0;
        double g = 0.0, wj = 0.0;
        if (p < p1) {
            if (one_pass) { j = j1; g = g1; wj = w1; }
            else {
                j = S.list ? __ldg(S.list + p) : p;
                g = AS.s[p];
                if ((P.wbits[j >> 5] >> (j & 31)) & 1u) wj = P.w[j];
            }
            flag = (wj != 0.0) || (fabs(g) > P.lam);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, flag);
        if (lane == 0) sh_cnt[wid] = __popc(bal);
        __syncthreads();
        int woff = 0, tot = 0;
        for (int w = 0; w < IR_W; ++w) { if (w < wid) woff += sh_cnt[w]; tot += sh_cnt[w]; }
        if (flag) {
            int o = base + woff + __popc(bal & ((1u << lane) - 1u));
            if (!FINEST) {   // coarse: interleave, column o goes to k_inner's block o mod G (balanced ranges, see
                             // k_inner): a PCD-CG step's active columns spread evenly over the blocks
                const int qb = nA / G, rb = nA % G, bb = o % G;
                o = bb * qb + min(bb, rb) + o / G;
            }
            AS.A[o] = j;
            AS.gA[o] = g;
            AS.hA[o] = (one_pass ? h1 : AS.Hs[p]) + P.eps_h;
            AS.wA[o] = wj;
        }
        base += tot;
        __syncthreads();
    }
    GS_MARK(5);
#ifdef GS_PHDBG
    if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int q2 = 0; q2 < 16; ++q2) atomicAdd(&ctl->tph[q2], ph_acc[q2]);
#endif
    if (blockIdx.x == 0 && threadIdx.x == 0) {   // the last-block decisions of k_gather_free
        ctl->nA = nA;
        const double vmax = sh_t[2];
        ctl->vmax = vmax;
        ctl->vmax_bits = 0ull;
        if (FINEST) {
            ctl->v1 = sh_t[0];
            ctl->l1 = sh_t[1];
            ctl->nAf = nA;
            ctl->F = ctl->L + P.lam * ctl->l1;
        }
        ctl->F_before = ctl->F;
        if (vmax / P.lam <= P.tol) { ctl->skip = 1; ctl->outcome = OUT_CONVERGED; ctl->level_conv = 1; }
    }
}

// ------------------------------------------------------------------ A1 for small m: margins from the support's columns
// z = X_S w_S (S = supp(w)) by the same block-cooperative column scatter as k_inner's S phase, instead of streaming all
// of X by rows: (1) the support list in column order from the support bitmap (block counts -> barrier -> in-order
// write), barrier; (2) my support columns (TMA ring, one shared m-vector) -> block partial, barrier; (3) my rows:
// z_i = sum of the block partials in block order, t, ell, r, D; L = sum ell, F = L + lam ||w||_1.
template <int GSCH>
__global__ void __launch_bounds__(256, 1) k_margins_small(Prm P, Seg S, int* slist, long long* acc) {
    extern __shared__ __align__(16) unsigned char smraw[];
    __shared__ double sh_w[IR_W * 4 + 8];
    __shared__ double sh_t[2];
    __shared__ double gsum[256];
    __shared__ int sh_cnt[IR_W + 2];
    constexpr int SST = ir_sst(GSCH);
    cg::grid_group grid = cg::this_grid();
    Ctl* c = P.ctl;
    const int m = P.m, G = gridDim.x;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* part = P.irpart;
    double* xs_sh = reinterpret_cast<double*>(smraw + ir_ring_bytes<GSCH>());
    int* s_idx = reinterpret_cast<int*>(smraw);
    float* s_val = reinterpret_cast<float*>(smraw + (size_t)4 * SST * IR_SCH);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smraw + (size_t)8 * SST * IR_SCH);
    SChunk* s_desc = reinterpret_cast<SChunk*>(s_bar + SST);
    // (1) support list, in column order
    const int nw = (P.n >> 5) + 1;
    const int wq = (nw + G - 1) / G;
    const int w0 = min(nw, (int)blockIdx.x * wq), w1 = min(nw, w0 + wq);
    int cnt = 0;
    for (int k = w0 + threadIdx.x; k < w1; k += blockDim.x) cnt += __popc(P.wbits[k]);
    {
        const double v[1] = {(double)cnt};
        ir_block_partials<1>(v, 0u, 0u, sh_w, part, 0);
    }
    grid.sync();
    if (wid == 0) {
        int off = 0, tot = 0;
        for (int b0 = 0; b0 < G; b0 += 32) {
            const int b = b0 + lane;
            const int x = b < G ? (int)ld_cg(part + b) : 0;
            off += __reduce_add_sync(0xffffffffu, b < (int)blockIdx.x ? x : 0);
            tot += __reduce_add_sync(0xffffffffu, x);
        }
        if (lane == 0) { sh_cnt[IR_W] = off; sh_cnt[IR_W + 1] = tot; }
    }
    __syncthreads();
    const int nS = sh_cnt[IR_W + 1];
    {
        int base = sh_cnt[IR_W];
        for (int k00 = w0; k00 < w1; k00 += blockDim.x) {
            const int k = k00 + threadIdx.x;
            const unsigned bits = k < w1 ? P.wbits[k] : 0u;
            const int pc = __popc(bits);
            int incl = pc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            if (lane == 31) sh_cnt[wid] = incl;
            __syncthreads();
            int woff = 0, tot = 0;
            for (int w = 0; w < IR_W; ++w) { if (w < wid) woff += sh_cnt[w]; tot += sh_cnt[w]; }
            int o = base + woff + incl - pc;
            for (unsigned b = bits; b; b &= b - 1) slist[o++] = (k << 5) + __ffs(b) - 1;
            base += tot;
            __syncthreads();
        }
    }
    fence_proxy_async_global();
    grid.sync();
    // (2) my support columns -> one shared m-vector -> my block partial
    const int q = (nS + G - 1) / G;
    const int p0 = min(nS, (int)blockIdx.x * q), p1 = min(nS, p0 + q);
    Seg SS = S;
    SS.list = slist;
    for (int i = threadIdx.x; i < m; i += blockDim.x) xs_sh[i] = 0.0;
    const bool producer = threadIdx.x == blockDim.x - 32;
    SProducer pr{p0, p0, p1, 0, (int)(S.nnz & ~3LL), nullptr};
    if (producer) pr.prefetch(SS, SST, s_desc, s_idx, s_val, s_bar);
    __syncthreads();
    long long nsc = 0;
    uint32_t s_phase = 0u;
    for (int st = 0;; st = (st + 1) % SST) {
        const SChunk d = s_desc[st];
        if (!d.ok) break;
        mbar_wait(s_bar + st, (s_phase >> st) & 1u);
        s_phase ^= 1u << st;
        const double cf = P.w[__ldg(slist + d.p)];
        const int* ci = S.idx ? s_idx + st * IR_SCH - d.a : S.rowtab - d.cb;
        const float* cv = s_val + st * IR_SCH - d.a;
        const int kend = min(d.ve, d.ce);
        constexpr int UB = IR_SCH / 256;
        // rows distinct within a column; the staged part has branch-free (predicated) loads, the global tail past
        // X's last 16-byte boundary (at most 3 nonzeros) its own loop (as in k_inner's S phase)
        for (int k0 = d.vb + threadIdx.x; k0 < kend; k0 += UB * (int)blockDim.x) {
            int r[UB];
            double xv[UB], a[UB];
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const int k = k0 + u * blockDim.x;
                r[u] = -1;
                xv[u] = 0.0;
                if (k < kend) { r[u] = ci[k]; xv[u] = (double)cv[k]; }
            }
#pragma unroll
            for (int u = 0; u < UB; ++u) a[u] = r[u] >= 0 ? xs_sh[r[u]] : 0.0;
#pragma unroll
            for (int u = 0; u < UB; ++u)
                if (r[u] >= 0) xs_sh[r[u]] = fma(xv[u], cf, a[u]);
        }
        for (int k = max(kend, d.vb) + threadIdx.x; k < d.ve; k += blockDim.x) {   // (a chunk may start past kend)
            const int r = seg_idx(S, k, d.cb);
            xs_sh[r] = fma((double)__ldg(S.val + k), cf, xs_sh[r]);
        }
        if (threadIdx.x == 0) nsc += d.ve - d.vb;
        __syncthreads();
        if (producer) {
            SChunk nd;
            if (pr.next(SS, nullptr, nd)) { s_desc[st] = nd; pr.issue(SS, nd, st, s_idx, s_val, s_bar); }
            else s_desc[st].ok = 0;
        }
    }
    __syncthreads();
    if (producer)
        for (int k = 0; k < SST; ++k) mbar_inval(s_bar + k);
    for (int i = threadIdx.x; i < m; i += blockDim.x) P.parts[(size_t)blockIdx.x * m + i] = xs_sh[i];
    acc_add(acc, nsc, threadIdx.x == 0 ? (long long)(p1 - p0) : 0);
    grid.sync();
    // (3) my rows
    const int R = (m + G - 1) / G;
    const int r0 = min(m, (int)blockIdx.x * R), r1 = min(m, r0 + R);
    const int nr = r1 - r0;
    double lsum = 0.0;
    if (nr > 0) {
        const int ng = max(1, (int)blockDim.x / nr);
        const int g = threadIdx.x / nr, rr = threadIdx.x % nr;
        double t = 0.0;
        if (g < ng) {
            const double* src = P.parts + r0 + rr;
            for (int b0 = g; b0 < G; b0 += 8 * ng) {
                double x[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int b = b0 + u * ng;
                    x[u] = b < G ? ld_cg(src + (size_t)b * m) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) t += x[u];
            }
            gsum[threadIdx.x] = t;
        }
        __syncthreads();
        for (int rr2 = threadIdx.x; rr2 < nr; rr2 += blockDim.x) {
            double z = 0.0;
            for (int g2 = 0; g2 < ng; ++g2) z += gsum[g2 * nr + rr2];
            const int i = r0 + rr2;
            const RowState st = row_state_i(P.y, P.b, i, z);
            P.z[i] = z;
            P.rD[i] = make_double2(st.r, st.D);
            lsum += st.ell;
        }
    }
    {
        const double v[1] = {lsum};
        ir_block_partials<1>(v, 0u, 0u, sh_w, part, 1);
    }
    grid.sync();
    if (blockIdx.x == 0) {
        ir_totals(part, 1, 1, 0u, 0u, sh_t);
        if (threadIdx.x == 0) { c->L = sh_t[0]; c->F = sh_t[0] + P.lam * c->l1; }
    }
}
