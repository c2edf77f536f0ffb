// ml.cu — libml: C ABI (include/ml.h) + host driver of the multilevel cycle (Algorithm 1).
//
// The host decides only what the paper's cycle needs at cycle granularity (level sizes); every
// data-dependent decision inside a relaxation (free set, step lengths, early stops) stays on the device in the
// control block `ml::Ctl`, so one relaxation is a fixed sequence of launches with no host synchronisation, and one
// ML-cycle costs one stream synchronisation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ml.h"
#include "ml_kernels.cuh"
#include "ml_merge.cuh"
#include "ml_select.cuh"

using namespace ml;

namespace {

constexpr int SM_MAX = IR_GMAX;   // partial buffers are sized for this many SMs; grids use the device's own count
constexpr int GRID_CAP = 148 * 4;   // grid-stride passes: 4 blocks per B200 SM (any count works, this sizes partials)
constexpr int TRACE_CAP = 1 << 16;
constexpr int NV_MAX = 96;   // widest reduction payload (doubles per block)
constexpr int SMALL_M = 8192;
constexpr int64_t CLAIM_NNZ = 16 << 20;   // k_heavy claims its units dynamically from this many nonzeros of X   // m-vectors up to this size are accumulated in shared memory (k_scatter_smem)


inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct Carve {                 // workspace layout; base == nullptr -> sizing only
    char* base;
    size_t off = 0;
    template <class T> T* take(size_t count) {
        size_t o = off;
        off = align_up(off + std::max<size_t>(count, 1) * sizeof(T));
        return base ? reinterpret_cast<T*>(base + o) : nullptr;
    }
};

struct UnitsMem { int4* u; double2* part; int* hcnt; int cap, hcap; };

// pass classes for accounting (device nonzero/segment counters) and optional CUDA-event timing
enum { CLS_MARGINS = 0, CLS_GATHER_FINE, CLS_GATHER_COARSE, CLS_SCATTER, CLS_HS, CLS_DIR, CLS_MPASS, CLS_APPLY,
       CLS_OUTER, CLS_UPDATE, CLS_SELECT, CLS_BOOK, CLS_API, CLS_INNER, CLS_N };

}  // namespace

struct ml_ctx {
    ml_data X;
    double lam;
    cudaStream_t st;
    char* ws;
    size_t ws_bytes;
    Prm P;
    ASet fine, coarse;
    Ctl* ctl;
    SelState* sel;
    TraceRow* trace;
    double2* hres;
    int* lvl;          // level lists
    size_t lvl_cap;
    unsigned char* lev;
    UnitsMem um[4];    // 0: all columns, 1: C list, 2: free set A, 3: rows
    int Gr, Gc;
    int gA, gM, gSeg, gHeavy;
    // small-m shared-memory scatter
    bool sm_scatter = false;
    int scat_W = 0, scat_P = 0, gMP = 1;
    int gFine2 = 0;          // grid of the two-pass finest gather's column-sum pass (occupancy x SMs)
    size_t scat_bytes = 0;
    bool sm_gather = false;
    bool sm_inner = false;   // persistent cooperative inner solver (k_inner), m-vectors in shared memory
    bool big_inner = false;  // k_inner<., true>: the same with the m-vectors in global memory (m > SMALL_M)
    int inner_W = 0, inner_P = 0;
    const void* inner_fn = nullptr;   // the k_inner instantiation in use
    const void* inner_fn_hv = nullptr;   // large m: the instantiation with the heavy-column path
    size_t inner_bytes_hv = 0;
    int sms = 148;                    // the device's SM count, capped at SM_MAX (cooperative grids: one CTA per SM)
    int coop_cap = 148;               // cooperative grids use at most this many CTAs (ml_set_sm_share)
    int scat_bps = 0, gath_bps = 0;   // blocks per SM of the cooperative API scatter / gather
    const void* gsmall_fn[2] = {nullptr, nullptr};   // k_gather_small<GSCH, false / true>
    size_t gsmall_bytes = 0;
    const void* msmall_fn = nullptr;   // k_margins_small<GSCH>
    int* slist = nullptr;
    size_t inner_bytes = 0;
    int gath_W = 0, gath_P = 0;
    size_t gath_bytes = 0;
    double* parts = nullptr;
    long long npos;
    long long launches = 0;
    // profiling: event pairs per pass class (enabled classes only)
    uint32_t prof_mask = 0;   // bit k: time pass class k (CLS_*)
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<int> ev_cls;      // class of each recorded pair (pair k = events 2k, 2k+1)
    long long prof_passes[16] = {0};
    std::string err;
    Ctl h;             // host mirror of the control block
    // merge-path column passes (ml_merge.cuh), large m: the static plan over all columns and one for lists
    bool mp = false;
    MPList mp_all, mp_l;
    int mp_tiles_cap = 0, mp_grid_all = 0, mp_grid_l = 0;
    int* mp_vptr = nullptr;
    int* mp_bsum = nullptr;
    double2* mp_out = nullptr;
    // index-free dense X (m <= SMALL_M, csc_row == csc_colptr == NULL, nnz == m n): the library's own column pointers
    // (j m) and the row table rowtab[t] = t that stands in for the staged row indices (Seg::rowtab)
    bool dense = false;
    int* dense_colptr = nullptr;
    int* rowtab = nullptr;
    // heavy-column path (large m): build scratch
    int* hv_hcols = nullptr;
    int* hv_lens = nullptr;
    int* hv_bsum = nullptr;
    int* hv_misc = nullptr;
    unsigned* hv_hist = nullptr;
    bool hv_built = false;   // hv_build ran (at ml_create for large X, else on the first ml_set_engine request)
    int hv_mode0 = 2;        // the heavy path's default mode (0 when built at ml_create for large X, else 2)
};

namespace {

// look-back status words of the compaction tiles: 64-column coarse tiles and 256-row / -column tiles (all zeroed at
// create: the words are epoch-tagged, and a stale word from another use of the memory must not match epoch 0)
inline size_t status_words(int64_t n, int64_t m) {
    return std::max<size_t>(((size_t)n + 63) / 64, ((size_t)m + TILE - 1) / TILE) + 2;
}
void carve_all(Carve& cv, ml_ctx* c, int64_t m, int64_t n, int64_t nnz) {
    const size_t nn = (size_t)n, mm = (size_t)m;
    const size_t ntile_n = (nn + TILE - 1) / TILE, ntile_m = (mm + TILE - 1) / TILE;
    const size_t hcap = (size_t)std::min<int64_t>(std::max(m, n), nnz / SPLIT_MIN) + 64;
    const size_t ucap = (size_t)(nnz / CHUNK) + hcap;
    Ctl* ctl = cv.take<Ctl>(1);
    SelState* sel = cv.take<SelState>(1);
    TraceRow* trace = cv.take<TraceRow>(TRACE_CAP);
    double* w = cv.take<double>(nn);
    uint32_t* wbits = cv.take<uint32_t>((nn + 31) / 32 + 1);
    double* z = cv.take<double>(mm);
    double2* rD = cv.take<double2>(mm);
    double* Xd = cv.take<double>(mm);
    double* Xs = cv.take<double>(mm);
    double* sv = cv.take<double>(mm);
    double* Xu = cv.take<double>(mm);
    double* Xz = cv.take<double>(mm);
    double* svz = cv.take<double>(mm);
    double2* sv2 = cv.take<double2>(mm > SMALL_M ? mm : 1);
    double* Xzu = cv.take<double>(mm);
    double* part = cv.take<double>((size_t)2 * GRID_CAP * NV_MAX);
    double2* tilepart = cv.take<double2>(ntile_n + 1);
    unsigned long long* status = cv.take<unsigned long long>(status_words(n, m));   // (64-column coarse tiles)
    double2* hres = cv.take<double2>(std::max(nn, mm));
    double* parts = cv.take<double>(mm <= SMALL_M ? (size_t)(SM_MAX * 4 + 1) * mm + SM_MAX * 4 + 64 : 1);
    double* irpart = cv.take<double>((size_t)IR_NSLOT * IR_GMAX);
    int* slist = cv.take<int>(mm <= SMALL_M ? nn + 1 : 1);   // k_margins_small: supp(w) in column order
    int* dense_colptr = cv.take<int>(mm <= SMALL_M ? nn + 1 : 1);   // index-free dense X (small m)
    int* rowtab = cv.take<int>(mm <= SMALL_M ? mm : 1);
    const size_t ucap2 = mm > SMALL_M ? nn + (size_t)nnz / IR_UNIT + 64 : 1;   // k_inner<., true>: column units
    int2* uext = cv.take<int2>(ucap2);
    int* upos = cv.take<int>(ucap2);
    double2* upart = cv.take<double2>(ucap2);
    int* ustart = cv.take<int>(mm > SMALL_M ? nn + 1 : 1);
    int* uend = cv.take<int>(mm > SMALL_M ? nn + 1 : 1);
    long long* unz = cv.take<long long>(ucap2 + 1);
    ASet fine, coarse;
    fine.A = cv.take<int>(nn); fine.gA = cv.take<double>(nn); fine.hA = cv.take<double>(nn); fine.wA = cv.take<double>(nn);
    coarse.A = cv.take<int>(nn); coarse.gA = cv.take<double>(nn); coarse.hA = cv.take<double>(nn); coarse.wA = cv.take<double>(nn);
    double* d = cv.take<double>(nn);
    double* Hd = cv.take<double>(nn);
    double* s = cv.take<double>(nn);
    double* Hs = cv.take<double>(nn);
    double* u = cv.take<double>(nn);
    fine.d = coarse.d = d; fine.Hd = coarse.Hd = Hd; fine.s = coarse.s = s; fine.Hs = coarse.Hs = Hs; fine.u = coarse.u = u;
    size_t lvl_cap = 2 * nn + 2 * SEL_LMAX + 64;
    int* lvl = cv.take<int>(lvl_cap);
    unsigned char* lev = cv.take<unsigned char>(nn);
    // merge-path plans (large m): tile starts and carries for all columns and for a list, list offsets, outputs
    const bool big = mm > SMALL_M;
    const size_t mtiles = big ? (nn + (size_t)nnz) / MP_TILE + 2 : 1;
    int2* mp_ts_all = cv.take<int2>(mtiles + 1);
    double2* mp_cv_all = cv.take<double2>(mtiles);
    int* mp_cx_all = cv.take<int>(mtiles);
    int2* mp_ts_l = cv.take<int2>(mtiles + 1);
    double2* mp_cv_l = cv.take<double2>(mtiles);
    int* mp_cx_l = cv.take<int>(mtiles);
    int* mp_vptr = cv.take<int>(big ? nn + 1 : 1);
    int* mp_bsum = cv.take<int>(big ? nn / MP_SCAN + 2 : 1);
    double2* mp_out = cv.take<double2>(big ? nn : 1);
    // heavy-column path of the large-m inner solver (ml_heavy.cuh): the S and G copies of H's nonzeros (at most all
    // of X's), its warp chunks, per-row products, the zeroing columns' unit list
    const size_t hvn = big ? (size_t)nnz + 3 * mm + 16 : 1;   // (rows padded to whole 4-entry vectors)
    HvPrm hv{};
    hv.hid = cv.take<int>(big ? nn : 1);
    hv.phid = cv.take<int>(big ? nn : 1);
    int* hv_hcols = cv.take<int>(HV_HMAX + 1);
    int* hv_lens = cv.take<int>(HV_HMAX + 1);
    hv.sval = cv.take<float>(hvn);
    hv.sidx = cv.take<uint16_t>(hvn);
    hv.soff = cv.take<int>(big ? mm + 8 : 1);
    hv.schunk = cv.take<HvChunk>(big ? ((size_t)nnz + 3 * mm) / (HV_WCH / 2) + mm / HV_WROWS + 16 : 1);   // (greedy chunks)
    hv.Xh = cv.take<double>(big ? mm + 2 : 1);
    hv.sH = cv.take<double>(HV_HMAX);
    hv.zunits = cv.take<int>(ucap2);
    int* hv_bsum = cv.take<int>(big ? std::max(nn, mm + 1) / 1024 + 64 : 1);
    int* hv_misc = cv.take<int>(64);
    unsigned* hv_hist = cv.take<unsigned>(big ? 65536 : 1);

    UnitsMem um[4];
    for (int k = 0; k < 4; ++k) {
        um[k].u = cv.take<int4>(ucap);
        um[k].part = cv.take<double2>(ucap);
        um[k].hcnt = cv.take<int>(hcap);
        um[k].cap = (int)std::min<size_t>(ucap, 0x7fffffff);
        um[k].hcap = (int)hcap;
    }
    if (!c) return;
    c->ctl = ctl; c->sel = sel; c->trace = trace; c->hres = hres;
    c->lvl = lvl; c->lvl_cap = lvl_cap; c->lev = lev; c->parts = parts;
    c->fine = fine; c->coarse = coarse;
    for (int k = 0; k < 4; ++k) c->um[k] = um[k];
    Prm& P = c->P;
    P.w = w; P.wbits = wbits; P.z = z; P.rD = rD; P.Xd = Xd; P.Xs = Xs; P.sv = sv; P.Xu = Xu; P.parts = parts;
    P.Xz = Xz; P.svz = svz; P.Xzu = Xzu; P.sv2 = sv2;
    P.irpart = irpart;
    P.uext = uext; P.upos = upos; P.upart = upart; P.ustart = ustart; P.uend = uend; P.unz = unz;
    c->slist = slist;
    c->dense_colptr = dense_colptr;
    c->rowtab = rowtab;
    c->mp_tiles_cap = (int)std::min<size_t>(mtiles - 1, 0x7fffffff);
    c->mp_all = MPList{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, mp_ts_all, mp_cv_all, mp_cx_all};
    c->mp_l = MPList{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, mp_ts_l, mp_cv_l, mp_cx_l};
    c->mp_vptr = mp_vptr;
    c->mp_bsum = mp_bsum;
    c->mp_out = mp_out;
    P.ctl = ctl; P.part = part; P.tilepart = tilepart; P.status = status; P.trace = trace;
    hv.on = 0;
    P.hv = hv;
    c->hv_hcols = hv_hcols;
    c->hv_lens = hv_lens;
    c->hv_bsum = hv_bsum;
    c->hv_misc = hv_misc;
    c->hv_hist = hv_hist;
}

int pick_G(double mean_len) {
    if (mean_len < 12) return 4;
    if (mean_len < 64) return 8;   // (cfg 4 rows, mean 50: the margins pass 1.38 -> 1.22 ms with 8 lanes instead of 16)
    if (mean_len < 160) return 16;
    return 32;
}

Units units_of(ml_ctx* c, int slot) {
    Units U;
    U.u = c->um[slot].u;
    U.part = c->um[slot].part;
    U.hcnt = c->um[slot].hcnt;
    U.cap = c->um[slot].cap;
    U.n = c->ctl ? &c->ctl->units_n[slot] : nullptr;
    U.h = c->ctl ? &c->ctl->units_h[slot] : nullptr;
    U.claim = nullptr;
    return U;
}
// the same for a k_heavy launch that claims its units dynamically (the claim counter zeroed on the stream first);
// only where there are many units (nnz >= 16 M): on small X the memset and the claims cost more than the balance gains
Units units_claim(ml_ctx* c, int slot) {
    Units U = units_of(c, slot);
    if (c->X.nnz < CLAIM_NNZ) return U;
    cudaMemsetAsync(&c->ctl->hclaim, 0, sizeof(unsigned), c->st);
    U.claim = &c->ctl->hclaim;
    return U;
}

Seg seg_rows(ml_ctx* c) { return Seg{c->X.csr_rowptr, c->X.csr_col, c->X.csr_val, c->X.nnz, nullptr, c->hres, 8 * c->Gr}; }
Seg seg_cols(ml_ctx* c, const int* list) {
    return Seg{c->X.csc_colptr, c->X.csc_row, c->X.csc_val, c->X.nnz, list, c->hres, 8 * c->Gc,
               c->dense ? c->rowtab : nullptr};
}

#define ML_LAUNCH(c, kernel, grid, ...)                                                        \
    do {                                                                                       \
        kernel<<<(grid), ML_NT, 0, (c)->st>>>(__VA_ARGS__);                                   \
        (c)->launches++;                                                                       \
    } while (0)

#define ML_DISPATCH_G(Gv, BODY)                                 \
    switch (Gv) {                                               \
        case 4: { constexpr int GG = 4; BODY; } break;          \
        case 8: { constexpr int GG = 8; BODY; } break;          \
        case 16: { constexpr int GG = 16; BODY; } break;        \
        default: { constexpr int GG = 32; BODY; } break;        \
    }

ml_status cuda_fail(ml_ctx* c, const char* where) {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return ML_OK;
    if (c) c->err = std::string(where) + ": " + cudaGetErrorString(e);
    return ML_E_CUDA;
}

// RAII pass timer: records an event pair around one logical pass of class `cls` when that class is profiled
struct PassScope {
    ml_ctx* c;
    int cls;
    long long pair = -1;
    PassScope(ml_ctx* c_, int cls_) : c(c_), cls(cls_) {
        c->prof_passes[cls]++;
        if (!(c->prof_mask & (1u << cls))) return;
        if (c->ev_used + 2 > c->ev_pool.size()) {
            for (int k = 0; k < 256; ++k) { cudaEvent_t e; cudaEventCreate(&e); c->ev_pool.push_back(e); }
        }
        pair = (long long)(c->ev_used / 2);
        cudaEventRecord(c->ev_pool[c->ev_used], c->st);
        c->ev_used += 2;
        c->ev_cls.push_back(cls);
    }
    ~PassScope() {
        if (pair >= 0) cudaEventRecord(c->ev_pool[2 * pair + 1], c->st);
    }
};
inline long long* acc_of(ml_ctx* c, int cls) { return &c->ctl->cls[0][cls]; }

ml_status sync_ctl(ml_ctx* c) {
    cudaMemcpyAsync(&c->h, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c->st);
    cudaError_t e = cudaStreamSynchronize(c->st);
    if (e != cudaSuccess) { c->err = std::string("sync: ") + cudaGetErrorString(e); return ML_E_CUDA; }
    return cuda_fail(c, "sync");
}

// ------------------------------------------------------------------ small helper kernels
__global__ void k_init_rows(Prm P, int m) {   // w = 0: z = 0, r = -y/2, D = 1/4, L = m log 2
    for (int i = blockIdx.x * ML_NT + threadIdx.x; i < m; i += gridDim.x * ML_NT) {
        P.z[i] = 0.0;
        RowState s = row_state_i(P.y, P.b, i, 0.0);
        P.rD[i] = make_double2(s.r, s.D);
        P.Xs[i] = 0.0;
        P.Xd[i] = 0.0;
        P.Xu[i] = 0.0;
        P.Xz[i] = 0.0;
        P.Xzu[i] = 0.0;
    }
}
__global__ void k_check_y(const int8_t* y, int m, Ctl* ctl, unsigned long long* npos) {
    int bad = 0;
    unsigned long long pos = 0;
    for (int i = blockIdx.x * ML_NT + threadIdx.x; i < m; i += gridDim.x * ML_NT) {
        bad |= (y[i] != 1 && y[i] != -1);
        pos += (y[i] == 1);
    }
    if (bad) atomicOr(&ctl->bad_y, 1);
    pos = (unsigned long long)warp_sum_ll((long long)pos);
    if ((threadIdx.x & 31) == 0 && pos) atomicAdd(npos, pos);
}
// X's index structure: pointers non-decreasing with ptr[0] = 0, ptr[len] = nnz; indices in [0, bound) and strictly
// ascending inside every segment (the column passes rely on distinct rows within a column); flags ctl->bad_y |= 2.
// Element-parallel (long rows of a dense X are not one warp's serial loop): a descent idx[k] <= idx[k-1] is legal only
// at a segment start, so the descents counted over all k >= 1 minus those at the starts of non-empty segments
// (each start counted once) must be 0; the difference is summed into ctl->idx_desc (>= 0 per array).
__global__ void k_check_index(const int* ptr, const int* idx, const float* val, int len, int bound, long long nnz, Ctl* ctl) {
    const int lane = threadIdx.x & 31;
    const long long T = (long long)gridDim.x * blockDim.x, t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    int bad = 0;
    long long net = 0;
    for (long long s = t0; s < len; s += T) {   // pointers; descents at segment starts (subtracted)
        const int b = ptr[s], e = ptr[s + 1];
        if (b > e || b < 0 || (long long)e > nnz || (s == 0 && b != 0) || (s == len - 1 && (long long)e != nnz)) {
            bad = 1;
            continue;
        }
        if (idx && b < e && b > 0 && idx[b] <= idx[b - 1]) net -= 1;
    }
    int nonfin = 0;
    for (long long k = t0; k < nnz; k += T) {   // ranges; every descent (added); values finite
        nonfin |= !isfinite(val[k]);
        if (!idx) continue;   // (index-free dense X: values only)
        const int r = idx[k];
        bad |= (r < 0) || (r >= bound);
        if (k > 0 && r <= idx[k - 1]) net += 1;
    }
    if (bad) atomicOr(&ctl->bad_y, 2);
    if (nonfin) atomicOr(&ctl->bad_y, 4);
    net = warp_sum_ll(net);
    if (lane == 0 && net != 0) atomicAdd((unsigned long long*)&ctl->idx_desc, (unsigned long long)net);
}
// finiteness of a caller's fp64 vector (LASSO targets b, ml_set_w): flags ctl->bad_y |= flag
__global__ void k_check_finite(const double* v, long long len, Ctl* ctl, int flag) {
    int nonfin = 0;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < len; k += (long long)gridDim.x * blockDim.x)
        nonfin |= !isfinite(v[k]);
    if (__any_sync(0xffffffffu, nonfin) && (threadIdx.x & 31) == 0) atomicOr(&ctl->bad_y, flag);
}
// an index list C: in [0, n) and strictly ascending (include/ml.h); flags ctl->bad_y |= 16
__global__ void k_check_list(const int* C, long long nC, int n, Ctl* ctl) {
    int bad = 0;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < nC; k += (long long)gridDim.x * blockDim.x) {
        const int j = C[k];
        bad |= (j < 0) || (j >= n) || (k > 0 && j <= C[k - 1]);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&ctl->bad_y, 16);
}
__global__ void k_clear_flag(Ctl* ctl, int flag) { ctl->bad_y &= ~flag; }
// max |X_ij| and the longest row (the large-m solver's fixed-point scale of X_A s)
__global__ void k_xstats(const float* val, long long nnz, const int* rowptr, int m, Ctl* ctl) {
    double mx = 0.0;
    int mr = 0;
    const long long T = (long long)gridDim.x * blockDim.x, t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (long long k = t0; k < nnz; k += T) mx = fmax(mx, fabs((double)val[k]));
    for (long long i = t0; i < m; i += T) mr = max(mr, rowptr[i + 1] - rowptr[i]);
    mx = warp_max(mx);
    mr = __reduce_max_sync(0xffffffffu, (unsigned)mr);
    if ((threadIdx.x & 31) == 0) {
        atomic_max_nonneg(&ctl->xmax, mx);
        atomicMax(&ctl->maxrow, mr);
    }
}
// index-free dense X: column pointers j m and the row table t
__global__ void k_dense_init(int* colptr, int* rowtab, int m, int n) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k <= n || k < m; k += gridDim.x * blockDim.x) {
        if (k <= n) colptr[k] = k * m;
        if (k < m) rowtab[k] = k;
    }
}
// support bitmap, |supp| and ||w||_1 from w (deterministic: per-block partials + last block)
__global__ void __launch_bounds__(ML_NT) k_w_stats(Prm P, int n) {
    __shared__ double sm[3 * ML_NW + 3];
    Red<2> r;
    r.zero();
    const int nwords = (n + 31) / 32;
    for (int k = blockIdx.x * ML_NT + threadIdx.x; k < nwords; k += gridDim.x * ML_NT) {
        uint32_t b = 0;
        for (int q = 0; q < 32; ++q) {
            const int j = k * 32 + q;
            if (j < n) {
                const double v = P.w[j];
                if (v != 0.0) { b |= 1u << q; r.s[0] += 1.0; r.s[1] += fabs(v); }
            }
        }
        P.wbits[k] = b;
    }
    if (grid_reduce(r, P.part, &P.ctl->red_ctr[7], sm)) {
        if (threadIdx.x == 0) { P.ctl->nS = (int)r.s[0]; P.ctl->l1 = r.s[1]; }
    }
}
__global__ void k_get_rows(Prm P, int m, double* z, double* r, double* D) {
    for (int i = blockIdx.x * ML_NT + threadIdx.x; i < m; i += gridDim.x * ML_NT) {
        if (z) z[i] = P.z[i];
        if (r) r[i] = P.rD[i].x;
        if (D) D[i] = P.rD[i].y;
    }
}
__global__ void k_dmul(Prm P, int m) {   // sv = D o Xs (hessvec)
    for (int i = blockIdx.x * ML_NT + threadIdx.x; i < m; i += gridDim.x * ML_NT) P.sv[i] = P.rD[i].y * P.Xs[i];
}
__global__ void k_set_C(Ctl* ctl, int nC, int slot) {
    ctl->nC = nC;
    ctl->units_n[slot] = 0;
    ctl->units_h[slot] = 0;
}
// ml_shrink_linesearch preparation: the restriction C becomes the free set of a one-off relaxation
__global__ void k_ls_prep(Prm P, ASet AS, const int* C, int nC, const double* g, const double* h, const double* dC) {
    for (int p = blockIdx.x * ML_NT + threadIdx.x; p < nC; p += gridDim.x * ML_NT) {
        const int j = C ? C[p] : p;
        const double w = P.w[j];
        AS.A[p] = j;
        AS.gA[p] = g[p];
        AS.wA[p] = w;
        if (dC) AS.d[p] = dC[p];
        else {
            const double hh = h[p] + P.eps_h;
            AS.d[p] = soft(w - g[p] / hh, P.lam / hh) - w;   // Eq. 5 with D = diag(h) + eps_h
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        Ctl* c = P.ctl;
        c->nA = nC; c->nC = nC; c->skip = 0; c->ls_ok = 0; c->outcome = OUT_NOSTEP; c->level = -1;
        c->acc_steps = 1;
        c->F_before = c->F;
    }
}

// ------------------------------------------------------------------ launch sequences
void launch_units_build(ml_ctx* c, int slot, const int* list, int nlist_host) {
    Units U = units_of(c, slot);
    const int grid = std::max(1, std::min(GRID_CAP, (nlist_host + ML_NT - 1) / ML_NT));
    ML_LAUNCH(c, k_units_build, grid, c->X.csc_colptr, list, (const int*)nullptr, nlist_host, U, 8 * c->Gc);
}

// A1: heavy rows, then the light row kernel with the fused epilogue
void launch_margins(ml_ctx* c) {
    PassScope ps(c, CLS_MARGINS);
    if (c->sm_inner) {   // small m: z = X_S w_S over the support's columns, one cooperative launch
        Prm Pc = c->P;
        Seg S = seg_cols(c, nullptr);
        int* sl = c->slist;
        long long* ac = acc_of(c, CLS_MARGINS);
        void* args[] = {(void*)&Pc, (void*)&S, (void*)&sl, (void*)&ac};
        cudaLaunchCooperativeKernel(c->msmall_fn, dim3(c->inner_P), dim3(32 * IR_W), args, c->inner_bytes, c->st);
        c->launches++;
        return;
    }
    Seg S = seg_rows(c);
    ML_LAUNCH(c, (k_heavy<OpMargin, false>), c->gHeavy, S, units_claim(c, 3), OpMargin{c->P.w, c->P.wbits},
              (const double*)nullptr, (double*)nullptr, (const int*)nullptr, (const int*)nullptr, acc_of(c, CLS_MARGINS));
    const int grid = std::max(1, std::min(GRID_CAP, (int)((c->X.m + TILE - 1) / TILE)));
    ML_DISPATCH_G(c->Gr, ML_LAUNCH(c, k_margins<GG>, grid, c->P, S, acc_of(c, CLS_MARGINS)));
}

// merge-path plan of a list (virtual offsets by a three-launch scan, then the tile starts); list == nullptr: the
// static all-columns plan built at create
MPList mp_plan(ml_ctx* c, const int* list, const int* nC_dev, int nC_host) {
    if (!list) return c->mp_all;
    MPList L = c->mp_l;
    L.colptr = c->X.csc_colptr; L.idx = c->X.csc_row; L.val = c->X.csc_val;
    L.list = list; L.vptr = c->mp_vptr; L.nC_dev = nC_dev; L.nC_host = nC_host;
    const int nb = std::max(1, (nC_host + MP_SCAN - 1) / MP_SCAN);
    ML_LAUNCH(c, k_vscan_sums, nb, c->X.csc_colptr, list, nC_dev, nC_host, c->mp_bsum);
    k_vscan_top<<<1, 1024, 0, c->st>>>(c->mp_bsum, nC_dev, nC_host);
    c->launches++;
    ML_LAUNCH(c, k_vscan_apply, nb, c->X.csc_colptr, list, nC_dev, nC_host, c->mp_bsum, c->mp_vptr);
    const long long tiles = ((long long)nC_host + c->X.nnz) / MP_TILE + 2;
    ML_LAUNCH(c, k_mp_search, (int)std::max<long long>(1, (tiles + ML_NT) / ML_NT), L, c->mp_tiles_cap);
    return L;
}
template <class Term>
void mp_pass(ml_ctx* c, const MPList& L, Term term, double2* out, const int* skip, long long* acc) {
    const bool lst = L.list != nullptr;
    k_mp_pass<Term><<<lst ? c->mp_grid_l : c->mp_grid_all, MP_NT, mp_smem_bytes(lst), c->st>>>(L, term, out, skip, acc);
    ML_LAUNCH(c, k_mp_fixup, std::max(1, std::min(GRID_CAP, (c->mp_tiles_cap + ML_NT - 1) / ML_NT)), L, out, skip);
    c->launches++;
}
template <class Term>
bool mp_setup_kernel(ml_ctx* c) {
    int occ_l = 0, occ_a = 0;
    if (cudaFuncSetAttribute(k_mp_pass<Term>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mp_smem_bytes(true)) != cudaSuccess)
        return false;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_l, k_mp_pass<Term>, MP_NT, mp_smem_bytes(true));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_a, k_mp_pass<Term>, MP_NT, mp_smem_bytes(false));
    if (occ_l < 1 || occ_a < 1) return false;
    c->mp_grid_l = occ_l * c->sms;
    c->mp_grid_all = occ_a * c->sms;
    return true;
}

// A2 + A3 over C (list == nullptr: all columns, finest) into the ASet
// RELAX(C) start + A2/A3 over C.  Small m: one cooperative launch (k_gather_small also does k_relax_begin's work);
// large m: k_relax_begin, then the segment-engine gather.
void launch_relax_start(ml_ctx* c, int first_of_level, int level, const int* list, int nC_host, ASet& AS) {
    const bool finest = list == nullptr;
    if (!c->sm_inner) ML_LAUNCH(c, k_relax_begin, 1, c->P, first_of_level, level, list, nC_host, 1);
    const int cls = finest ? CLS_GATHER_FINE : CLS_GATHER_COARSE;
    PassScope ps(c, cls);
    Seg S = seg_cols(c, list);
    if (c->sm_inner) {   // small m: one cooperative launch (k_gather_small), (r, D) in shared memory
        Prm Pc = c->P;
        ASet A2 = AS;
        long long* ac = acc_of(c, cls);
        int fl = first_of_level, lv = level, nl = nC_host;
        void* args[] = {(void*)&Pc, (void*)&S, (void*)&A2, (void*)&ac, (void*)&fl, (void*)&lv, (void*)&nl};
        cudaLaunchCooperativeKernel(finest ? c->gsmall_fn[1] : c->gsmall_fn[0], dim3(c->inner_P), dim3(32 * IR_W), args,
                                    c->gsmall_bytes, c->st);
        c->launches++;
        return;
    }
    if (c->mp) {   // merge-path column sums into mp_out, then the free-set compaction from them
        MPList L = mp_plan(c, list, nullptr, nC_host);
        mp_pass(c, L, TermGH{c->P.rD}, c->mp_out, &c->ctl->skip, acc_of(c, cls));
        Seg So = S;
        So.hres = c->mp_out;
        const int ts = finest ? TILE : 64;
        const int grid = std::max(1, std::min(GRID_CAP, (nC_host + ts - 1) / ts));
        if (finest) ML_LAUNCH(c, (k_gather_free<32, true, true>), grid, c->P, So, AS, (long long*)nullptr);
        else ML_LAUNCH(c, (k_gather_free<32, false, true>), grid, c->P, So, AS, (long long*)nullptr);
        return;
    }
    ML_LAUNCH(c, (k_heavy<OpGH, false>), c->gHeavy, S, units_claim(c, list ? 1 : 0), OpGH{c->P.rD},
              (const double*)nullptr, (double*)nullptr, &c->ctl->skip, (const int*)nullptr, acc_of(c, cls));
    const int ts = finest ? TILE : 64;   // (k_gather_free's tile size)
    const int grid = std::max(1, std::min(GRID_CAP, (nC_host + ts - 1) / ts));
    if (finest && c->Gc == 4 && !list) {
        // Columns of a few nonzeros (cfg 5): the sums of all columns by the lean thread-per-column pass (32 registers,
        // 8 resident blocks per SM, no block barriers), then the compaction from S.hres.  Fused, the compaction's
        // barriers and look-back chain ran at 3 blocks per SM: 1.30 ms against 0.51 + 0.2 ms for the two passes.
        if (!c->gFine2) {   // whole waves: the tile loop is grid-strided (1184 blocks at 6 per SM left a third wave of a
                            // third of the blocks running alone: ncu, 55 % of the warp slots active)
            int occ = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gather_out<4, 3, OpGH>, ML_NT, 0) != cudaSuccess || occ < 1)
                occ = 4;
            cudaGetLastError();
            c->gFine2 = occ * c->sms;
        }
        const int g2 = std::max(1, std::min(c->gFine2, (nC_host + TILE - 1) / TILE));
        ML_LAUNCH(c, (k_gather_out<4, 3, OpGH>), g2, S, OpGH{c->P.rD}, (const int*)nullptr, nC_host, (double*)nullptr,
                  (double*)nullptr, acc_of(c, cls));
        ML_LAUNCH(c, (k_gather_free<32, true, true>), grid, c->P, S, AS, (long long*)nullptr);
        return;
    }
    if (finest) { ML_DISPATCH_G(c->Gc, ML_LAUNCH(c, (k_gather_free<GG, true>), grid, c->P, S, AS, acc_of(c, cls))); }
    else { ML_DISPATCH_G(c->Gc, ML_LAUNCH(c, (k_gather_free<GG, false>), grid, c->P, S, AS, acc_of(c, cls))); }
}

// X_C coef scatter for the API (A5): the result lands in `out` (atomic path: out zeroed by the caller; small-m path:
// per-block shared-memory m-vectors, partials summed in block order).
void launch_scatter(ml_ctx* c, int cls, const int* list, int slot, const int* nseg_dev, int nseg_host, const double* coef,
                    double* out) {
    Seg S = seg_cols(c, list);
    PassScope ps(c, cls);
    if (c->sm_scatter) {
        Prm Pc = c->P;
        int m = (int)c->X.m;
        long long* ac = acc_of(c, cls);
        double* parts = c->parts;
        void* args[] = {(void*)&S, (void*)&nseg_dev, (void*)&nseg_host, (void*)&coef, (void*)&parts, (void*)&m,
                        (void*)&ac, (void*)&Pc, (void*)&out};
        cudaLaunchCooperativeKernel((const void*)k_scatter_smem, dim3(c->scat_P), dim3(32 * c->scat_W), args,
                                    c->scat_bytes, c->st);
        c->launches++;
        return;
    }
    ML_LAUNCH(c, (k_heavy<OpDot, true>), c->gHeavy, S, units_claim(c, slot), OpDot{nullptr}, coef, out,
              (const int*)nullptr, (const int*)nullptr, acc_of(c, cls));
    ML_DISPATCH_G(c->Gc, ML_LAUNCH(c, k_scatter<GG>, c->gSeg, S, nseg_dev, nseg_host, coef, out, acc_of(c, cls)));
}

// out = X_C^T v for the API (mode 0: out0 = g, out1 = h via OpGH is api_gather; here mode 1: dot products)
void launch_gather_dot(ml_ctx* c, int cls, const int* list, int slot, const int* nseg_dev, int nseg_host, const double* v,
                       double* out) {
    PassScope ps(c, cls);
    Seg S = seg_cols(c, list);
    if (c->sm_gather) {
        k_gather_smem<<<c->gath_P, 32 * c->gath_W, c->gath_bytes, c->st>>>(S, nseg_dev, nseg_host, v, (int)c->X.m, out,
                                                                         acc_of(c, cls));
        c->launches++;
        return;
    }
    ML_LAUNCH(c, (k_heavy<OpDot, false>), c->gHeavy, S, units_claim(c, slot), OpDot{v}, (const double*)nullptr,
              (double*)nullptr, (const int*)nullptr, (const int*)nullptr, acc_of(c, cls));
    ML_DISPATCH_G(c->Gc, ML_LAUNCH(c, (k_gather_out<GG, 1, OpDot>), c->gSeg, S, OpDot{v}, nseg_dev, nseg_host, out,
                                   (double*)nullptr, acc_of(c, cls)));
}

// R3-R18 on the free set in AS (its gather already ran): one cooperative launch of the persistent inner solver runs
// the K inner iterations, the outer line search and the update, and writes the relaxation's trace row.
void launch_relax_body(ml_ctx* c, ASet& AS, int K, int inner_cg) {
    PassScope ps(c, CLS_INNER);
    Prm Pc = c->P;
    ASet A2 = AS;
    Seg S = seg_cols(c, AS.A);
    int Kk = K, icg = inner_cg;
    long long* a1 = acc_of(c, CLS_SCATTER);
    long long* a2 = acc_of(c, CLS_HS);
    void* args[] = {(void*)&Pc, (void*)&A2, (void*)&S, (void*)&Kk, (void*)&icg, (void*)&a1, (void*)&a2};
    const bool hv = c->inner_fn_hv && c->P.hv.on && c->P.hv.mode != 2;
    cudaLaunchCooperativeKernel(hv ? c->inner_fn_hv : c->inner_fn, dim3(c->inner_P), dim3(32 * IR_W), args,
                                hv ? c->inner_bytes_hv : c->inner_bytes, c->st);
    c->launches++;
}

void set_params(ml_ctx* c, const ml_solve_opts* o) {
    Prm& P = c->P;
    P.eps_h = o->eps_h;
    P.sigma_in = o->sigma_in;
    P.sigma_out = o->sigma_out;
    P.beta_ls = o->beta;
    P.tol = o->tol_kkt;
    P.eta = o->eta;
    P.max_ls = std::max(1, std::min(o->max_ls, ML_MAXLS));
    P.inner_cg = o->inner_cg;
    P.pcd_snap = o->pcd_snap;
}

// level sizes (P:194, P:602 via P:798; DESIGN section 3 S9-S10): k[0] = n, returns L
int level_sizes(int64_t nAf, int64_t nS, int64_t n, std::vector<int64_t>& k) {
    k.assign(1, n);
    int64_t k1 = std::max<int64_t>((nAf + 1) / 2, nS);
    if (k1 >= n) return 0;
    k.push_back(k1);
    while (k.back() != nS && (int)k.size() < SEL_LMAX + 1) k.push_back(std::max<int64_t>((k.back() + 1) / 2, nS));
    return (int)k.size() - 1;
}

// A8: radix select + emission of C_1..C_L into c->lvl (offsets returned)
void launch_select(ml_ctx* c, SelIn in, int nin_host, int L, const std::vector<int64_t>& targets, int* out,
                   const std::vector<int64_t>& loff) {
    I64x32 T{}, O{};
    for (int l = 0; l < L; ++l) { T.v[l] = targets[l]; O.v[l] = loff[l]; }
    // targets / offsets travel as kernel arguments (no host->device copies); one cooperative launch, a block per
    // 256 candidates (at most one per SM)
    PassScope ps(c, CLS_SELECT);
    int G = std::max(1, std::min(c->coop_cap, (nin_host + ML_NT - 1) / ML_NT));
    SelState* stp = c->sel;
    int Lv = L;
    void* args[] = {(void*)&in, (void*)&stp, (void*)&Lv, (void*)&T, (void*)&out, (void*)&O};
    cudaLaunchCooperativeKernel((const void*)k_select_coop, dim3(G), dim3(ML_NT), args, 0, c->st);
    c->launches++;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

void ml_default_opts(ml_solve_opts* o) {
    std::memset(o, 0, sizeof(*o));
    o->tol_kkt = 1e-6;
    o->max_cycles = 1000;
    o->nu = 1;
    o->nu_c = 5;
    o->K_fine = 2;
    o->K_mid = 3;
    o->K_coarse = 5;
    o->sigma_out = 1e-2;
    o->sigma_in = 1e-2;
    o->beta = 0.5;
    o->max_ls = 40;
    o->eps_h = 1e-12;
    o->multilevel = 1;
    o->inner_cg = 2;
    o->eta = 0.0;
    o->pcd_snap = 1;
    o->continuation = 0;
}

size_t ml_workspace_bytes(int64_t m, int64_t n, int64_t nnz) {
    if (m < 1 || n < 1 || nnz < 0) return 0;
    Carve cv{nullptr};
    carve_all(cv, nullptr, m, n, nnz);
    return cv.off + 256;
}

const char* ml_status_str(ml_status s) {
    switch (s) {
        case ML_OK: return "ok";
        case ML_E_INVAL: return "invalid argument";
        case ML_E_CUDA: return "CUDA error";
        case ML_E_WORKSPACE: return "workspace too small";
        case ML_E_STAGNATION: return "line search stagnation";
        case ML_E_NOT_CONVERGED: return "not converged";
        case ML_E_CONTRACT: return "objective increased (contract violation)";
        case ML_E_NONFINITE: return "non-finite input";
    }
    return "unknown";
}

const char* ml_last_error(const ml_ctx* c) { return c ? c->err.c_str() : "null context"; }
int64_t ml_kernel_launches(const ml_ctx* c) { return c ? c->launches : 0; }

// exclusive scan of a[0 .. n) in place (ml_heavy.cuh's three kernels; bsum holds n / 1024 + 1 ints)
void scan_excl(ml_ctx* c, int* a, long long n, int* bsum) {
    const int nbk = (int)((n + 1023) / 1024);
    k_scan_local<<<nbk, 256, 0, c->st>>>(a, (int)n, bsum);
    k_scan_bsum<<<1, 1024, 0, c->st>>>(bsum, nbk);
    k_scan_add<<<nbk, 256, 0, c->st>>>(a, (int)n, bsum);
    c->launches += 3;
}
// The heavy-column path (ml_heavy.cuh), built once per context: H = the longest columns (>= HV_MINLEN nonzeros, at
// most HV_HMAX, all columns of the shortest length taken or none), ids by decreasing length; the S copy (rows) and
// the G copy (bands) with their chunk schedules.  Off when H holds less than a tenth of X's nonzeros.
ml_status hv_build(ml_ctx* c) {
    HvPrm& hv = c->P.hv;
    hv.on = 0;
    const int m = (int)c->X.m, n = (int)c->X.n;
    const int* colptr = c->X.csc_colptr;
    auto sync = [&]() { return cudaStreamSynchronize(c->st) == cudaSuccess; };
    unsigned* hist = c->hv_hist;
    cudaMemsetAsync(hist, 0, sizeof(unsigned) * 65536, c->st);
    ML_LAUNCH(c, k_hv_lenhist, GRID_CAP, colptr, n, hist);
    std::vector<unsigned> hh(65536);
    cudaMemcpyAsync(hh.data(), hist, sizeof(unsigned) * 65536, cudaMemcpyDeviceToHost, c->st);
    if (!sync()) return cuda_fail(c, "hv_build");
    long long cum = 0;
    int T = 65536;
    for (int L = 65535; L >= HV_MINLEN; --L) {
        if (cum + hh[L] > HV_HMAX) break;
        cum += hh[L];
        T = L;
    }
    const int nh = (int)cum;
    if (nh == 0) return ML_OK;
    // heavy columns in column order, then ids by decreasing length (ties: column order)
    ML_LAUNCH(c, k_hv_flags, GRID_CAP, colptr, n, T, hv.phid);
    scan_excl(c, hv.phid, n, c->hv_bsum);
    ML_LAUNCH(c, k_hv_cols, GRID_CAP, colptr, n, T, hv.phid, c->hv_hcols, c->hv_lens);
    std::vector<int> hc(nh), hl(nh), ord(nh);
    cudaMemcpyAsync(hc.data(), c->hv_hcols, sizeof(int) * nh, cudaMemcpyDeviceToHost, c->st);
    cudaMemcpyAsync(hl.data(), c->hv_lens, sizeof(int) * nh, cudaMemcpyDeviceToHost, c->st);
    if (!sync()) return cuda_fail(c, "hv_build");
    long long nnzh = 0;
    for (int h = 0; h < nh; ++h) { ord[h] = h; nnzh += hl[h]; }
    if ((double)nnzh < 0.1 * (double)c->X.nnz) return ML_OK;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return hl[a] > hl[b]; });
    std::vector<int> hs(nh);
    for (int h = 0; h < nh; ++h) hs[h] = hc[ord[h]];
    cudaMemcpyAsync(c->hv_hcols, hs.data(), sizeof(int) * nh, cudaMemcpyHostToDevice, c->st);
    ML_LAUNCH(c, k_hv_hid, GRID_CAP, n, const_cast<int*>(hv.hid));
    ML_LAUNCH(c, k_hv_hid_set, 64, c->hv_hcols, nh, const_cast<int*>(hv.hid));
    // S copy: heavy entries per row, scanned to the row starts (soff)
    int* misc = c->hv_misc;
    cudaMemsetAsync(misc, 0, sizeof(int) * 64, c->st);
    int* hrp = const_cast<int*>(hv.soff);
    ML_LAUNCH(c, k_hv_rowcnt, GRID_CAP, c->X.csr_rowptr, c->X.csr_col, m, hv.hid, hrp, misc);
    cudaMemsetAsync(hrp + m, 0, sizeof(int), c->st);
    scan_excl(c, hrp, (long long)m + 1, c->hv_bsum);
    int maxcnt = 0;
    cudaMemcpyAsync(&maxcnt, misc, sizeof(int), cudaMemcpyDeviceToHost, c->st);
    if (!sync()) return cuda_fail(c, "hv_build");
    if (maxcnt < 1 || maxcnt > HV_WCH) return ML_OK;
    // warp chunks, greedily on the host: whole rows while the chunk holds at most HV_WCH entries and HV_WROWS rows
    std::vector<int> hr((size_t)m + 1);
    cudaMemcpyAsync(hr.data(), hrp, sizeof(int) * ((size_t)m + 1), cudaMemcpyDeviceToHost, c->st);
    if (!sync()) return cuda_fail(c, "hv_build");
    std::vector<HvChunk> chs;
    chs.reserve((size_t)m / HV_WROWS + (size_t)hr[m] / (HV_WCH / 2) + 16);
    for (int r = 0; r < m;) {
        const int r0 = r;
        while (r < m && r - r0 < HV_WROWS && hr[r + 1] - hr[r0] <= HV_WCH) ++r;
        chs.push_back(HvChunk{hr[r0], hr[r], r0, r - r0, hv_lg(r - r0), 0, 0, 0});
    }
    if (chs.size() > ((size_t)c->X.nnz + 3 * (size_t)m) / (HV_WCH / 2) + (size_t)m / HV_WROWS + 16) return ML_OK;   // (the workspace's chunk list)
    const int nts = (int)chs.size();
    cudaMemcpyAsync(const_cast<HvChunk*>(hv.schunk), chs.data(), sizeof(HvChunk) * chs.size(), cudaMemcpyHostToDevice,
                    c->st);
    ML_LAUNCH(c, k_hv_rowfill, GRID_CAP, c->X.csr_rowptr, c->X.csr_col, c->X.csr_val, m, hv.hid, hrp,
              const_cast<float*>(hv.sval), const_cast<uint16_t*>(hv.sidx));
    if (!sync()) return cuda_fail(c, "hv_build");
    cudaMemsetAsync(hv.Xh, 0, sizeof(double) * (size_t)m, c->st);
    cudaMemsetAsync(hv.sH, 0, sizeof(double) * HV_HMAX, c->st);
    hv.nh = nh;
    hv.nts = nts;
    hv.nnzh = nnzh;
    // on by default (chosen per relaxation by the free set's share of H) when H holds >= HV_AUTO nonzeros: below
    // that a warp gets too few chunks to amortise its ring, and the heavy instantiation's larger shared memory costs
    // the H sigma gathers L1 (measured: cfg 5 solve 460 -> 422 ms; cfg 3-4 slower with it)
    hv.mode = (long long)nnzh >= HV_AUTO ? 0 : 2;
    c->hv_mode0 = hv.mode;
    hv.frac = 0.25;
    hv.on = 1;
    return cuda_fail(c, "hv_build");
}

static ml_status create_impl(const ml_data* X, const double* b, double lambda, void* cuda_stream, void* ws,
                             size_t ws_bytes, ml_ctx** out) {
    if (!X || !out) return ML_E_INVAL;
    *out = nullptr;
    if (X->m < 1 || X->n < 1 || X->nnz < 0 || X->nnz >= 2147483647LL || X->m >= 2147483647LL || X->n >= 2147483647LL)
        return ML_E_INVAL;
    if (!(lambda > 0.0) || !std::isfinite(lambda)) return ML_E_INVAL;
    const bool has_csr = X->csr_rowptr != nullptr;   // (optional when m <= SMALL_M: checked once the solver path is known)
    // index-free dense X: no CSC pointers or row indices, every column full (nnz = m n), read by columns (small m)
    const bool dense = !X->csc_colptr && !X->csc_row && X->nnz == X->m * X->n;
    if (dense && (X->m > SMALL_M || has_csr || !X->csc_val || (!X->y && !b))) return ML_E_INVAL;
    if (!dense && (!X->csc_colptr || (!X->y && !b) || (X->nnz > 0 && (!X->csc_row || !X->csc_val)) ||
                   (has_csr && X->nnz > 0 && (!X->csr_col || !X->csr_val))))
        return ML_E_INVAL;
    // the index / value arrays are streamed with 16-byte vector loads and TMA bulk copies: 16-byte alignment
    auto mis16 = [](const void* p) { return ((uintptr_t)p & 15u) != 0; };
    if (mis16(X->csc_row) || mis16(X->csc_val) || (has_csr && (mis16(X->csr_col) || mis16(X->csr_val))) ||
        ((uintptr_t)X->csc_colptr & 3u) || (has_csr && ((uintptr_t)X->csr_rowptr & 3u)) || ((uintptr_t)b & 7u))
        return ML_E_INVAL;
    const size_t need = ml_workspace_bytes(X->m, X->n, X->nnz);
    if (!ws || ws_bytes < need) return ML_E_WORKSPACE;
    ml_ctx* c = new ml_ctx();
    c->X = *X;
    c->lam = lambda;
    c->st = (cudaStream_t)cuda_stream;
    {
        int dev = 0, sms = 0;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
            c->sms = std::min(sms, SM_MAX);   // (the partial buffers are sized for at most SM_MAX blocks)
        c->coop_cap = c->sms;
    }
    c->ws = (char*)align_up((size_t)ws);
    c->ws_bytes = ws_bytes;
    Carve cv{c->ws};
    carve_all(cv, c, X->m, X->n, X->nnz);
    if (dense) {
        c->dense = true;
        c->X.csc_colptr = c->dense_colptr;   // (filled below; csc_row stays NULL: Seg::idx == nullptr selects the
    }                                         //  index-free reads)
    Prm& P = c->P;
    P.m = (int)X->m;
    P.n = (int)X->n;
    P.y = X->y;
    P.b = b;
    P.lam = lambda;
    ml_solve_opts o;
    ml_default_opts(&o);
    set_params(c, &o);
    c->Gr = pick_G((double)X->nnz / (double)X->m);
    c->Gc = pick_G((double)X->nnz / (double)X->n);
    c->gA = std::max(1, std::min(GRID_CAP, (int)((X->n + ML_NT - 1) / ML_NT)));
    c->gM = std::max(1, std::min(GRID_CAP, (int)((X->m + ML_NT - 1) / ML_NT)));
    c->gSeg = std::max(1, std::min(GRID_CAP, (int)((X->n + ML_NT - 1) / ML_NT)));
    c->gHeavy = std::max(1, std::min(GRID_CAP, (int)((X->nnz / CHUNK + std::min<int64_t>(std::max(X->m, X->n), X->nnz / SPLIT_MIN) + 8) / ML_NW + 1)));
    {   // whole waves only: the unit loop is grid-strided, so a partial second wave (592 blocks at 3 per SM) only
        // delays the blocks that start late
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_heavy<OpGH, false>, ML_NT, 0) == cudaSuccess && occ > 0)
            c->gHeavy = std::max(1, std::min(c->gHeavy, occ * c->sms));
        cudaGetLastError();
    }
    if (X->m <= SMALL_M) {   // shared-memory passes: W warps per block, private m-vectors / shared sv + TMA rings
        int W = 16;
        while (W > 1 && scatter_smem_bytes(W, (int)X->m) > 200 * 1024) --W;
        size_t bytes = scatter_smem_bytes(W, (int)X->m);
        if (W >= 2 && bytes <= 220 * 1024 &&
            cudaFuncSetAttribute(k_scatter_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess) {
            int bps = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_scatter_smem, 32 * W, bytes);
            bps = std::min(bps, 4);
            c->sm_scatter = bps >= 1;
            c->scat_W = W;
            c->scat_bytes = bytes;
            c->scat_bps = bps;
            c->scat_P = c->sms * bps;
            c->gMP = std::max(1, std::min(GRID_CAP, (int)((X->m + 15) / 16)));
            c->gMP = std::max(c->gMP, (int)((X->m + ML_NT - 1) / ML_NT));
        }
        W = 16;
        while (W > 1 && gather_smem_bytes(W, (int)X->m) > 200 * 1024) --W;
        bytes = gather_smem_bytes(W, (int)X->m);
        if (W >= 2 && bytes <= 220 * 1024 &&
            cudaFuncSetAttribute(k_gather_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess) {
            const int bps = std::max(1, std::min(4, (int)((228 * 1024) / (bytes + 1024))));
            c->sm_gather = true;
            c->gath_W = W;
            c->gath_bytes = bytes;
            c->gath_bps = bps;
            c->gath_P = c->sms * bps;
        }
        // persistent inner solver: 1024-element G chunks when the two m-vectors leave room, else 512
        const bool big_g = inner_smem_bytes<1024>((int)X->m) <= IR_SMEM_MAX;
        const void* kfn = big_g ? (const void*)k_inner<1024, IN_GST, false> : (const void*)k_inner<512, IN_GST, false>;
        bytes = big_g ? inner_smem_bytes<1024>((int)X->m) : inner_smem_bytes<512>((int)X->m);
        if (bytes <= IR_SMEM_MAX && X->m <= (int64_t)IR_RS * std::min(c->sms, IR_GMAX) &&
            cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess) {
            int bps = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kfn, 32 * IR_W, bytes);
            const void* g0 = big_g ? (const void*)k_gather_small<1024, false> : (const void*)k_gather_small<512, false>;
            const void* g1 = big_g ? (const void*)k_gather_small<1024, true> : (const void*)k_gather_small<512, true>;
            const size_t gb = big_g ? gather_small_smem_bytes<1024>((int)X->m) : gather_small_smem_bytes<512>((int)X->m);
            const void* mf = big_g ? (const void*)k_margins_small<1024> : (const void*)k_margins_small<512>;
            int gps0 = 0, gps1 = 0, mps = 0;
            if (gb <= 220 * 1024 &&
                cudaFuncSetAttribute(g0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gb) == cudaSuccess &&
                cudaFuncSetAttribute(g1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gb) == cudaSuccess &&
                cudaFuncSetAttribute(mf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess) {
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&gps0, g0, 32 * IR_W, gb);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&gps1, g1, 32 * IR_W, gb);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&mps, mf, 32 * IR_W, bytes);
            }
            if (bps >= 1 && gps0 >= 1 && gps1 >= 1 && mps >= 1) {
                c->msmall_fn = mf;
                c->sm_inner = true;
                c->inner_fn = kfn;
                c->inner_bytes = bytes;
                c->inner_P = std::min(c->sms, IR_GMAX);
                c->gsmall_fn[0] = g0;
                c->gsmall_fn[1] = g1;
                c->gsmall_bytes = gb;
            }
        }
        cudaGetLastError();
    }
    if (!c->sm_inner) {   // large m: the persistent solver with global m-vectors
        // (measured: <256, 8> and <512, 4> rings were slower on cfg 3-4); a second instantiation carries the
        // heavy-column path (its shared memory would shrink L1 for the default one)
        const void* kfn = (const void*)k_inner<1024, IN_GST, true>;
        const size_t b = inner_big_smem_bytes<1024, IN_GST>();
        const void* kfh = (const void*)k_inner<IR_HSCH, IR_HST, true, true>;
        const size_t bh = std::max(inner_big_smem_bytes<IR_HSCH, IR_HST>(), hv_smem_bytes());
        int bps = 0, bph = 0;
        if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b) == cudaSuccess)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kfn, 32 * IR_W, b);
        if (cudaFuncSetAttribute(kfh, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bh) == cudaSuccess)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bph, kfh, 32 * IR_W, bh);
        cudaGetLastError();
        if (bps >= 1) {
            c->big_inner = true;
            c->inner_fn = kfn;
            c->inner_bytes = b;
            c->inner_P = std::min(c->sms, IR_GMAX);
            if (bph >= 1) { c->inner_fn_hv = kfh; c->inner_bytes_hv = bh; }
        }
    }
    if (!c->sm_inner && mp_setup_kernel<TermGH>(c) && mp_setup_kernel<TermV2>(c) && mp_setup_kernel<TermV1>(c)) {
        c->mp = false;   // large m: merge-path column passes (ml_merge.cuh) on request (ml_set_engine bit 0)
        c->mp_all.colptr = X->csc_colptr; c->mp_all.idx = X->csc_row; c->mp_all.val = X->csc_val;
        c->mp_all.list = nullptr; c->mp_all.vptr = X->csc_colptr; c->mp_all.nC_dev = nullptr; c->mp_all.nC_host = (int)X->n;
    }
    cudaGetLastError();
    if (!has_csr && !c->sm_inner) {   // the large-m margins and heavy-row schedule read X by rows
        delete c;
        return ML_E_INVAL;
    }
    // zero the control block, trace, bitmap, iterate and the heavy-unit counters
    cudaMemsetAsync(c->ctl, 0, sizeof(Ctl), c->st);
    cudaMemsetAsync(P.w, 0, sizeof(double) * X->n, c->st);
    cudaMemsetAsync(P.wbits, 0, sizeof(uint32_t) * ((X->n + 31) / 32 + 1), c->st);
    cudaMemsetAsync(P.status, 0, sizeof(unsigned long long) * status_words(X->n, X->m), c->st);
    for (int k = 0; k < 4; ++k) cudaMemsetAsync(c->um[k].hcnt, 0, sizeof(int) * c->um[k].hcap, c->st);
    Ctl init;
    std::memset(&init, 0, sizeof(init));
    init.trace_cap = TRACE_CAP;
    init.L = b ? 0.0 : (double)X->m * std::log(2.0);   // (the first margins pass recomputes L)
    init.F = init.L;
    cudaMemcpyAsync(c->ctl, &init, sizeof(Ctl), cudaMemcpyHostToDevice, c->st);
    unsigned long long* npos_dev = reinterpret_cast<unsigned long long*>(&c->ctl->dsupp);
    if (!b) ML_LAUNCH(c, k_check_y, c->gM, X->y, (int)X->m, c->ctl, npos_dev);   // (squared loss: no labels)
    if (dense) ML_LAUNCH(c, k_dense_init, GRID_CAP, c->dense_colptr, c->rowtab, (int)X->m, (int)X->n);
    ML_LAUNCH(c, k_check_index, GRID_CAP, c->X.csc_colptr, X->csc_row, X->csc_val, (int)X->n, (int)X->m, X->nnz, c->ctl);
    if (has_csr) ML_LAUNCH(c, k_check_index, GRID_CAP, X->csr_rowptr, X->csr_col, X->csr_val, (int)X->m, (int)X->n, X->nnz, c->ctl);
    if (b) ML_LAUNCH(c, k_check_finite, c->gM, b, (long long)X->m, c->ctl, 8);
    ML_LAUNCH(c, k_init_rows, c->gM, P, (int)X->m);
    if (c->big_inner) ML_LAUNCH(c, k_xstats, GRID_CAP, X->csc_val, X->nnz, X->csr_rowptr, (int)X->m, c->ctl);
    if (c->big_inner && c->inner_fn_hv && has_csr && X->nnz >= HV_AUTO) {   // large X: the heavy path by default
        c->hv_built = true;
        const ml_status hs = hv_build(c);
        if (hs != ML_OK) { *out = c; return hs; }
    }
    if (c->mp_grid_all)   // the static merge-path plan over all columns (X is fixed for the context's life)
        ML_LAUNCH(c, k_mp_search, std::max(1, (c->mp_tiles_cap + ML_NT) / ML_NT), c->mp_all, c->mp_tiles_cap);
    // static heavy schedules: all columns (slot 0) and all rows (slot 3)
    {
        Units U = units_of(c, 0);
        ML_LAUNCH(c, k_units_build, c->gSeg, c->X.csc_colptr, (const int*)nullptr, (const int*)nullptr, (int)X->n, U, 8 * c->Gc);
        Units R = units_of(c, 3);
        if (has_csr)
            ML_LAUNCH(c, k_units_build, c->gM, X->csr_rowptr, (const int*)nullptr, (const int*)nullptr, (int)X->m, R, 8 * c->Gr);
    }
    ml_status s = sync_ctl(c);
    if (s != ML_OK) { *out = c; return s; }
    if (c->h.bad_y || c->h.idx_desc != 0) {   // bit 0: labels not +-1; bit 1 / descents: malformed CSR / CSC;
        // bit 2: non-finite X values; bit 3: non-finite LASSO targets
        const bool index = (c->h.bad_y & 3) || c->h.idx_desc != 0;
        delete c;
        return index ? ML_E_INVAL : ML_E_NONFINITE;
    }
    c->npos = (long long)c->h.dsupp;
    long long zero = 0;
    cudaMemcpyAsync(&c->ctl->dsupp, &zero, sizeof(long long), cudaMemcpyHostToDevice, c->st);
    if (c->h.units_n[0] > c->um[0].cap || c->h.units_n[3] > c->um[3].cap) { c->err = "unit capacity"; delete c; return ML_E_WORKSPACE; }
    s = sync_ctl(c);
    *out = c;
    return s;
}

ml_status ml_create(const ml_data* X, double lambda, void* cuda_stream, void* ws, size_t ws_bytes, ml_ctx** out) {
    return create_impl(X, nullptr, lambda, cuda_stream, ws, ws_bytes, out);
}
ml_status ml_create_lasso(const ml_data* X, const double* b, double lambda, void* cuda_stream, void* ws, size_t ws_bytes,
                          ml_ctx** out) {
    if (!b) return ML_E_INVAL;
    return create_impl(X, b, lambda, cuda_stream, ws, ws_bytes, out);
}

ml_status ml_destroy(ml_ctx* c) {
    if (!c) return ML_E_INVAL;
    cudaStreamSynchronize(c->st);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    delete c;
    return ML_OK;
}

ml_status ml_set_w(ml_ctx* c, const double* w_dev) {
    if (!c || !w_dev) return ML_E_INVAL;
    ML_LAUNCH(c, k_check_finite, c->gA, w_dev, (long long)c->X.n, c->ctl, 32);
    ml_status s = sync_ctl(c);
    if (s != ML_OK) return s;
    if (c->h.bad_y & 32) {   // w is left unchanged
        ML_LAUNCH(c, k_clear_flag, 1, c->ctl, 32);
        return ML_E_NONFINITE;
    }
    cudaMemcpyAsync(c->P.w, w_dev, sizeof(double) * c->X.n, cudaMemcpyDeviceToDevice, c->st);
    ML_LAUNCH(c, k_w_stats, c->gA, c->P, (int)c->X.n);
    return cuda_fail(c, "ml_set_w");
}

ml_status ml_get_w(ml_ctx* c, double* w_dev) {
    if (!c || !w_dev) return ML_E_INVAL;
    cudaMemcpyAsync(w_dev, c->P.w, sizeof(double) * c->X.n, cudaMemcpyDeviceToDevice, c->st);
    return cuda_fail(c, "ml_get_w");
}

ml_status ml_get_rows(ml_ctx* c, double* z, double* r, double* D) {
    if (!c) return ML_E_INVAL;
    ML_LAUNCH(c, k_get_rows, c->gM, c->P, (int)c->X.m, z, r, D);
    return cuda_fail(c, "ml_get_rows");
}

// C == NULL with nC == n, or nC entries strictly ascending in [0, n): one device pass and a stream synchronisation
static ml_status check_list(ml_ctx* c, const int32_t* C, int64_t nC) {
    if (!C) return nC == c->X.n ? ML_OK : ML_E_INVAL;
    if (nC < 0 || nC > c->X.n) return ML_E_INVAL;
    if (nC == 0) return ML_OK;
    ML_LAUNCH(c, k_check_list, std::max(1, std::min(GRID_CAP, (int)((nC + ML_NT - 1) / ML_NT))), C, (long long)nC,
              (int)c->X.n, c->ctl);
    ml_status s = sync_ctl(c);
    if (s != ML_OK) return s;
    if (c->h.bad_y & 16) {
        ML_LAUNCH(c, k_clear_flag, 1, c->ctl, 16);
        c->err = "C: indices must be strictly ascending in [0, n)";
        return ML_E_INVAL;
    }
    return ML_OK;
}

// gather g_C / h_C over an explicit list (API path)
static void api_gather(ml_ctx* c, const int32_t* C, int nC, double* g_C, double* h_C) {
    int slot = C ? 1 : 0;
    if (C) {
        ML_LAUNCH(c, k_set_C, 1, c->ctl, nC, 1);
        launch_units_build(c, 1, C, nC);
    }
    PassScope ps(c, CLS_API);
    Seg S = seg_cols(c, C);
    ML_LAUNCH(c, (k_heavy<OpGH, false>), c->gHeavy, S, units_claim(c, slot), OpGH{c->P.rD}, (const double*)nullptr,
              (double*)nullptr, (const int*)nullptr, (const int*)nullptr, acc_of(c, CLS_API));
    // (thread-per-column tiles, Gc == 4: 32 registers, latency-bound serial column loops: 8 resident blocks per SM)
    const int grid = std::max(1, std::min((c->Gc == 4 ? 2 : 1) * GRID_CAP, (nC + TILE - 1) / TILE));
    ML_DISPATCH_G(c->Gc, ML_LAUNCH(c, (k_gather_out<GG, 0, OpGH>), grid, S, OpGH{c->P.rD}, (const int*)nullptr, nC,
                                   g_C, h_C, acc_of(c, CLS_API)));
}

ml_status ml_eval_f_grad(ml_ctx* c, const int32_t* C, int64_t nC, double* F_host, double* g_C, double* h_C) {
    if (!c) return ML_E_INVAL;
    if (ml_status s = check_list(c, C, nC)) return s;
    launch_margins(c);
    if ((g_C || h_C) && nC > 0) api_gather(c, C, (int)nC, g_C, h_C);
    if (F_host) {
        ml_status s = sync_ctl(c);
        if (s != ML_OK) return s;
        *F_host = c->h.F;
    }
    return cuda_fail(c, "ml_eval_f_grad");
}

ml_status ml_diag_hess(ml_ctx* c, const int32_t* C, int64_t nC, double* h_C) {
    if (!c || !h_C) return ML_E_INVAL;
    if (ml_status s = check_list(c, C, nC)) return s;
    if (nC > 0) api_gather(c, C, (int)nC, nullptr, h_C);
    return cuda_fail(c, "ml_diag_hess");
}

ml_status ml_hessvec(ml_ctx* c, const int32_t* C, int64_t nC, const double* v_C, double* Hv_C) {
    if (!c || !v_C || !Hv_C) return ML_E_INVAL;
    if (ml_status s = check_list(c, C, nC)) return s;
    if (nC == 0) return ML_OK;
    const int slot = C ? 1 : 0;
    if (C) {
        ML_LAUNCH(c, k_set_C, 1, c->ctl, (int)nC, 1);
        launch_units_build(c, 1, C, (int)nC);
    }
    cudaMemsetAsync(c->P.Xs, 0, sizeof(double) * c->X.m, c->st);
    launch_scatter(c, CLS_API, C, slot, nullptr, (int)nC, v_C, c->P.Xs);   // X_C v
    ML_LAUNCH(c, k_dmul, c->gM, c->P, (int)c->X.m);                                   // D o X_C v
    launch_gather_dot(c, CLS_API, C, slot, nullptr, (int)nC, c->P.sv, Hv_C);
    cudaMemsetAsync(c->P.Xs, 0, sizeof(double) * c->X.m, c->st);
    return cuda_fail(c, "ml_hessvec");
}

ml_status ml_shrink_linesearch(ml_ctx* c, const int32_t* C, int64_t nC, const double* g_C, const double* h_C,
                               const double* d_C, const double* Xd, const ml_solve_opts* o, double* alpha_host,
                               double* F_new_host) {
    if (!c || !g_C || (!d_C && !h_C)) return ML_E_INVAL;
    if (ml_status s = check_list(c, C, nC)) return s;
    ml_solve_opts def;
    ml_default_opts(&def);
    set_params(c, o ? o : &def);
    ASet& AS = c->coarse;
    const int n = (int)nC;
    ML_LAUNCH(c, k_ls_prep, c->gA, c->P, AS, C, n, g_C, h_C, d_C);
    if (Xd) cudaMemcpyAsync(c->P.Xd, Xd, sizeof(double) * c->X.m, cudaMemcpyDeviceToDevice, c->st);
    else {
        const int slot = C ? 1 : 0;
        if (C) {
            ML_LAUNCH(c, k_set_C, 1, c->ctl, n, 1);
            launch_units_build(c, 1, C, n);
        }
        cudaMemsetAsync(c->P.Xd, 0, sizeof(double) * c->X.m, c->st);
        launch_scatter(c, CLS_API, C, slot, nullptr, n, AS.d, c->P.Xd);
    }
    const int nblkA = c->gA;
    ML_LAUNCH(c, k_outer_ls<4>, nblkA + c->gM, c->P, AS, 0, nblkA);
    ML_LAUNCH(c, k_outer_ls<ML_MAXLS - 4>, nblkA + c->gM, c->P, AS, 4, nblkA);
    ML_LAUNCH(c, k_update, nblkA + c->gM, c->P, AS, nblkA);
    ml_status s = sync_ctl(c);
    if (s != ML_OK) return s;
    if (alpha_host) *alpha_host = c->h.ls_ok ? c->h.alpha : 0.0;
    if (F_new_host) *F_new_host = c->h.F;
    if (c->h.outcome == OUT_STAGNATION) return ML_E_STAGNATION;
    return ML_OK;
}

ml_status ml_select_coarse(ml_ctx* c, const double* g, int64_t k_total, int32_t* C_out, int64_t* nC_out_host) {
    if (!c || !g || !C_out) return ML_E_INVAL;
    ml_status s = sync_ctl(c);
    if (s != ML_OK) return s;
    const int64_t n = c->X.n, nS = c->h.nS;
    int64_t T = std::max<int64_t>(0, std::min<int64_t>(k_total - nS, n - nS));
    SelIn in{nullptr, g, nullptr, (int)n, c->P.w, c->lev};
    std::vector<int64_t> targets{T}, loff{0};
    launch_select(c, in, (int)n, 1, targets, C_out, loff);
    if (nC_out_host) *nC_out_host = nS + T;
    return cuda_fail(c, "ml_select_coarse");
}

ml_status ml_solve(ml_ctx* c, const ml_solve_opts* o_in, ml_solve_report* rep) {
    if (!c || !rep) return ML_E_INVAL;
    ml_solve_opts o;
    if (o_in) o = *o_in; else ml_default_opts(&o);
    if (o.K_fine < 1 || o.K_mid < 1 || o.K_coarse < 1 || o.nu < 1 || o.nu_c < 1) return ML_E_INVAL;
    set_params(c, &o);
    std::memset(rep, 0, sizeof(*rep));
    const long long launches0 = c->launches;
    long long nnz0 = 0;
    const long long passes0 = c->prof_passes[CLS_MARGINS] + c->prof_passes[CLS_GATHER_FINE] +
                              c->prof_passes[CLS_GATHER_COARSE] + c->prof_passes[CLS_SCATTER] + c->prof_passes[CLS_HS];
    const int n = (int)c->X.n;
    Ctl* ctl = c->ctl;
    // S1: w = 0, z = 0 (per-sample state refreshed by the first margins pass)
    cudaMemsetAsync(c->P.w, 0, sizeof(double) * n, c->st);
    cudaMemsetAsync(c->P.wbits, 0, sizeof(uint32_t) * ((n + 31) / 32 + 1), c->st);
    {
        Ctl h0;
        ml_status s = sync_ctl(c);
        if (s != ML_OK) return s;
        h0 = c->h;
        for (int k = 0; k < 16; ++k) nnz0 += h0.cls[0][k];
        h0.nS = 0; h0.l1 = 0.0; h0.ntrace = 0; h0.level_conv = 0; h0.skip = 0;
        h0.vmax_bits = 0ull; h0.dsupp = 0;
        cudaMemcpyAsync(ctl, &h0, sizeof(Ctl), cudaMemcpyHostToDevice, c->st);
    }
    auto eval_and_fine_relax = [&](bool relax) {
        // S2/S15 EVAL_ALL (margins from scratch + full gather with the free set), then S4/S17 RELAX(C0, E)
        launch_margins(c);
        launch_relax_start(c, 1, 0, nullptr, n, c->fine);
        if (relax) {
            launch_relax_body(c, c->fine, o.K_fine, o.inner_cg);
            for (int it = 1; it < o.nu; ++it) {
                launch_relax_start(c, 0, 0, nullptr, n, c->fine);
                launch_relax_body(c, c->fine, o.K_fine, o.inner_cg);
            }
        }
    };
    double v1_0 = -1.0;
    if (o.continuation) {
        // Continuation (DESIGN Q28): EVAL_ALL at w = 0 gives lambda_max = vmax + lambda; one finest
        // relaxation at each of lambda_4 = (lambda_max + lambda) / 2 > lambda_3 > lambda_2 (linearly spaced down to
        // lambda), each with its own free-set gather; then the solve at lambda from that warm start.
        launch_margins(c);
        launch_relax_start(c, 1, 0, nullptr, n, c->fine);
        ml_status s0 = sync_ctl(c);
        if (s0 != ML_OK) return s0;
        v1_0 = c->h.v1;
        if (c->h.vmax / c->lam > o.tol_kkt) {
            const double lam1 = c->lam, lam4 = 0.5 * ((c->h.vmax + lam1) + lam1);
            for (int kk = 4; kk >= 2; --kk) {
                c->P.lam = lam1 + (lam4 - lam1) * (double)(kk - 1) / 3.0;
                launch_relax_start(c, 1, 0, nullptr, n, c->fine);
                launch_relax_body(c, c->fine, o.K_fine, o.inner_cg);
            }
            c->P.lam = lam1;
        }
    }
    eval_and_fine_relax(true);
    ml_status s = sync_ctl(c);
    if (s != ML_OK) return s;
    if (v1_0 < 0.0) v1_0 = c->h.v1;
    bool converged = c->h.vmax / c->lam <= o.tol_kkt;
    int cycle = 0;
    int64_t max_supp = c->h.nS;
    std::vector<int64_t> k;
    if (!converged) {
        for (cycle = 1; cycle <= o.max_cycles; ++cycle) {
            const int64_t nS = c->h.nS, nAf = c->h.nAf;
            if (o.multilevel && nS > 0) {
                const int L = level_sizes(nAf, nS, n, k);
                if (L >= 1) {
                    std::vector<int64_t> targets(L), loff(L);
                    int64_t acc = 0;
                    for (int l = 1; l <= L; ++l) { targets[l - 1] = k[l] - nS; loff[l - 1] = acc; acc += k[l]; }
                    SelIn in{c->fine.A, c->fine.gA, &ctl->nAf, 0, c->P.w, c->lev};
                    launch_select(c, in, (int)nAf, L, targets, c->lvl, loff);
                    for (int l = L; l >= 1; --l) {
                        const int* Cl = c->lvl + loff[l - 1];
                        const int nCl = (int)k[l];
                        ML_LAUNCH(c, k_set_C, 1, ctl, nCl, 1);
                        if (!c->sm_inner) launch_units_build(c, 1, Cl, nCl);   // heavy units of the generic gathers
                        const int reps = (l == L) ? o.nu_c : o.nu;
                        const int K = (l == L) ? o.K_coarse : o.K_mid;
                        for (int r = 0; r < reps; ++r) {
                            launch_relax_start(c, r == 0 ? 1 : 0, l, Cl, nCl, c->coarse);
                            launch_relax_body(c, c->coarse, K, o.inner_cg);
                        }
                    }
                }
            }
            eval_and_fine_relax(true);
            s = sync_ctl(c);
            if (s != ML_OK) return s;
            max_supp = std::max<int64_t>(max_supp, c->h.nS);
            if (c->h.vmax / c->lam <= o.tol_kkt) { converged = true; break; }
        }
    }
    // the returned w is the evaluated one (DESIGN Q17): the last finest relaxation was skipped on convergence.
    // On NOT_CONVERGED, re-evaluate so that F / kappa describe the returned w.
    if (!converged) {
        eval_and_fine_relax(false);
        s = sync_ctl(c);
        if (s != ML_OK) return s;
    }
    const Ctl& h = c->h;
    rep->F = h.F;
    rep->vinf = h.vmax;
    rep->kappa = h.vmax / c->lam;
    rep->v1 = h.v1;
    const long long minpm = std::min<long long>(c->npos, c->X.m - c->npos);
    rep->paper_ratio = (v1_0 > 0 && minpm > 0) ? h.v1 / (v1_0 * (double)minpm / (double)c->X.m) : 0.0;
    rep->cycles = std::min(cycle, o.max_cycles);
    rep->nnz_w = h.nS;
    rep->max_supp = std::max<int64_t>(max_supp, h.nS);
    rep->nnz_touched = -nnz0;
    for (int k = 0; k < 16; ++k) rep->nnz_touched += h.cls[0][k];
    rep->x_passes = c->prof_passes[CLS_MARGINS] + c->prof_passes[CLS_GATHER_FINE] + c->prof_passes[CLS_GATHER_COARSE] +
                    c->prof_passes[CLS_SCATTER] + c->prof_passes[CLS_HS] - passes0;
    // relaxations per level from the device trace
    const int nt = std::min(h.ntrace, TRACE_CAP);
    std::vector<TraceRow> tr(nt);
    if (nt) {   // on the context's stream (include/ml.h: all work is enqueued there)
        cudaMemcpyAsync(tr.data(), c->trace, sizeof(TraceRow) * nt, cudaMemcpyDeviceToHost, c->st);
        cudaStreamSynchronize(c->st);
    }
    for (const TraceRow& r : tr) {
        rep->relax_per_level[std::min(std::max(r.level, 0), 31)]++;
        if (r.F_after > r.F_before + 1e-12 * std::fabs(r.F_before)) rep->status = ML_E_CONTRACT;
    }
    for (int l = 0; l < 32; ++l) rep->relaxations += rep->relax_per_level[l];
    rep->kernel_launches = c->launches - launches0;
    if (rep->status == 0 && !converged) rep->status = ML_E_NOT_CONVERGED;
    ml_status fin = cuda_fail(c, "ml_solve");
    if (fin != ML_OK) return fin;
    return (ml_status)rep->status;
}

ml_status ml_profile(ml_ctx* c, uint32_t class_mask) {
    if (!c) return ML_E_INVAL;
    cudaStreamSynchronize(c->st);
    c->prof_mask = class_mask;
    c->ev_used = 0;
    c->ev_cls.clear();
    for (int k = 0; k < 16; ++k) c->prof_passes[k] = 0;
    long long z[2][16] = {{0}};
    cudaMemcpyAsync(&c->ctl->cls[0][0], z, sizeof(z), cudaMemcpyHostToDevice, c->st);
    return cuda_fail(c, "ml_profile");
}

ml_status ml_profile_read(ml_ctx* c, double* ms, int64_t* passes, int64_t* nnz, int64_t* segs) {
    if (!c) return ML_E_INVAL;
    ml_status s = sync_ctl(c);
    if (s != ML_OK) return s;
    for (int k = 0; k < 16; ++k) {
        if (ms) ms[k] = 0.0;
        if (passes) passes[k] = c->prof_passes[k];
        if (nnz) nnz[k] = c->h.cls[0][k];
        if (segs) segs[k] = c->h.cls[1][k];
    }
    if (ms)
        for (size_t p = 0; p < c->ev_cls.size(); ++p) {
            float t = 0.f;
            if (cudaEventElapsedTime(&t, c->ev_pool[2 * p], c->ev_pool[2 * p + 1]) == cudaSuccess) ms[c->ev_cls[p]] += t;
        }
    return cuda_fail(c, "ml_profile_read");
}

// diagnostics: ns per phase of the persistent inner solver (block 0), accumulated since the last reset
// Batched replicas: cap the cooperative grids (k_inner, k_gather_small, k_margins_small,
// k_select_coop) at `blocks` CTAs, so that several contexts on their own streams run side by side on one GPU.
ml_status ml_set_engine(ml_ctx* c, uint32_t flags) {
    if (!c) return ML_E_INVAL;
    const bool want = (flags & 1u) != 0;
    if (want && c->mp_grid_all == 0) return ML_E_INVAL;   // (small m: the shared-memory passes; no merge-path plan)
    c->mp = want;
    c->P.dyn = (flags & 8u) ? 1 : 0;   // bit 3: dynamic unit claims in the large-m inner solver whatever the unit count
    if ((flags & (16u | 64u)) && !c->hv_built) {   // the heavy path's copy is built on first request (X is fixed)
        c->hv_built = true;
        if (c->big_inner && c->inner_fn_hv && c->X.csr_rowptr) {
            const ml_status hs = hv_build(c);
            if (hs != ML_OK) return hs;
        }
    }
    if ((flags & 16u) && !c->P.hv.on) return ML_E_INVAL;
    // bit 4: always; bit 6: by the free set's share of H; bit 5: never; none: the context's default (hv_build)
    c->P.hv.mode = (flags & 16u) ? 1 : (flags & 64u) ? 0 : (flags & 32u) ? 2 : c->hv_mode0;
    return ML_OK;
}

ml_status ml_heavy_info(ml_ctx* c, int64_t* info_host) {
    if (!c || !info_host) return ML_E_INVAL;
    const ml_status st = sync_ctl(c);
    if (st != ML_OK) return st;
    const HvPrm& hv = c->P.hv;
    info_host[0] = hv.on;
    info_host[1] = hv.on ? hv.nh : 0;
    info_host[2] = hv.on ? hv.nnzh : 0;
    info_host[3] = hv.on ? hv.nts : 0;
    info_host[4] = 0;
    info_host[5] = 0;
    info_host[6] = c->h.hv_relax;
    info_host[7] = hv.mode;
    return ML_OK;
}

ml_status ml_set_sm_share(ml_ctx* c, int blocks) {
    if (!c) return ML_E_INVAL;
    const int full = std::min(c->sms, IR_GMAX);
    if (blocks <= 0 || blocks > c->sms) blocks = c->sms;
    if (c->sm_inner && c->X.m > (int64_t)IR_RS * std::min(blocks, IR_GMAX)) {   // k_inner: at most IR_RS rows per block
        c->err = "ml_set_sm_share: too few blocks for m (at most 64 rows per block on the small-m path)";
        return ML_E_INVAL;
    }
    c->coop_cap = blocks;
    if (c->sm_inner || c->big_inner) c->inner_P = std::min(blocks, full);
    if (c->sm_scatter) c->scat_P = blocks * c->scat_bps;   // the API's cooperative scatter / gather
    if (c->sm_gather) c->gath_P = blocks * c->gath_bps;
    return ML_OK;
}

ml_status ml_inner_phases(ml_ctx* c, uint64_t* ns_host, int reset) {
    if (!c) return ML_E_INVAL;
    ml_status s = sync_ctl(c);
    if (s != ML_OK) return s;
    for (int k = 0; k < 16; ++k) if (ns_host) ns_host[k] = c->h.tph[k];
    if (reset) { unsigned long long z[16] = {0}; cudaMemcpyAsync(c->ctl->tph, z, sizeof(z), cudaMemcpyHostToDevice, c->st); }
    return cuda_fail(c, "ml_inner_phases");
}

// trace access for tests (not part of the paper's call set)
int64_t ml_trace(ml_ctx* c, void* rows_host, int64_t cap) {
    if (!c) return -1;
    if (sync_ctl(c) != ML_OK) return -1;
    const int nt = std::min(c->h.ntrace, TRACE_CAP);
    const int k = (int)std::min<int64_t>(nt, cap);
    if (rows_host && k) {
        cudaMemcpyAsync(rows_host, c->trace, sizeof(TraceRow) * k, cudaMemcpyDeviceToHost, c->st);
        cudaStreamSynchronize(c->st);
    }
    return nt;
}

}  // extern "C"

#ifdef IR_HVDBG
// (debug builds only) the heavy sweep alone on this context's S copy, in a kernel of its own: cycles vs k_inner's
__global__ void __launch_bounds__(256, 1) k_hv_sweep_alone(HvPrm hv) {
    double* s = reinterpret_cast<double*>(hv_dyn + HV_SH_OFF);
    for (int i = threadIdx.x; i < HV_HMAX; i += blockDim.x) s[i] = 0.001 * (i & 255);
    __syncthreads();
    hv_sweep(hv);
}
extern "C" double ml_debug_hv_sweep(ml_ctx* c, int reps, int nv) {
    if (!c || !c->P.hv.on) return -1.0;
    const size_t smem = hv_smem_bytes();
    cudaFuncSetAttribute(k_hv_sweep_alone, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0, c->st);
        (void)nv;
        k_hv_sweep_alone<<<c->inner_P, 256, smem, c->st>>>(c->P.hv);
        cudaEventRecord(e1, c->st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}
#endif
