// ml_heavy.cuh — the heavy-column path of the large-m inner solver: X_A s for the longest columns without atomics
// (A5; DESIGN section 8.2 "heavy columns").
//
// On the Zipf designs (cfg 3-5) a few thousand columns hold most of X's nonzeros (cfg 5: the 8192 longest columns
// hold 65 % of 2e8), and they are the columns of every free set.  Through the column units of k_inner their X_A s
// products are 64-bit reductions into global memory, bound by the REDG issue rate of the load/store units (~1.3 LSU
// cycles per lane, B300_MICROARCH.md: 0.8-0.9 nonzeros per SM clock).  Here the heavy set H (at most HV_HMAX
// columns, the longest, chosen once at ml_create) gets a row-major copy of its nonzeros (fp32 value + 16 bits holding
// 8 x the heavy id, the byte offset of s_H[id]; 6 bytes; every row padded to a whole number of 4-entry vectors with
// zero entries): the "S copy".  s_H (the inner direction on H, HV_HMAX doubles) is staged in shared memory, and each
// row's sum over its heavy entries is formed in registers and written once (Xh): no atomics.
// The copy is cut into warp chunks of whole rows (at most HV_WCH entries and HV_WROWS rows); every warp streams its
// own chunks through a private HV_WST-stage TMA ring (its lane 0 issues the bulk copies of the values, the ids and
// the chunk's slice of row starts) and reduces a chunk with groups of L = 2^lg lanes per row (lg per chunk from its
// row count: one round of 32 / L rows); no block barriers.  Each row is a fixed-order sum: bitwise reproducible.
// X_A z (the snap path's zeroing columns, z = s there: rare) and H sigma of the heavy columns stay on the column
// units (fixed-point reductions, L2 gathers of D o X sigma).
#pragma once
#include "ml_common.cuh"

namespace ml {

constexpr int HV_HMAX = 8192;              // heavy columns at most (s_H: 64 KB of shared memory)
#ifndef HV_WCH_V
#define HV_WCH_V 768
#endif
#ifndef HV_WST_V
#define HV_WST_V 2
#endif
constexpr int HV_WCH = HV_WCH_V;           // entries per warp chunk at most (build knobs: -DHV_WCH_V, -DHV_WST_V)
#ifndef HV_WROWS_V
#define HV_WROWS_V 32
#endif
constexpr int HV_WROWS = HV_WROWS_V;       // rows per warp chunk at most (one round of groups of 32 / 2^lg lanes)
constexpr int HV_WST = HV_WST_V;           // stages of a warp's ring
constexpr int HV_MINLEN = 32;              // shortest heavy column
constexpr long long HV_AUTO = 1LL << 26;   // the path is on by default when H holds this many nonzeros (ml.cu)
constexpr int HV_W = 8;                    // warps per block (k_inner)
// a stage: values (HV_WCH + 8 from a 16-byte boundary), ids, row starts (HV_WROWS + 1 from a 16-byte boundary)
constexpr size_t HV_WSTAGE = (((size_t)(HV_WCH + 8) * 6 + (size_t)(HV_WROWS + 8) * 4) + 15) / 16 * 16;
constexpr size_t HV_WRING = (size_t)HV_WST * HV_WSTAGE + 64 + (size_t)32 * HV_WST;   // + the stages' mbarriers (64 B)
                                                                                    // and chunk descriptors
// dynamic shared memory of the sub-phase (it aliases the column rings of k_inner)
constexpr size_t HV_SH_OFF = 0;                                            // s_H
constexpr size_t HV_SRING_OFF = (size_t)8 * HV_HMAX;                       // the warps' rings
static_assert(HV_SRING_OFF % 16 == 0 && HV_WSTAGE % 16 == 0 && HV_WRING % 16 == 0, "ring alignment");
__host__ __device__ constexpr size_t hv_smem_bytes() { return HV_SRING_OFF + (size_t)HV_W * HV_WRING; }

// a warp chunk: heavy entries [e0, e1) of rows [r0, r0 + nr) (their starts at soff[r0 .. r0 + nr]); L = 2^lg
struct HvChunk { int e0, e1, r0, nr, lg, pad0, pad1, pad2; };

// the heavy path's device state (Prm::hv)
struct HvPrm {
    int on;                 // built (m > SMALL_M, enough heavy nonzeros, rows of at most HV_WCH / 2 heavy entries)
    int nh;                 // |H|
    int nts;                // warp chunks
    int mode;               // 0: per relaxation (nnz(A ∩ H) >= frac nnz(H)), 1: always, 2: never (ml_set_engine)
    double frac;
    long long nnzh;         // nonzeros of H
    const int* hid;         // [n] heavy id of column j (by decreasing length), or -1
    const float* sval; const uint16_t* sidx;   // the S copy: values and heavy ids, row by row
    const int* soff;        // [m + 1] row starts in the S copy
    const HvChunk* schunk;  // [nts]
    double* sH;             // [HV_HMAX] the S coefficient of each heavy column of A this iteration (0 elsewhere)
    double* Xh;             // [m] X_H s_H
    int* zunits;            // [units] this iteration's units of the zeroing heavy columns (X_A z goes through them)
    int* phid;              // [n] heavy id of free-set position p this relaxation (-1: light)
};

// The dynamic shared memory of the calling kernel (every extern __shared__ array names the same base): s_H and the
// rings are addressed through it, so that the out-of-line hv_sweep still emits shared loads.
extern __shared__ __align__(16) unsigned char hv_dyn[];

// Rows of a staged chunk by groups of L = 2^LG lanes.  Lane gl takes the row's 4-entry vectors gl, gl + L, ... (one
// 16-byte load of values and one 8-byte load of ids per vector; the copy pads every row to whole vectors with zero
// entries, so no element is masked), two vectors at a time: loads, then the s_H gathers, then the fused multiply-adds
// in order; then the group's fixed shuffle tree; Xh[row].
// (ncu, cfg 5: the sweep is bound by shared-memory wavefronts.  With one 4-byte and one 2-byte load per entry the 16
// rows a warp reads together start at arbitrary offsets: 2.6 wavefronts per request of values and 2.7 of ids against
// 1, 182 M of the 324 M wavefronts of a launch; vectors need a quarter of the requests.)
static_assert(8 * HV_HMAX <= 65536, "8 * id must fit the copy's 16-bit ids");
__device__ __forceinline__ double hv_sh(const unsigned char* sb, uint32_t off8) {
    return *reinterpret_cast<const double*>(sb + (off8 & 0xfff8u));
}
template <int LG>
__device__ __forceinline__ void hv_rows(const float* sv, const uint16_t* si, const int* so, const HvChunk& ch, double* Xh) {
    constexpr int L = 1 << LG, NG = 32 >> LG;
    const int lane = threadIdx.x & 31, grp = lane >> LG, gl = lane & (L - 1);
    const int eb = ch.e0 & ~7, ob = ch.r0 & 3;
    const unsigned char* sb = hv_dyn + HV_SH_OFF;
    const float4* sv4 = reinterpret_cast<const float4*>(sv);
    const uint2* si4 = reinterpret_cast<const uint2*>(si);
    for (int r = grp; r - grp < ch.nr; r += NG) {   // (every lane runs every round: the shuffles need all lanes)
        double acc = 0.0, acc1 = 0.0;   // (one chain per vector of the pair)
        int b4 = 0, e4 = 0;   // the row's vectors [b4, e4): rows are padded to whole vectors (k_hv_rowcnt / k_hv_rowfill)
        if (r < ch.nr) { b4 = (so[ob + r] - eb) >> 2; e4 = (so[ob + r + 1] - eb) >> 2; }
        for (int v = b4 + gl; v < e4; v += 2 * L) {
            const bool in1 = v + L < e4;
            const float4 x0 = sv4[v];
            const uint2 i0 = si4[v];
            const float4 x1 = in1 ? sv4[v + L] : make_float4(0.f, 0.f, 0.f, 0.f);
            const uint2 i1 = in1 ? si4[v + L] : make_uint2(0u, 0u);
            // the copy stores 8 * id: a 16-bit half is the byte offset into s_H (any value stays inside its 64 KB)
            double g[8];
            g[0] = hv_sh(sb, i0.x & 0xffffu); g[1] = hv_sh(sb, i0.x >> 16);
            g[2] = hv_sh(sb, i0.y & 0xffffu); g[3] = hv_sh(sb, i0.y >> 16);
            g[4] = hv_sh(sb, i1.x & 0xffffu); g[5] = hv_sh(sb, i1.x >> 16);
            g[6] = hv_sh(sb, i1.y & 0xffffu); g[7] = hv_sh(sb, i1.y >> 16);
            acc = fma((double)x0.x, g[0], acc); acc = fma((double)x0.y, g[1], acc);
            acc = fma((double)x0.z, g[2], acc); acc = fma((double)x0.w, g[3], acc);
            acc1 = fma((double)x1.x, g[4], acc1); acc1 = fma((double)x1.y, g[5], acc1);
            acc1 = fma((double)x1.z, g[6], acc1); acc1 = fma((double)x1.w, g[7], acc1);
        }
        acc += acc1;
#pragma unroll
        for (int d = L >> 1; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
        if (gl == 0 && r < ch.nr) Xh[ch.r0 + r] = acc;
    }
}

// This warp's chunks (an equal share of all warps of the grid, in order) through its private ring.
// (out of line: called once per S phase, so that its loop gets registers of its own instead of k_inner's spills)
__device__ __noinline__ void hv_sweep(const HvPrm hv, unsigned long long* dbg = nullptr) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef IR_HVDBG
    const unsigned long long t_start = clock64();
#endif
    unsigned char* ring = hv_dyn + HV_SRING_OFF + (size_t)w * HV_WRING;   // (a shared address the compiler can see)
    uint64_t* bar = reinterpret_cast<uint64_t*>(ring + (size_t)HV_WST * HV_WSTAGE);
    const long long gw = (long long)blockIdx.x * HV_W + w, NW = (long long)gridDim.x * HV_W;
    const int c0 = (int)(hv.nts * gw / NW), c1 = (int)(hv.nts * (gw + 1) / NW);
    // A stage's chunk descriptor sits in shared memory next to the barriers: lane 0 writes it when it issues the
    // stage's copies, every lane reads it when the stage is consumed.  The descriptor of the chunk issued at the end
    // of an iteration is loaded at its start, so that no L2 round trip of a descriptor is left on the warp's critical
    // path (two per 768-entry chunk before: ~1400 of ~1900 cycles per chunk).
    HvChunk* dsc = reinterpret_cast<HvChunk*>(ring + (size_t)HV_WST * HV_WSTAGE + 64);
    auto issue = [&](const HvChunk& k, int st) {
        const int a0 = k.e0 & ~7, a1 = (k.e1 + 7) & ~7;
        const int o0 = k.r0 & ~3, o1 = (k.r0 + k.nr + 1 + 3) & ~3;
        unsigned char* b = ring + (size_t)st * HV_WSTAGE;
        const uint32_t n = (uint32_t)(a1 - a0), no = (uint32_t)(o1 - o0);
        dsc[st] = k;
        mbar_arrive_expect_tx(bar + st, 6u * n + 4u * no);
        bulk_g2s(b, hv.sval + a0, 4u * n, bar + st);
        bulk_g2s(b + (size_t)(HV_WCH + 8) * 4, hv.sidx + a0, 2u * n, bar + st);
        bulk_g2s(b + (size_t)(HV_WCH + 8) * 6, hv.soff + o0, 4u * no, bar + st);
    };
    if (lane == 0) {
        for (int k = 0; k < HV_WST; ++k) mbar_init(bar + k, 1);
        fence_mbar_init();
        for (int k = 0; k < HV_WST && c0 + k < c1; ++k) issue(hv.schunk[c0 + k], k);
    }
    __syncwarp();
    uint32_t phase = 0u;
    for (int c = c0, st = 0; c < c1; ++c, st = (st + 1) % HV_WST) {
        const bool more = c + HV_WST < c1;
        HvChunk nxt;
        if (more) nxt = hv.schunk[c + HV_WST];   // (every lane, one address: a broadcast load, used at the end)
        mbar_wait(bar + st, (phase >> st) & 1u);
        phase ^= 1u << st;
        const HvChunk ch = dsc[st];
        const unsigned char* b = ring + (size_t)st * HV_WSTAGE;
        const float* sv = reinterpret_cast<const float*>(b);
        const uint16_t* si = reinterpret_cast<const uint16_t*>(b + (size_t)(HV_WCH + 8) * 4);
        const int* so = reinterpret_cast<const int*>(b + (size_t)(HV_WCH + 8) * 6);
        switch (ch.lg) {
            case 0: hv_rows<0>(sv, si, so, ch, hv.Xh); break;
            case 1: hv_rows<1>(sv, si, so, ch, hv.Xh); break;
            case 2: hv_rows<2>(sv, si, so, ch, hv.Xh); break;
            case 3: hv_rows<3>(sv, si, so, ch, hv.Xh); break;
            case 4: hv_rows<4>(sv, si, so, ch, hv.Xh); break;
            default: hv_rows<5>(sv, si, so, ch, hv.Xh); break;
        }
        __syncwarp();   // stage st consumed by every lane (its descriptor too)
        if (lane == 0 && more) issue(nxt, st);
        __syncwarp();   // (the next descriptor of stage st is visible to every lane)
    }
    __syncwarp();
    if (lane == 0)
        for (int k = 0; k < HV_WST; ++k) mbar_inval(bar + k);
#ifdef IR_HVDBG   // (per-warp sweep cycles: sum, max, count; and the cycles from the first issue to the first stage)
    if (dbg && lane == 0) {
        const unsigned long long dt = clock64() - t_start;
        atomicAdd(dbg, dt);
        atomicMax(dbg + 1, dt);
        atomicAdd(dbg + 2, 1ull);
    }
#endif
    __syncwarp();
}

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
// heavy entries per row (cnt), their maximum
__global__ void k_hv_rowcnt(const int* rowptr, const int* col, int m, const int* hid, int* cnt, int* maxcnt) {
    int mx = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        int c = 0;
        for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) c += __ldg(hid + col[k]) >= 0;
        c = (c + 3) & ~3;   // rows are padded to whole 4-entry vectors (zero value, id 0): hv_rows needs no element masks
        cnt[i] = c;
        mx = max(mx, c);
    }
    mx = (int)__reduce_max_sync(0xffffffffu, (unsigned)mx);
    if ((threadIdx.x & 31) == 0) atomicMax(maxcnt, mx);
}
// warp chunks (built greedily on the host): whole rows, at most HV_WCH heavy entries and HV_WROWS rows
__host__ __device__ __forceinline__ int hv_lg(int rows) {   // groups of L = 32 / (rows rounded up to 2^k) lanes
    int lg = 5;
    while (lg > 0 && (32 >> lg) < rows) --lg;
    return lg;
}
// the S copy's entries of each row, rotated by a hash of the row: the rows' entries are in column order, so the
// heaviest columns would otherwise sit at the same place in every row and the s_H gathers of the rows a warp reads
// together would hit the same shared-memory banks
__global__ void k_hv_rowfill(const int* rowptr, const int* col, const float* val, int m, const int* hid, const int* hrp,
                             float* sval, uint16_t* sidx) {
    // Placement inside a row (any order is valid: a row's sum is over all its entries).  hv_rows gathers s_H[id] for 16
    // lanes per shared-memory phase: with the usual 16 rows per round (L = 2), lane gl of row r reads position
    // p = 4 gl + t (+ 8 for the second vector of a pair, + 16 per iteration).  The gathers of a phase fall into 16
    // distinct 8-byte banks when id mod 16 = rho(p, r) below, so each entry is placed at a position that wants its
    // residue as long as the row has one (ncu: 2.3 wavefronts per gather request with hashed rotations); rows of more
    // than HV_PLACE entries keep the rotation.
    constexpr int HV_PLACE = 192;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const int o = hrp[i], L = hrp[i + 1] - o;   // (L: the padded length, a multiple of 4)
        if (L == 0) continue;
        if (L > HV_PLACE) {
            int q = (int)(((unsigned)i * 2654435761u) >> 8) % L, placed = 0;
            for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) {
                const int h = __ldg(hid + col[k]);
                if (h >= 0) {
                    sval[o + q] = val[k];
                    sidx[o + q] = (uint16_t)(8 * h);   // (the byte offset of s_H[h])
                    q = q + 1 == L ? 0 : q + 1;
                    ++placed;
                }
            }
            for (; placed < L; ++placed) {   // the padding: zero entries of heavy column 0
                sval[o + q] = 0.0f;
                sidx[o + q] = 0;
                q = q + 1 == L ? 0 : q + 1;
            }
            continue;
        }
        float ev[HV_PLACE];      // the row's heavy entries, then sorted by residue
        uint16_t eh[HV_PLACE];
        float bv[HV_PLACE];
        uint16_t bh[HV_PLACE];
        int cnt[17];
        for (int r = 0; r < 17; ++r) cnt[r] = 0;
        int c = 0;
        for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) {
            const int h = __ldg(hid + col[k]);
            if (h >= 0) { ev[c] = val[k]; eh[c] = (uint16_t)h; cnt[(h & 15) + 1] += 1; ++c; }
        }
        for (int r = 0; r < 16; ++r) cnt[r + 1] += cnt[r];   // bucket starts
        int fill[16], head[16];
        for (int r = 0; r < 16; ++r) { fill[r] = cnt[r]; head[r] = cnt[r]; }
        for (int e = 0; e < c; ++e) { const int r = eh[e] & 15; bv[fill[r]] = ev[e]; bh[fill[r]] = eh[e]; fill[r] += 1; }
        // positions that find an entry of the residue they want
        const int rr = i & 7;
        for (int p2 = 0; p2 < L; ++p2) {
            const int want = 8 * ((p2 >> 2) & 1) + ((rr + p2 + 4 * ((p2 >> 3) & 1)) & 7);
            if (head[want] < cnt[want + 1]) {
                sval[o + p2] = bv[head[want]];
                sidx[o + p2] = (uint16_t)(8 * bh[head[want]]);
                head[want] += 1;
            } else sidx[o + p2] = 0xffffu;   // (free: filled below)
        }
        // the entries left over, in bucket order, into the free positions; then the padding (zero entries of column 0)
        int r = 0;
        for (int p2 = 0; p2 < L; ++p2) {
            if (sidx[o + p2] != 0xffffu) continue;
            while (r < 16 && head[r] >= cnt[r + 1]) ++r;
            if (r < 16) {
                sval[o + p2] = bv[head[r]];
                sidx[o + p2] = (uint16_t)(8 * bh[head[r]]);
                head[r] += 1;
            } else { sval[o + p2] = 0.0f; sidx[o + p2] = 0; }
        }
    }
}

}  // namespace ml
