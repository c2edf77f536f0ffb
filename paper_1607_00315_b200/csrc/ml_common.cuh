// ml_common.cuh — device helpers for libml (sm_100a).
//
// Reductions are fixed-shape trees (warp shuffles -> shared memory -> one "last block" that sums the per-block
// partials in block order), so every floating-point result is bitwise reproducible for a given launch shape.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef ML_NT
#define ML_NT 256          // threads per block for every kernel
#endif
#define ML_NW (ML_NT / 32)
#define ML_MAXLS 40        // line-search trials evaluated (Eq. 4 backtracking, DESIGN Q7)

namespace ml {

// ------------------------------------------------------------------ loads
// Streaming loads of X (values / indices): read-only path, no L1 allocation.
__device__ __forceinline__ int4 ld_stream_i4(const int* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ float4 ld_stream_f4(const float* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
// L2-coherent load (bypasses L1) for data written by other blocks of the same launch.
template <class T> __device__ __forceinline__ T ld_cg(const T* p) { return __ldcg(p); }

// ------------------------------------------------------------------ warp / group reductions
template <int G> __device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum(double v) { return group_sum<32>(v); }
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------------ block + grid reductions
// A reduction payload: NS sums, NM maxima (non-negative values), NN minima.
template <int NS, int NM = 0, int NN = 0> struct Red {
    double s[NS > 0 ? NS : 1];
    double mx[NM > 0 ? NM : 1];
    double mn[NN > 0 ? NN : 1];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int k = 0; k < NS; ++k) s[k] = 0.0;
#pragma unroll
        for (int k = 0; k < NM; ++k) mx[k] = 0.0;
#pragma unroll
        for (int k = 0; k < NN; ++k) mn[k] = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    }
    static constexpr int NV = NS + NM + NN;
};

// Block-wide reduction; every thread returns with the block totals.  smem: NV * ML_NW doubles + NV.
template <int NS, int NM, int NN>
__device__ __forceinline__ void block_reduce(Red<NS, NM, NN>& r, double* sm) {
    constexpr int NV = Red<NS, NM, NN>::NV;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NS; ++k) { double v = warp_sum(r.s[k]); if (lane == 0) sm[k * ML_NW + wid] = v; }
#pragma unroll
    for (int k = 0; k < NM; ++k) { double v = warp_max(r.mx[k]); if (lane == 0) sm[(NS + k) * ML_NW + wid] = v; }
#pragma unroll
    for (int k = 0; k < NN; ++k) { double v = warp_min(r.mn[k]); if (lane == 0) sm[(NS + NM + k) * ML_NW + wid] = v; }
    __syncthreads();
    if (wid == 0) {
        for (int k = 0; k < NV; ++k) {
            double v = (lane < ML_NW) ? sm[k * ML_NW + lane] : (k < NS ? 0.0 : (k < NS + NM ? 0.0 : __longlong_as_double(0x7ff0000000000000LL)));
            if (k < NS) v = warp_sum(v);
            else if (k < NS + NM) v = warp_max(v);
            else v = warp_min(v);
            if (lane == 0) sm[NV * ML_NW + k] = v;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NS; ++k) r.s[k] = sm[NV * ML_NW + k];
#pragma unroll
    for (int k = 0; k < NM; ++k) r.mx[k] = sm[NV * ML_NW + NS + k];
#pragma unroll
    for (int k = 0; k < NN; ++k) r.mn[k] = sm[NV * ML_NW + NS + NM + k];
    __syncthreads();
}

// Grid-wide reduction through per-block partials and the last-arriving block.  Returns true in exactly one
// block (the last to arrive); there every thread holds the grid totals.  The last block sums the partials in
// block-index order with a fixed thread assignment, so the result does not depend on arrival order.
// part: gridDim.x * NV doubles; ctr: a zeroed counter (reset here for the next launch).
template <int NS, int NM, int NN>
__device__ bool grid_reduce(Red<NS, NM, NN>& r, double* part, unsigned* ctr, double* sm) {
    constexpr int NV = Red<NS, NM, NN>::NV;
    __shared__ bool s_last;
    block_reduce(r, sm);
    if (threadIdx.x == 0) {
        double* pb = part + (size_t)blockIdx.x * NV;
#pragma unroll
        for (int k = 0; k < NS; ++k) pb[k] = r.s[k];
#pragma unroll
        for (int k = 0; k < NM; ++k) pb[NS + k] = r.mx[k];
#pragma unroll
        for (int k = 0; k < NN; ++k) pb[NS + NM + k] = r.mn[k];
        __threadfence();
        unsigned prev = atomicAdd(ctr, 1u);
        s_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    r.zero();
    for (unsigned b = threadIdx.x; b < gridDim.x; b += ML_NT) {
        const double* pb = part + (size_t)b * NV;
#pragma unroll
        for (int k = 0; k < NS; ++k) r.s[k] += ld_cg(pb + k);
#pragma unroll
        for (int k = 0; k < NM; ++k) r.mx[k] = fmax(r.mx[k], ld_cg(pb + NS + k));
#pragma unroll
        for (int k = 0; k < NN; ++k) r.mn[k] = fmin(r.mn[k], ld_cg(pb + NS + NM + k));
    }
    block_reduce(r, sm);
    if (threadIdx.x == 0) *ctr = 0u;
    return true;
}

// ------------------------------------------------------------------ per-sample logistic quantities
// t = y z; e = exp(-|t|); ell = log(1+e^{-t}) = max(-t,0) + log1p(e); q = tau(-t); D = tau(t) tau(-t) = e/(1+e)^2;
// r = (tau(t) - 1) y = -y q   (stable forms SURVEY App. A.5)
struct RowState { double r, D, ell; };
__device__ __forceinline__ RowState row_state(double z, double y) {
    double t = y * z;
    double e = exp(-fabs(t));
    double ope = 1.0 + e;
    RowState s;
    s.ell = (t < 0.0 ? -t : 0.0) + log1p(e);
    double q = (t <= 0.0) ? 1.0 / ope : e / ope;
    s.r = -y * q;
    s.D = e / (ope * ope);
    return s;
}
__device__ __forceinline__ double logloss(double t) { return (t < 0.0 ? -t : 0.0) + log1p(exp(-fabs(t))); }
__device__ __forceinline__ double tau_neg(double t) {   // tau(-t)
    double e = exp(-fabs(t));
    return (t <= 0.0) ? 1.0 / (1.0 + e) : e / (1.0 + e);
}
// ell(t + delta) - ell(t), term-by-term difference (DESIGN Q26)
__device__ __forceinline__ double dloss(double t, double delta) {
    if (fabs(delta) <= 1.0) return log1p(tau_neg(t) * expm1(-delta));
    return logloss(t + delta) - logloss(t);
}
// The sample loss of either instance of Eq. 1: logistic with labels y, or squared with targets b (the
// LASSO of Eq. 2 with H = X^T X, g = -X^T b: ell_i = (z_i - b_i)^2 / 2, r_i = z_i - b_i, D_i = 1); b = nullptr selects
// the logistic loss.  Multiplying by y = +-1 is exact, so the logistic values are bitwise those of row_state / dloss
// with t = y z and delta = y dz.
__device__ __forceinline__ RowState row_state_i(const int8_t* y, const double* b, int i, double z) {
    if (b) { const double r = z - b[i]; return RowState{r, 1.0, 0.5 * r * r}; }
    return row_state(z, (double)y[i]);
}
__device__ __forceinline__ double dloss_i(const int8_t* y, const double* b, int i, double z, double dz) {   // ell_i(z + dz) - ell_i(z)
    if (b) { const double r = z - b[i]; return dz * (r + 0.5 * dz); }
    const double yy = (double)y[i];
    return dloss(yy * z, yy * dz);
}
__device__ __forceinline__ double soft(double t, double a) {   // Eq. 6
    double s = fabs(t) - a;
    if (s <= 0.0) return 0.0;
    return t > 0.0 ? s : -s;
}
__device__ __forceinline__ double sgn(double x) { return x > 0.0 ? 1.0 : -1.0; }

// non-negative double max via the int64 bit pattern (order-preserving for x >= 0)
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// ------------------------------------------------------------------ TMA bulk copies + mbarriers (sm_90+ / sm_100a)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
    asm volatile("mbarrier.inval.shared.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// fire-and-forget fp64 reduction to global memory (RED, not a generic-address ATOM)
__device__ __forceinline__ void red_add_global(double* p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "d"(v) : "memory");
}
// fixed-point reduction: v rounded to the nearest multiple of 1 / q, added as a 64-bit integer.  Integer addition is
// associative, so the sum does not depend on the order of the reductions (bitwise reproducible)
__device__ __forceinline__ void red_add_fixed(double* p, double v, double q) {
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "l"((unsigned long long)__double2ll_rn(v * q))
                 : "memory");
}
__device__ __forceinline__ double ld_fixed(const double* p, double qi) {
    return (double)(long long)__ldcg(reinterpret_cast<const unsigned long long*>(p)) * qi;
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy (TMA, 1-D): bytes multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

}  // namespace ml
