// taylor.cu -- K4, the fused Taylor-order kernels (own translation unit, see taylor.cuh).
#include "taylor.cuh"

#include <algorithm>

#include "primitives.cuh"

namespace pb {

// ================================================================================================
// K4  fused Taylor order:  hterm = H term ; term' = (0,-dt/n) hterm ; c += term' ; |term'|^2, |c|^2
//     (csr_matvec, subspace.hpp:35-43 + propagator.hpp:68-84; arithmetic recipe SURVEY App. C.1)
// ================================================================================================

// Paired orders.  The reference's loop body (SINGLE: c += term, both norms, stop rule) moves c through HBM once per
// order.  The series can only stop at order k if order k-1 already satisfied `tn <= rtol*rn`, so when it did not
// (streak == 0) nobody needs c_k or |c_k| before order k+1 has run:
//   DEFER   (order k)   only term_k = b H term_{k-1} and |term_k|^2; c is neither read nor written.
//   CATCHUP (order k+1) c = (c + term_k) + term_{k+1} in the reference's order of additions, |c_k|^2 and |c_{k+1}|^2
//                       from the two intermediate values, then the stop rule for k and for k+1.
// Same operations on the same operands and the same reduction shapes as SINGLE, hence bit-identical results; a
// deferred order moves 12z + 40n bytes instead of 12z + 72n (term_k[i] is the diagonal entry of row i's gather in
// the catch-up launch, so that read costs no extra DRAM traffic).  The three modes are separate kernels (each row
// loop keeps its 32 registers = 8 resident CTAs per SM, which this latency-bound traversal needs); the host issues
// DEFER/CATCHUP pairs, and a DEFER launch that finds streak != 0 does nothing but raise `bail`: every later launch
// returns at once and the host resumes from that order with SINGLE launches.

/// Control-block flag read at kernel entry through L1 (ld.global.ca).  Every thread of the grid reads the same word:
/// as volatile (L2-coherent) loads those ~1e4 warp requests serialise on one L2 slice and cost ~3 us per launch and
/// flag; through L1 one request per SM reaches L2.  Safe: the flags are written by EARLIER launches (L1 is invalidated
/// at kernel boundaries) or, in this launch, only after every CTA has read them.
__device__ __forceinline__ int ld_flag(const int* p) {
    int v;
    asm volatile("ld.global.ca.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

/// One application of the stop rule (propagator.hpp:76-84) by the last CTA's thread 0.
__device__ __forceinline__ void taylor_apply_rule(TaylorCtl* ctl, int order, double tn2, double rn2, double rtol) {
    const double tn = __dsqrt_rn(tn2), rn = __dsqrt_rn(rn2);
    if (order > ctl->order_used) ctl->order_used = order;
    ctl->last_order = order;
    ctl->last_term_norm = tn;
    ctl->last_c_norm = rn;
    const int streak = (tn <= __dmul_rn(rtol, rn)) ? ctl->streak + 1 : 0;
    ctl->streak = streak;
    if (streak >= 2) ctl->done = 1;
}

/// SINGLE.  EXPECT: the launch of the FIRST order also produces what csr_expectation (subspace.hpp:46-55),
/// state_norm and expmv's finiteness check (propagator.hpp:55-57) need from the input vector x = term_in -- the row
/// sums (H x)_i are the very ones the first order computes -- so the resident step needs no separate <x|H|x> pass:
/// expect_out[0] = sum_i Re(conj(x_i) (H x)_i), [1] = sum |x_i|^2, [2] = #non-finite coefficients.
template <bool EXPECT>
__global__ void __launch_bounds__(NT, EXPECT ? 6 : 8) taylor_order_kernel_t(uint32_t n, const uint32_t* __restrict__ row_ptr,
                                                            const int32_t* __restrict__ col,
                                                            const double* __restrict__ val,
                                                            const double2* __restrict__ term_in,
                                                            double2* __restrict__ term_out, double2* __restrict__ c,
                                                            double b, int order, double rtol,
                                                            double* __restrict__ partials, TaylorCtl* ctl,
                                                            int ignore_stop, double* __restrict__ tot_out,
                                                            double* __restrict__ expect_out) {
    constexpr int K = EXPECT ? 5 : 2;
    __shared__ double smem[NT / 32];
    if (!ignore_stop && (ld_flag(&ctl->done) | ld_flag(&ctl->bail))) return;
    double acc[K];
#pragma unroll
    for (int j = 0; j < K; ++j) acc[j] = 0.0;
    // PRE: the next row's extent is requested while this row's entries are gathered (one dependent DRAM latency
    // less per row); it costs two registers, which the SINGLE variant does not have at 32
    constexpr bool PRE = EXPECT;
    uint32_t i = blockIdx.x * NT + threadIdx.x;
    uint32_t kb_next = 0, ke_next = 0;
    if (PRE && i < n) {
        kb_next = __ldg(row_ptr + i);
        ke_next = __ldg(row_ptr + i + 1);
    }
    for (; i < n; i += gridDim.x * NT) {
        uint32_t kb, ke;
        if (PRE) {
            kb = kb_next;
            ke = ke_next;
            const uint32_t inext = i + gridDim.x * NT;
            if (inext < n) {
                kb_next = __ldg(row_ptr + inext);
                ke_next = __ldg(row_ptr + inext + 1);
            }
        } else {
            kb = __ldg(row_ptr + i);
            ke = __ldg(row_ptr + i + 1);
        }
        double ar = 0.0, ai = 0.0;
        for (uint32_t k = kb; k < ke; ++k) {
            const double v = __ldg(val + k);
            const double2 x = __ldg(term_in + __ldg(col + k));
            ar = __dadd_rn(ar, __dmul_rn(v, x.x));
            ai = __dadd_rn(ai, __dmul_rn(v, x.y));
        }
        if (EXPECT) {
            const double2 xi = __ldg(term_in + i);
            // real(conj(x) * row) = xr*rr - (-xi)*ri
            acc[2] = __dadd_rn(acc[2], __dsub_rn(__dmul_rn(xi.x, ar), __dmul_rn(-xi.y, ai)));
            acc[3] = __dadd_rn(acc[3], __dadd_rn(__dmul_rn(xi.x, xi.x), __dmul_rn(xi.y, xi.y)));
            if (!isfinite(xi.x) || !isfinite(xi.y)) acc[4] = acc[4] + 1.0;
        }
        // (0, b) * (ar, ai) exactly as the compiler expands std::complex multiplication
        const double tr = __dsub_rn(__dmul_rn(0.0, ar), __dmul_rn(b, ai));
        const double ti = __dadd_rn(__dmul_rn(0.0, ai), __dmul_rn(b, ar));
        double2 cc = c[i];
        cc.x = __dadd_rn(cc.x, tr);
        cc.y = __dadd_rn(cc.y, ti);
        term_out[i] = make_double2(tr, ti);
        c[i] = cc;
        acc[0] = __dadd_rn(acc[0], __dadd_rn(__dmul_rn(tr, tr), __dmul_rn(ti, ti)));
        acc[1] = __dadd_rn(acc[1], __dadd_rn(__dmul_rn(cc.x, cc.x), __dmul_rn(cc.y, cc.y)));
    }
    double tot[K];
    if (grid_sum<K>(acc, partials, &ctl->ticket, tot, smem) && threadIdx.x == 0) {
        if (EXPECT) {
            expect_out[0] = tot[2];
            expect_out[1] = tot[3];
            expect_out[2] = tot[4];
        }
        if (tot_out) {  // sharded: the sums are all-reduced first, taylor_stop_kernel applies the rule
            tot_out[0] = tot[0];
            tot_out[1] = tot[1];
            return;
        }
        taylor_apply_rule(ctl, order, tot[0], tot[1], rtol);
        __threadfence();
    }
}

/// DEFER: term_out = b H term_in and |term_out|^2 only.
__global__ void __launch_bounds__(NT, 8) taylor_defer_kernel(uint32_t n, const uint32_t* __restrict__ row_ptr,
                                                          const int32_t* __restrict__ col,
                                                          const double* __restrict__ val,
                                                          const double2* __restrict__ term_in,
                                                          double2* __restrict__ term_out, double b, int order,
                                                          double* __restrict__ partials, TaylorCtl* ctl) {
    __shared__ double smem[NT / 32];
    if (ld_flag(&ctl->done) | ld_flag(&ctl->bail)) return;
    // the control block is only rewritten by the last CTA of a launch, after every CTA has passed this point (the bail
    // write below only adds a second reason to return for the CTAs that see it)
    if (ld_flag(&ctl->streak) != 0) {  // the series may stop at this order: it has to run SINGLE
        if (blockIdx.x == 0 && threadIdx.x == 0) *(volatile int*)&ctl->bail = order;
        return;
    }
    double acc[1] = {0.0};
    // PRE: the next row's extent is requested while this row's entries are gathered (one dependent DRAM latency
    // less per row); it costs two registers, which the SINGLE variant does not have at 32
    constexpr bool PRE = true;
    uint32_t i = blockIdx.x * NT + threadIdx.x;
    uint32_t kb_next = 0, ke_next = 0;
    if (PRE && i < n) {
        kb_next = __ldg(row_ptr + i);
        ke_next = __ldg(row_ptr + i + 1);
    }
    for (; i < n; i += gridDim.x * NT) {
        uint32_t kb, ke;
        if (PRE) {
            kb = kb_next;
            ke = ke_next;
            const uint32_t inext = i + gridDim.x * NT;
            if (inext < n) {
                kb_next = __ldg(row_ptr + inext);
                ke_next = __ldg(row_ptr + inext + 1);
            }
        } else {
            kb = __ldg(row_ptr + i);
            ke = __ldg(row_ptr + i + 1);
        }
        double ar = 0.0, ai = 0.0;
        for (uint32_t k = kb; k < ke; ++k) {
            const double v = __ldg(val + k);
            const double2 x = __ldg(term_in + __ldg(col + k));
            ar = __dadd_rn(ar, __dmul_rn(v, x.x));
            ai = __dadd_rn(ai, __dmul_rn(v, x.y));
        }
        const double tr = __dsub_rn(__dmul_rn(0.0, ar), __dmul_rn(b, ai));
        const double ti = __dadd_rn(__dmul_rn(0.0, ai), __dmul_rn(b, ar));
        term_out[i] = make_double2(tr, ti);
        acc[0] = __dadd_rn(acc[0], __dadd_rn(__dmul_rn(tr, tr), __dmul_rn(ti, ti)));
    }
    double tot[1];
    if (grid_sum<1>(acc, partials, &ctl->ticket, tot, smem) && threadIdx.x == 0) {
        ctl->pending = 1;
        ctl->pending_tn2 = tot[0];
        ctl->deferred += 1;
        if (order > ctl->order_used) ctl->order_used = order;
        ctl->last_order = order;
        __threadfence();
    }
}

/// CATCHUP: the order after a deferred one (term_in = the deferred order's term).
/// 40 registers (6 resident CTAs per SM; the host sizes the grid to one wave): capping it at 32 spills the three
/// accumulators to local memory and is slower (0.969 vs 0.958 ms of expmv per step on config 2).
__global__ void __launch_bounds__(NT, 6) taylor_catchup_kernel(uint32_t n, const uint32_t* __restrict__ row_ptr,
                                                            const int32_t* __restrict__ col,
                                                            const double* __restrict__ val,
                                                            const double2* __restrict__ term_in,
                                                            double2* __restrict__ term_out, double2* __restrict__ c,
                                                            double b, int order, double rtol,
                                                            double* __restrict__ partials, TaylorCtl* ctl) {
    __shared__ double smem[NT / 32];
    if (ld_flag(&ctl->done) | ld_flag(&ctl->bail)) return;
    double acc[3] = {0.0, 0.0, 0.0};
    // PRE: the next row's extent is requested while this row's entries are gathered (one dependent DRAM latency
    // less per row); it costs two registers, which the SINGLE variant does not have at 32
    constexpr bool PRE = true;
    uint32_t i = blockIdx.x * NT + threadIdx.x;
    uint32_t kb_next = 0, ke_next = 0;
    if (PRE && i < n) {
        kb_next = __ldg(row_ptr + i);
        ke_next = __ldg(row_ptr + i + 1);
    }
    for (; i < n; i += gridDim.x * NT) {
        uint32_t kb, ke;
        if (PRE) {
            kb = kb_next;
            ke = ke_next;
            const uint32_t inext = i + gridDim.x * NT;
            if (inext < n) {
                kb_next = __ldg(row_ptr + inext);
                ke_next = __ldg(row_ptr + inext + 1);
            }
        } else {
            kb = __ldg(row_ptr + i);
            ke = __ldg(row_ptr + i + 1);
        }
        double ar = 0.0, ai = 0.0;
        for (uint32_t k = kb; k < ke; ++k) {
            const double v = __ldg(val + k);
            const double2 x = __ldg(term_in + __ldg(col + k));
            ar = __dadd_rn(ar, __dmul_rn(v, x.x));
            ai = __dadd_rn(ai, __dmul_rn(v, x.y));
        }
        const double tr = __dsub_rn(__dmul_rn(0.0, ar), __dmul_rn(b, ai));
        const double ti = __dadd_rn(__dmul_rn(0.0, ai), __dmul_rn(b, ar));
        term_out[i] = make_double2(tr, ti);
        acc[0] = __dadd_rn(acc[0], __dadd_rn(__dmul_rn(tr, tr), __dmul_rn(ti, ti)));
        double2 cc = c[i];
        const double2 tp = __ldg(term_in + i);
        cc.x = __dadd_rn(cc.x, tp.x);
        cc.y = __dadd_rn(cc.y, tp.y);
        acc[2] = __dadd_rn(acc[2], __dadd_rn(__dmul_rn(cc.x, cc.x), __dmul_rn(cc.y, cc.y)));
        cc.x = __dadd_rn(cc.x, tr);
        cc.y = __dadd_rn(cc.y, ti);
        c[i] = cc;
        acc[1] = __dadd_rn(acc[1], __dadd_rn(__dmul_rn(cc.x, cc.x), __dmul_rn(cc.y, cc.y)));
    }
    double tot[3];
    if (grid_sum<3>(acc, partials, &ctl->ticket, tot, smem) && threadIdx.x == 0) {
        taylor_apply_rule(ctl, order - 1, ctl->pending_tn2, tot[2], rtol);  // streak was 0: cannot stop here
        taylor_apply_rule(ctl, order, tot[0], tot[1], rtol);
        ctl->pending = 0;
        __threadfence();
    }
}


// ------------------------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------------------------
template <class K>
static int resident_ctas(K kernel, int fallback) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, NT, 0) != cudaSuccess || per_sm < 1) per_sm = fallback;
    return per_sm;
}

void taylor_launch_single(bool expect, int grid, int sm_count, cudaStream_t stream, uint32_t n, const uint32_t* row_ptr,
                          const int32_t* col, const double* val, const double2* term_in, double2* term_out, double2* c,
                          double b, int order, double rtol, double* partials, TaylorCtl* ctl, int ignore_stop,
                          double* tot_out, double* expect_out) {
    if (expect) {
        // this variant needs more registers: size its grid to what is resident so the launch is a single wave
        static const int per_sm = resident_ctas(taylor_order_kernel_t<true>, 4);
        taylor_order_kernel_t<true><<<std::min(grid, sm_count * per_sm), NT, 0, stream>>>(
            n, row_ptr, col, val, term_in, term_out, c, b, order, rtol, partials, ctl, ignore_stop, tot_out, expect_out);
    } else {
        taylor_order_kernel_t<false><<<grid, NT, 0, stream>>>(n, row_ptr, col, val, term_in, term_out, c, b, order, rtol,
                                                              partials, ctl, ignore_stop, tot_out, expect_out);
    }
}

void taylor_launch_defer(int grid, cudaStream_t stream, uint32_t n, const uint32_t* row_ptr, const int32_t* col,
                         const double* val, const double2* term_in, double2* term_out, double b, int order,
                         double* partials, TaylorCtl* ctl) {
    taylor_defer_kernel<<<grid, NT, 0, stream>>>(n, row_ptr, col, val, term_in, term_out, b, order, partials, ctl);
}

void taylor_launch_catchup(int grid, int sm_count, cudaStream_t stream, uint32_t n, const uint32_t* row_ptr,
                           const int32_t* col, const double* val, const double2* term_in, double2* term_out, double2* c,
                           double b, int order, double rtol, double* partials, TaylorCtl* ctl) {
    static const int per_sm = resident_ctas(taylor_catchup_kernel, 4);
    taylor_catchup_kernel<<<std::min(grid, sm_count * per_sm), NT, 0, stream>>>(n, row_ptr, col, val, term_in, term_out,
                                                                               c, b, order, rtol, partials, ctl);
}

}  // namespace pb
