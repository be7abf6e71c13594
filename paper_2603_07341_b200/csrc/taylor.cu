// taylor.cu -- K4, the fused Taylor-order kernels (own translation unit, see taylor.cuh).
#include "taylor.cuh"

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>

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
                                                            double* __restrict__ expect_out, int first_from_x) {
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
        double2 cc;
        if (EXPECT) {
            const double2 xi = __ldg(term_in + i);
            cc = xi;  // first_from_x: the state is only in term_in so far (c is written, not read)
            // real(conj(x) * row) = xr*rr - (-xi)*ri
            acc[2] = __dadd_rn(acc[2], __dsub_rn(__dmul_rn(xi.x, ar), __dmul_rn(-xi.y, ai)));
            acc[3] = __dadd_rn(acc[3], __dadd_rn(__dmul_rn(xi.x, xi.x), __dmul_rn(xi.y, xi.y)));
            if (!isfinite(xi.x) || !isfinite(xi.y)) acc[4] = acc[4] + 1.0;
        }
        // (0, b) * (ar, ai) exactly as the compiler expands std::complex multiplication
        const double tr = __dsub_rn(__dmul_rn(0.0, ar), __dmul_rn(b, ai));
        const double ti = __dadd_rn(__dmul_rn(0.0, ai), __dmul_rn(b, ar));
        if (!(EXPECT && first_from_x)) cc = c[i];
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



// ================================================================================================
// K4, tile form (sm_100: bulk-copy pipeline).  The row kernels above make every thread walk a chain of dependent global
// loads -- row_ptr -> col/val -> x, and the x of entry k+1 only after the multiply-add of entry k -- about 5 exposed
// DRAM latencies per row, and fetch col/val with 32 scattered 4/8-byte requests per warp instruction (the L1 wavefront
// pipe is their co-bottleneck).  Here a CTA takes TR consecutive rows per tile.  What is CONTIGUOUS for a tile -- its
// row_ptr slice and its run of col and val -- is fetched by a producer warp with 1-D bulk copies (cp.async.bulk,
// completion on an mbarrier with expect_tx) into a shared-memory ring, a few tiles ahead.  A consumer thread still owns
// one row, but reads its extent, columns and values from shared memory, so it can issue ALL x gathers of the row back to
// back (they are the only scattered global loads left) and then add the products in ascending column order: ONE exposed
// latency per row, the same multiplies and additions in the same order as the row kernels and the reference
// (csr_matvec, subspace.hpp:35-43), hence bit-identical coefficients.  Consumer warps never meet at a CTA barrier: a
// warp releases a stage with one mbarrier arrive.  Every mode runs on the same persistent grid, so SINGLE / DEFER /
// CATCHUP / FIRST share one reduction shape.
// ================================================================================================
/// Alternating sweep of the tile kernels (see taylor_tile_kernel): pays when the gathered vector fits the L2 -- C2, 53 MB:
/// expmv -2.2 % -- and costs when it does not (3e7 rows, 480 MB: +2.2 %, a downward sweep is the slower direction
/// for DRAM), so it is used for vectors up to the L2 size.  PB200_TAYLOR_ONE_WAY=1: never (A/B measurements).
static const bool g_alternate = std::getenv("PB200_TAYLOR_ONE_WAY") == nullptr;
static int sweep_reverse(uint32_t n, int order) {
    static const size_t l2_bytes = [] {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev) != cudaSuccess)
            cudaGetLastError();
        return size_t(v > 0 ? v : 0);
    }();
    return (g_alternate && size_t(n) * 16 <= l2_bytes) ? (order & 1) : 0;
}

namespace tile {

#ifndef TILE_TR
#define TILE_TR 256
#endif
#ifndef TILE_STAGES
#define TILE_STAGES 2
#endif
#ifndef TILE_MINB
#define TILE_MINB 1
#endif
#ifndef TILE_EVICT_FIRST
#define TILE_EVICT_FIRST 1  // the matrix streams through once per launch: evict-first in L2 (C4 expmv -1.4 %, C2 +-0)
#endif
#ifndef TILE_STAGES_CODED
#define TILE_STAGES_CODED 3
#endif
constexpr int TR = TILE_TR;        // rows per tile = consumer threads per CTA
constexpr int NTHREADS = TR + 32;  // + one producer warp
/// Ring depth: a stage of the coded form is about half the size, so it affords one more.
template <bool CODED>
__host__ __device__ constexpr int stages() {
    return CODED ? TILE_STAGES_CODED : TILE_STAGES;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    do {  // try_wait suspends the thread in hardware for a bounded time; loop until the phase has completed
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!ok);
}
/// 1-D bulk copy global -> shared; src, dst and bytes are multiples of 16.  The matrix streams through once per
/// launch: with TILE_EVICT_FIRST it is marked evict-first in L2 so that it does not push out the vector being gathered.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
#if TILE_EVICT_FIRST
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
#else
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
#endif
}

enum Mode { SINGLE = 0, FIRST = 1, DEFER = 2, CATCHUP = 3 };

/// What a consumer does with a finished row sum (ar, ai) = (H term_in)_i: the new term, the c update of its mode and
/// the partial sums (acc[0] |term|^2, acc[1] |c|^2, acc[2] CATCHUP: |c + previous term|^2 / FIRST: <x|H|x>, acc[3..4]
/// FIRST: |x|^2, #non-finite).  Same operations in the same order as the row kernels and propagator.hpp:68-84.
template <int MODE>
__host__ __device__ constexpr int mode_sums() {
    return MODE == FIRST ? 5 : (MODE == CATCHUP ? 3 : (MODE == DEFER ? 1 : 2));
}
template <int MODE>
__device__ __forceinline__ void finish_row(uint32_t i, double ar, double ai, double2 cc, double2 tp, double b,
                                           double2* __restrict__ term_out, double2* __restrict__ c,
                                           double (&acc)[mode_sums<MODE>()]) {
    constexpr bool HAS_C = MODE != DEFER;
    if (MODE == FIRST) {
        // real(conj(x) * row) = xr*rr - (-xi)*ri
        acc[2] = __dadd_rn(acc[2], __dsub_rn(__dmul_rn(tp.x, ar), __dmul_rn(-tp.y, ai)));
        acc[3] = __dadd_rn(acc[3], __dadd_rn(__dmul_rn(tp.x, tp.x), __dmul_rn(tp.y, tp.y)));
        if (!isfinite(tp.x) || !isfinite(tp.y)) acc[4] = acc[4] + 1.0;
    }
    // (0, b) * (ar, ai) exactly as the compiler expands std::complex multiplication
    const double tr = __dsub_rn(__dmul_rn(0.0, ar), __dmul_rn(b, ai));
    const double ti = __dadd_rn(__dmul_rn(0.0, ai), __dmul_rn(b, ar));
    term_out[i] = make_double2(tr, ti);
    acc[0] = __dadd_rn(acc[0], __dadd_rn(__dmul_rn(tr, tr), __dmul_rn(ti, ti)));
    if (HAS_C) {
        if (MODE == CATCHUP) {
            cc.x = __dadd_rn(cc.x, tp.x);
            cc.y = __dadd_rn(cc.y, tp.y);
            acc[2] = __dadd_rn(acc[2], __dadd_rn(__dmul_rn(cc.x, cc.x), __dmul_rn(cc.y, cc.y)));
        }
        cc.x = __dadd_rn(cc.x, tr);
        cc.y = __dadd_rn(cc.y, ti);
        c[i] = cc;
        acc[1] = __dadd_rn(acc[1], __dadd_rn(__dmul_rn(cc.x, cc.x), __dmul_rn(cc.y, cc.y)));
    }
}

/// Reduction of the consumers' partial sums (fixed tree inside the CTA, per-CTA partials combined by the last CTA in
/// CTA order) and, in that last CTA, the stop rule of the launch's mode.  Called by the TR consumer threads only.
template <int MODE, int K, bool SHARD = false>
__device__ __forceinline__ void reduce_and_rule(double (&acc)[K], double* red, double* __restrict__ partials,
                                                TaylorCtl* ctl, int order, double rtol, double* __restrict__ tot_out,
                                                double* __restrict__ expect_out, int part = 0) {
    const uint32_t tid = threadIdx.x;
    auto consumer_sync = [] { asm volatile("bar.sync 1, %0;" ::"n"(TR) : "memory"); };
    const int lane = tid & 31, warp = tid >> 5;
    double blk[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
        const double w = warp_sum(acc[q]);
        consumer_sync();
        if (lane == 0) red[warp] = w;
        consumer_sync();
        double tsum = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < TR / 32; ++w2) tsum = __dadd_rn(tsum, red[w2]);
        blk[q] = tsum;
    }
    uint32_t* flag = reinterpret_cast<uint32_t*>(red + 12);
    if (tid == 0) {
#pragma unroll
        for (int q = 0; q < K; ++q) partials[size_t(q) * gridDim.x + blockIdx.x] = blk[q];
        __threadfence();
        *flag = (atomicAdd(&ctl->ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
    }
    consumer_sync();
    if (*flag == 0) return;
    __threadfence();
    double tot[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
        double a = 0.0;
        for (uint32_t g = tid; g < gridDim.x; g += TR) a = __dadd_rn(a, __ldcg(partials + size_t(q) * gridDim.x + g));
        const double w = warp_sum(a);
        consumer_sync();
        if (lane == 0) red[warp] = w;
        consumer_sync();
        double tsum = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < TR / 32; ++w2) tsum = __dadd_rn(tsum, red[w2]);
        tot[q] = tsum;
    }
    if (tid != 0) return;
    ctl->ticket = 0;
    if (SHARD) {
        // a shard only deposits the sums of this launch (its part of the rows): they are all-reduced with the other
        // part's and the other ranks', taylor_stop_kernel / taylor_stop_pair_kernel apply the rule (sharded.cuh).
        // A deferred order's |term|^2 waits in slot 3 for the catch-up order's all-reduce.
        if (MODE == DEFER) {
            tot_out[3] = tot[0];
        } else {
            tot_out[0] = tot[0];
            tot_out[1] = tot[1];
            if (MODE == CATCHUP) tot_out[2] = tot[2];
        }
        if (MODE == FIRST) {  // <x|H|x>, |x|^2, #non-finite of this part's rows
            expect_out[0] = tot[2];
            expect_out[1] = tot[3];
            expect_out[2] = tot[4];
            if (part == 0) expect_out[3] = expect_out[4] = expect_out[5] = 0.0;
        }
        // one launch for all rows: the other part's slots hold the previous all-reduce's sums (it works in place)
        if (part == 0) tot_out[4] = tot_out[5] = tot_out[6] = tot_out[7] = 0.0;
        __threadfence();
        return;
    }
    if (MODE == FIRST) {
        expect_out[0] = tot[2];
        expect_out[1] = tot[3];
        expect_out[2] = tot[4];
    }
    if (MODE == DEFER) {
        ctl->pending = 1;
        ctl->pending_tn2 = tot[0];
        ctl->deferred += 1;
        if (order > ctl->order_used) ctl->order_used = order;
        ctl->last_order = order;
    } else if (tot_out) {  // sharded: the sums are all-reduced first, taylor_stop_kernel applies the rule
        tot_out[0] = tot[0];
        tot_out[1] = tot[1];
    } else if (MODE == CATCHUP) {
        taylor_apply_rule(ctl, order - 1, ctl->pending_tn2, tot[2], rtol);  // streak was 0: cannot stop here
        taylor_apply_rule(ctl, order, tot[0], tot[1], rtol);
        ctl->pending = 0;
    } else {
        taylor_apply_rule(ctl, order, tot[0], tot[1], rtol);
    }
    __threadfence();
}

struct Layout {  // byte offsets inside the dynamic shared memory of one CTA
    uint32_t ecap;   // entries a stage holds (TR * max_row + slack for the aligned start)
    uint32_t rp, col, val, stage_bytes, bars, vt, total;
};
/// CODED: the stage holds a 2-byte value code per entry instead of the 8-byte value, and the model's table of
/// distinct matrix elements (vt_n doubles) sits behind the reduction scratch.
template <bool CODED>
__host__ __device__ inline Layout make_layout(int max_row, int vt_n) {
    Layout L;
    L.ecap = uint32_t(TR) * uint32_t(max_row) + 16;
    uint32_t o = 0;
    L.rp = o;
    o += (TR + 4) * 4;
    L.col = o;
    o += L.ecap * 4;
    o = (o + 15) & ~15u;
    L.val = o;
    o += L.ecap * (CODED ? 2 : 8);
    L.stage_bytes = (o + 127) & ~127u;
    L.bars = L.stage_bytes * stages<CODED>();  // full[STAGES], empty[STAGES]
    L.vt = L.bars + 2 * stages<CODED>() * 8 + 128;  // + reduction scratch
    L.total = L.vt + (CODED ? uint32_t(vt_n) * 8 : 0);
    return L;
}

/// Resident CTAs per SM the kernels are compiled for -- and the grid every mode uses (SMs x this), so that SINGLE,
/// DEFER, CATCHUP and FIRST share one reduction shape whatever their register appetite.
#ifndef TILE_WIDE_CTAS
#define TILE_WIDE_CTAS 3
#endif
#ifndef TILE_NARROW_CTAS
#define TILE_NARROW_CTAS 4
#endif
template <int MAXR>
constexpr int tile_ctas_per_sm() {
    return MAXR <= 5 ? TILE_NARROW_CTAS : TILE_WIDE_CTAS;
}

/// SHARD (a rank's rows of a sharded space, columns >= n index the halo): `part` selects the rows of this launch -- 1:
/// rows WITHOUT halo columns (they run while the halo exchange is in flight), 2: rows WITH halo columns (after it has
/// landed), 0: all rows -- decided per row from the columns already in shared memory; the partial sums are deposited in
/// tot_out[0..3] for the all-reduce instead of applying the stop rule here.
template <int MODE, int MAXR, bool CODED, bool SHARD = false>
__global__ void __launch_bounds__(NTHREADS, tile_ctas_per_sm<MAXR>()) taylor_tile_kernel(uint32_t n, const uint32_t* __restrict__ row_ptr,
                                                               const int32_t* __restrict__ col,
                                                               const double* __restrict__ val,
                                                               const uint16_t* __restrict__ code,
                                                               const double* __restrict__ diag,
                                                               const double* __restrict__ vtab, int vt_n,
                                                               const double2* __restrict__ term_in,
                                                               double2* __restrict__ term_out, double2* __restrict__ c,
                                                               double b, int order, double rtol, int max_row,
                                                               double* __restrict__ partials, TaylorCtl* ctl,
                                                               int ignore_stop, double* __restrict__ tot_out,
                                                               double* __restrict__ expect_out, int first_from_x,
                                                               int part, int reverse, int prefetch) {
    constexpr bool HAS_C = MODE != DEFER;
    constexpr int K = mode_sums<MODE>();
    extern __shared__ __align__(128) unsigned char smem[];
    // Programmatic dependent launch (launch_r): the NEXT order's CTAs may become resident as this order's CTAs retire and
    // run their prologue (barrier init, value table) there; they touch nothing this order writes -- the stop flags
    // included -- before griddepcontrol.wait below, which returns once the previous grid has completed and flushed.
    // Both instructions do nothing in a launch without the attribute.
    asm volatile("griddepcontrol.launch_dependents;");
    constexpr int STAGES = stages<CODED>();
    constexpr uint32_t AL = CODED ? 7u : 3u;  // the slices start at a 16-byte boundary of the narrowest array
    const Layout L = make_layout<CODED>(max_row, vt_n);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* empty = full + STAGES;
    double* red = reinterpret_cast<double*>(smem + L.bars + 2 * STAGES * 8);
    const uint32_t ntiles = (n + TR - 1) / TR;
    // Sweep direction: consecutive orders walk the rows in OPPOSITE directions.  The vector an order gathers is the one
    // the previous order wrote; the rows that launch wrote last are the ones still in L2, so this launch starts there.
    auto tile_of = [&](uint32_t t) { return reverse ? ntiles - 1 - t : t; };
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, TR / 32);  // one arrive per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const double* vt_s = reinterpret_cast<const double*>(smem + L.vt);
    if (CODED) {
        double* vt_w = reinterpret_cast<double*>(smem + L.vt);
        for (int q = int(tid); q < vt_n; q += NTHREADS) vt_w[q] = __ldg(vtab + q);
    }
    __syncthreads();

    // ---------------- producer (one lane of the last warp) streams the tiles of this CTA into the ring ----------------
    // Its state lives here because it runs in two parts: with `prefetch` (an order whose predecessor in the stream is the
    // previous order of the same series: the matrix is read-only there) the first STAGES tiles are requested BEFORE
    // griddepcontrol.wait, i.e. while the previous order's last CTAs are still running; the rest after the role split.
    uint32_t pt = blockIdx.x, pj = 0;
    uint32_t e0n = 0, e1n = 0;  // boundaries of the NEXT tile, requested one iteration ahead (two dependent loads otherwise)
    auto produce = [&](uint32_t jmax) {
        for (; pt < ntiles && pj < jmax; ++pj, pt += gridDim.x) {
            const int s = int(pj % STAGES);
            const uint32_t e0 = e0n, e1 = e1n;
            const uint32_t tn = pt + gridDim.x;
            if (tn < ntiles) {
                e0n = __ldg(row_ptr + size_t(tile_of(tn)) * TR);
                e1n = __ldg(row_ptr + min(size_t(tile_of(tn) + 1) * TR, size_t(n)));
            }
            if (pj >= STAGES) mbar_wait(empty + s, ((pj / STAGES) - 1) & 1);
            unsigned char* st = smem + size_t(s) * L.stage_bytes;
            const uint32_t r0 = tile_of(pt) * TR;
            const uint32_t rows = min(uint32_t(TR), n - r0);
            const uint32_t rp_bytes = ((rows + 1 + 3) & ~3u) * 4;
            const uint32_t a0 = e0 & ~AL;
            const uint32_t cnt = (e1 - a0 + AL) & ~AL;
            mbar_expect_tx(full + s, rp_bytes + cnt * (CODED ? 6 : 12));
            bulk_load(st + L.rp, row_ptr + r0, rp_bytes, full + s);
            if (cnt) {
                bulk_load(st + L.col, col + a0, cnt * 4, full + s);
                if (CODED)
                    bulk_load(st + L.val, code + a0, cnt * 2, full + s);
                else
                    bulk_load(st + L.val, val + a0, cnt * 8, full + s);
            }
        }
    };
    if (tid == TR) {
        if (pt < ntiles) {
            e0n = __ldg(row_ptr + size_t(tile_of(pt)) * TR);
            e1n = __ldg(row_ptr + min(size_t(tile_of(pt) + 1) * TR, size_t(n)));
        }
        if (prefetch) produce(STAGES);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    bool quit = !ignore_stop && (ld_flag(&ctl->done) | ld_flag(&ctl->bail));
    if (!quit && MODE == DEFER && ld_flag(&ctl->streak) != 0) {  // the series may stop at this order: it has to run SINGLE
        if (blockIdx.x == 0 && threadIdx.x == 0) *(volatile int*)&ctl->bail = order;
        quit = true;
    }
    if (quit) {
        // the shared memory must outlive the bulk copies already under way
        if (tid == TR)
            for (uint32_t q = 0; q < pj; ++q) mbar_wait(full + q, 0);
        return;
    }

    if (tid >= TR) {
        if (tid == TR) produce(0xffffffffu);
        return;
    }

    // ---------------- consumers: one row per thread and tile ----------------
    double acc[K];
#pragma unroll
    for (int q = 0; q < K; ++q) acc[q] = 0.0;
    uint32_t j = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; ++j, t += gridDim.x) {
        const int s = int(j % STAGES);
        unsigned char* st = smem + size_t(s) * L.stage_bytes;
        const uint32_t* rp_s = reinterpret_cast<const uint32_t*>(st + L.rp);
        const int32_t* col_s = reinterpret_cast<const int32_t*>(st + L.col);
        const double* val_s = reinterpret_cast<const double*>(st + L.val);
        const uint16_t* code_s = reinterpret_cast<const uint16_t*>(st + L.val);
        const uint32_t i = tile_of(t) * TR + tid;
        const bool live = i < n;
        // independent of the ring: this row's slice of c and (catch-up / first order) of the previous term
        double2 cc = make_double2(0.0, 0.0), tp = make_double2(0.0, 0.0);
        // (first_from_x: the state is only in term_in so far -- the first order writes c, it does not read it)
        // (SHARD: only once the row is known to belong to this launch's part, with the gathers)
        if (!SHARD) {
            if (HAS_C && live && !(MODE == FIRST && first_from_x)) cc = c[i];
            if ((MODE == CATCHUP || MODE == FIRST) && live) tp = __ldg(term_in + i);
            if (MODE == FIRST && first_from_x) cc = tp;
        }
        double dg = 0.0;  // the row's diagonal element when the model's diagonals are not in the table
        if (CODED && diag != nullptr && live) dg = __ldg(diag + i);
        mbar_wait(full + s, (j / STAGES) & 1);
        double ar = 0.0, ai = 0.0;
        bool mine = live;
        if (live) {
            const uint32_t base = rp_s[0] & ~AL;  // the slices start at the 16-byte boundary below the first entry
            const uint32_t kb = rp_s[tid] - base;
            const uint32_t len = rp_s[tid + 1] - base - kb;
            if (SHARD && part != 0) {
                bool halo = false;
#pragma unroll
                for (int u = 0; u < MAXR; ++u)
                    if (uint32_t(u) < len) halo |= uint32_t(col_s[kb + u]) >= n;
                mine = halo == (part == 2);
            }
            if (mine) {
                double2 x[MAXR];
#pragma unroll
                for (int u = 0; u < MAXR; ++u)
                    if (uint32_t(u) < len) x[u] = __ldg(term_in + col_s[kb + u]);
                if (SHARD) {
                    if (HAS_C && !(MODE == FIRST && first_from_x)) cc = c[i];
                    if (MODE == CATCHUP || MODE == FIRST) tp = __ldg(term_in + i);
                    if (MODE == FIRST && first_from_x) cc = tp;
                }
#pragma unroll
                for (int u = 0; u < MAXR; ++u)
                    if (uint32_t(u) < len) {
                        double v;
                        if (CODED) {
                            const uint32_t cd = code_s[kb + u];
                            v = cd == CODE_DIAG ? dg : vt_s[cd];
                        } else {
                            v = val_s[kb + u];
                        }
                        ar = __dadd_rn(ar, __dmul_rn(v, x[u].x));
                        ai = __dadd_rn(ai, __dmul_rn(v, x[u].y));
                    }
            }
        }
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(empty + s);  // this warp has read everything it needs from the stage
        if (mine) finish_row<MODE>(i, ar, ai, cc, tp, b, term_out, c, acc);
    }

    reduce_and_rule<MODE, K, SHARD>(acc, red, partials, ctl, order, rtol, tot_out, expect_out, part);
}

template <int MODE, int MAXR, bool CODED>
static bool launch_r(int sm_count, cudaStream_t stream, uint32_t n, const uint32_t* row_ptr, const int32_t* col,
                     const double* val, const TaylorCodes* codes, const double2* term_in, double2* term_out, double2* c,
                     double b, int order, double rtol, double* partials, TaylorCtl* ctl, int ignore_stop, double* tot_out,
                     double* expect_out, int first_from_x) {
    const int vt_n = CODED ? codes->vt_n : 0;
    const Layout L = make_layout<CODED>(MAXR, vt_n);
    static int ready = 0;     // 1: usable, -1: not (the launch falls back to the row kernels)
    static uint32_t smem_set = 0;  // dynamic shared memory the kernel is currently allowed
    if (ready == 0 || (ready > 0 && L.total > smem_set)) {
        ready = -1;
        int occ = 0;
        if (cudaFuncSetAttribute(taylor_tile_kernel<MODE, MAXR, CODED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(L.total)) == cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, taylor_tile_kernel<MODE, MAXR, CODED>, NTHREADS,
                                                          L.total) == cudaSuccess &&
            occ >= 1) {
            ready = 1;
            smem_set = L.total;
        } else {
            cudaGetLastError();
        }
    }
    if (ready < 0) return false;
    const uint32_t ntiles = (n + TR - 1) / TR;
    const uint32_t grid =
        std::max<uint32_t>(1, std::min<uint32_t>(ntiles, uint32_t(sm_count) * uint32_t(tile_ctas_per_sm<MAXR>())));
    // consecutive orders as programmatic dependent launches (see the kernel's prologue); PB200_NO_PDL=1: plain launches
    static const bool pdl = std::getenv("PB200_NO_PDL") == nullptr;
    // orders >= 2 follow the previous order of the same series in the stream: H_eff is read-only between them, so the
    // producer MAY request its first tiles before the previous order has completed.  Measured: no gain (C2 expmv 0.614
    // either way, C4 2.22 vs 2.23 ms; profiles/r2_experiments.md), so it is off unless PB200_PDL_PREFETCH=1.
    static const bool pre = std::getenv("PB200_PDL_PREFETCH") != nullptr;
    const int prefetch = pdl && pre && MODE != FIRST && order >= 2 ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    const uint16_t* code_p = CODED ? codes->code : nullptr;
    const double* diag_p = CODED ? codes->diag : nullptr;
    const double* vtab_p = CODED ? codes->vtab : nullptr;
    const cudaError_t err = cudaLaunchKernelEx(&cfg, taylor_tile_kernel<MODE, MAXR, CODED>, n, row_ptr, col, val, code_p,
                                               diag_p, vtab_p, vt_n, term_in, term_out, c, b, order, rtol, int(MAXR),
                                               partials, ctl, ignore_stop, tot_out, expect_out, first_from_x, 0,
                                               int(sweep_reverse(n, order)), prefetch);
    if (err != cudaSuccess) throw std::runtime_error(std::string("taylor_tile_kernel launch: ") + cudaGetErrorString(err));
    return true;
}

template <int MODE, bool CODED>
static bool launch_c(int sm_count, cudaStream_t stream, uint32_t n, const uint32_t* row_ptr, const int32_t* col,
                     const double* val, const TaylorCodes* codes, const double2* term_in, double2* term_out, double2* c,
                     double b, int order, double rtol, int max_row, double* partials, TaylorCtl* ctl, int ignore_stop,
                     double* tot_out, double* expect_out, int first_from_x) {
    // instantiations by row-length bound: 1D models (<= 5 entries), 2D (<= 7), 3D (<= 9)
    if (max_row <= 5)
        return launch_r<MODE, 5, CODED>(sm_count, stream, n, row_ptr, col, val, codes, term_in, term_out, c, b, order, rtol,
                                        partials, ctl, ignore_stop, tot_out, expect_out, first_from_x);
    if (max_row <= 7)
        return launch_r<MODE, 7, CODED>(sm_count, stream, n, row_ptr, col, val, codes, term_in, term_out, c, b, order, rtol,
                                        partials, ctl, ignore_stop, tot_out, expect_out, first_from_x);
    return launch_r<MODE, 9, CODED>(sm_count, stream, n, row_ptr, col, val, codes, term_in, term_out, c, b, order, rtol,
                                    partials, ctl, ignore_stop, tot_out, expect_out, first_from_x);
}

template <int MODE>
static bool launch(int sm_count, cudaStream_t stream, uint32_t n, const uint32_t* row_ptr, const int32_t* col,
                   const double* val, const TaylorCodes* codes, const double2* term_in, double2* term_out, double2* c,
                   double b, int order, double rtol, int max_row, double* partials, TaylorCtl* ctl, int ignore_stop,
                   double* tot_out, double* expect_out, int first_from_x = 0) {
    if (max_row < 1 || max_row > 9) return false;
    if (codes != nullptr && codes->code != nullptr && codes->vt_n > 0 && codes->vt_n <= TAYLOR_VT_MAX)
        return launch_c<MODE, true>(sm_count, stream, n, row_ptr, col, val, codes, term_in, term_out, c, b, order, rtol,
                                    max_row, partials, ctl, ignore_stop, tot_out, expect_out, first_from_x);
    return launch_c<MODE, false>(sm_count, stream, n, row_ptr, col, val, nullptr, term_in, term_out, c, b, order, rtol,
                                 max_row, partials, ctl, ignore_stop, tot_out, expect_out, first_from_x);
}

// ---- shards: the same kernels with the row filter; two waves of CTAs instead of a persistent grid, so that CTAs retire
// while the launch runs and the transport's kernels (halo exchange on its own, higher-priority stream) find room
constexpr int SHARD_WAVES = 2;
template <int MODE, int MAXR, bool CODED>
static bool launch_shard_r(int part, int sm_count, cudaStream_t stream, uint32_t n, const uint32_t* row_ptr,
                           const int32_t* col, const double* val, const TaylorCodes* codes, const double2* term_in,
                           double2* term_out, double2* c, double b, int order, double* partials, TaylorCtl* ctl,
                           double* tot_out, double* expect_out, int first_from_x) {
    const int vt_n = CODED ? codes->vt_n : 0;
    const Layout L = make_layout<CODED>(MAXR, vt_n);
    static int ready = 0;
    static uint32_t smem_set = 0;
    if (ready == 0 || (ready > 0 && L.total > smem_set)) {
        ready = -1;
        int occ = 0;
        if (cudaFuncSetAttribute(taylor_tile_kernel<MODE, MAXR, CODED, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(L.total)) == cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, taylor_tile_kernel<MODE, MAXR, CODED, true>, NTHREADS,
                                                          L.total) == cudaSuccess &&
            occ >= 1) {
            ready = 1;
            smem_set = L.total;
        } else {
            cudaGetLastError();
        }
    }
    if (ready < 0) return false;
    const uint32_t ntiles = (n + TR - 1) / TR;
    const uint32_t grid = std::max<uint32_t>(
        1, std::min<uint32_t>(ntiles, uint32_t(sm_count) * uint32_t(tile_ctas_per_sm<MAXR>()) * SHARD_WAVES));
    taylor_tile_kernel<MODE, MAXR, CODED, true><<<grid, NTHREADS, L.total, stream>>>(
        n, row_ptr, col, val, CODED ? codes->code : nullptr, CODED ? codes->diag : nullptr, CODED ? codes->vtab : nullptr,
        vt_n, term_in, term_out, c, b, order, 0.0, MAXR, partials, ctl, 0, tot_out, expect_out, first_from_x, part,
        sweep_reverse(n, order), 0);
    return true;
}
template <int MODE>
static bool launch_shard(int part, int sm_count, cudaStream_t stream, uint32_t n, const uint32_t* row_ptr,
                         const int32_t* col, const double* val, const TaylorCodes* codes, const double2* term_in,
                         double2* term_out, double2* c, double b, int order, int max_row, double* partials,
                         TaylorCtl* ctl, double* tot_out, double* expect_out = nullptr, int first_from_x = 0) {
#define PB_SHARD_ARGS \
    part, sm_count, stream, n, row_ptr, col, val, codes, term_in, term_out, c, b, order, partials, ctl, tot_out, expect_out, \
        first_from_x
    if (codes != nullptr && codes->code != nullptr && codes->vt_n > 0 && codes->vt_n <= TAYLOR_VT_MAX) {
        if (max_row <= 5) return launch_shard_r<MODE, 5, true>(PB_SHARD_ARGS);
        if (max_row <= 7) return launch_shard_r<MODE, 7, true>(PB_SHARD_ARGS);
        return launch_shard_r<MODE, 9, true>(PB_SHARD_ARGS);
    }
    if (val == nullptr) return false;
    if (max_row <= 5) return launch_shard_r<MODE, 5, false>(PB_SHARD_ARGS);
    if (max_row <= 7) return launch_shard_r<MODE, 7, false>(PB_SHARD_ARGS);
    return launch_shard_r<MODE, 9, false>(PB_SHARD_ARGS);
#undef PB_SHARD_ARGS
}

}  // namespace tile

static const bool g_use_tiles = std::getenv("PB200_TAYLOR_ROWS") == nullptr;

// ================================================================================================
// K4 on a shard: row-list form.  A Taylor order on a sharded space runs as TWO launches -- the rows without halo
// columns while the halo exchange is in flight, then the rows with halo columns -- and its norms are global: every
// launch only deposits its partial sums (tot_out[0..3] = |term|^2, |c|^2, |c + pending term|^2, deferred |term|^2);
// the sums of the two launches are all-reduced together and taylor_stop_kernel / taylor_stop_pair_kernel apply the
// stop rule identically on every rank.  Same row arithmetic as the kernels above.
// ================================================================================================
template <int MODE>  // tile::SINGLE, tile::DEFER, tile::CATCHUP
__global__ void __launch_bounds__(NT) taylor_rows_kernel(uint32_t nrows, const uint32_t* __restrict__ rows,
                                                         const uint32_t* __restrict__ row_ptr,
                                                         const int32_t* __restrict__ col, const double* __restrict__ val,
                                                         const double2* __restrict__ term_in,
                                                         double2* __restrict__ term_out, double2* __restrict__ c, double b,
                                                         int order, double* __restrict__ partials, TaylorCtl* ctl,
                                                         double* __restrict__ tot_out) {
    __shared__ double smem[NT / 32];
    if (ld_flag(&ctl->done) | ld_flag(&ctl->bail)) return;
    if (MODE == tile::DEFER && ld_flag(&ctl->streak) != 0) {  // the series may stop at this order: it has to run SINGLE
        if (blockIdx.x == 0 && threadIdx.x == 0) *(volatile int*)&ctl->bail = order;
        return;
    }
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (uint32_t t = blockIdx.x * NT + threadIdx.x; t < nrows; t += gridDim.x * NT) {
        const uint32_t i = __ldg(rows + t);
        const uint32_t kb = __ldg(row_ptr + i), ke = __ldg(row_ptr + i + 1);
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
        const double t2 = __dadd_rn(__dmul_rn(tr, tr), __dmul_rn(ti, ti));
        if (MODE == tile::DEFER) {
            acc[3] = __dadd_rn(acc[3], t2);
            continue;
        }
        acc[0] = __dadd_rn(acc[0], t2);
        double2 cc = c[i];
        if (MODE == tile::CATCHUP) {
            const double2 tp = __ldg(term_in + i);
            cc.x = __dadd_rn(cc.x, tp.x);
            cc.y = __dadd_rn(cc.y, tp.y);
            acc[2] = __dadd_rn(acc[2], __dadd_rn(__dmul_rn(cc.x, cc.x), __dmul_rn(cc.y, cc.y)));
        }
        cc.x = __dadd_rn(cc.x, tr);
        cc.y = __dadd_rn(cc.y, ti);
        c[i] = cc;
        acc[1] = __dadd_rn(acc[1], __dadd_rn(__dmul_rn(cc.x, cc.x), __dmul_rn(cc.y, cc.y)));
    }
    double tot[4];
    if (grid_sum<4>(acc, partials, &ctl->ticket, tot, smem) && threadIdx.x == 0) {
        if (MODE == tile::DEFER) {
            tot_out[3] = tot[3];
        } else {
            tot_out[0] = tot[0];
            tot_out[1] = tot[1];
            if (MODE == tile::CATCHUP) tot_out[2] = tot[2];
        }
        __threadfence();
    }
}

void taylor_launch_rows(int mode, int grid, cudaStream_t stream, uint32_t nrows, const uint32_t* rows,
                        const uint32_t* row_ptr, const int32_t* col, const double* val, const double2* term_in,
                        double2* term_out, double2* c, double b, int order, double* partials, TaylorCtl* ctl,
                        double* tot_out) {
    if (mode == tile::DEFER)
        taylor_rows_kernel<tile::DEFER><<<grid, NT, 0, stream>>>(nrows, rows, row_ptr, col, val, term_in, term_out, c, b, order,
                                                                partials, ctl, tot_out);
    else if (mode == tile::CATCHUP)
        taylor_rows_kernel<tile::CATCHUP><<<grid, NT, 0, stream>>>(nrows, rows, row_ptr, col, val, term_in, term_out, c, b,
                                                                  order, partials, ctl, tot_out);
    else
        taylor_rows_kernel<tile::SINGLE><<<grid, NT, 0, stream>>>(nrows, rows, row_ptr, col, val, term_in, term_out, c, b,
                                                                 order, partials, ctl, tot_out);
}

bool taylor_tiles_usable(int max_row) { return g_use_tiles && max_row >= 1 && max_row <= 9; }

bool taylor_launch_tile_shard(int mode, int part, int sm_count, cudaStream_t stream, uint32_t n, const uint32_t* row_ptr,
                              const int32_t* col, const double* val, const TaylorCodes* codes, const double2* term_in,
                              double2* term_out, double2* c, double b, int order, int max_row, double* partials,
                              TaylorCtl* ctl, double* tot_out, double* expect_out, int first_from_x) {
    if (!taylor_tiles_usable(max_row)) return false;
    if (mode == tile::DEFER)
        return tile::launch_shard<tile::DEFER>(part, sm_count, stream, n, row_ptr, col, val, codes, term_in, term_out, nullptr,
                                               b, order, max_row, partials, ctl, tot_out);
    if (mode == tile::CATCHUP)
        return tile::launch_shard<tile::CATCHUP>(part, sm_count, stream, n, row_ptr, col, val, codes, term_in, term_out, c, b,
                                                 order, max_row, partials, ctl, tot_out);
    if (mode == tile::FIRST)
        return tile::launch_shard<tile::FIRST>(part, sm_count, stream, n, row_ptr, col, val, codes, term_in, term_out, c, b,
                                               order, max_row, partials, ctl, tot_out, expect_out, first_from_x);
    return tile::launch_shard<tile::SINGLE>(part, sm_count, stream, n, row_ptr, col, val, codes, term_in, term_out, c, b,
                                            order, max_row, partials, ctl, tot_out);
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
                          double* tot_out, double* expect_out, int max_row, const TaylorCodes* codes,
                          int first_from_x) {
    if (g_use_tiles && max_row > 0) {
        const bool ok = expect ? tile::launch<tile::FIRST>(sm_count, stream, n, row_ptr, col, val, codes, term_in, term_out,
                                                           c, b, order, rtol, max_row, partials, ctl, ignore_stop, tot_out,
                                                           expect_out, first_from_x)
                               : tile::launch<tile::SINGLE>(sm_count, stream, n, row_ptr, col, val, codes, term_in, term_out,
                                                            c, b, order, rtol, max_row, partials, ctl, ignore_stop, tot_out,
                                                            expect_out);
        if (ok) return;
    }
    if (expect) {
        // this variant needs more registers: size its grid to what is resident so the launch is a single wave
        static const int per_sm = resident_ctas(taylor_order_kernel_t<true>, 4);
        taylor_order_kernel_t<true><<<std::min(grid, sm_count * per_sm), NT, 0, stream>>>(
            n, row_ptr, col, val, term_in, term_out, c, b, order, rtol, partials, ctl, ignore_stop, tot_out, expect_out,
            first_from_x);
    } else {
        taylor_order_kernel_t<false><<<grid, NT, 0, stream>>>(n, row_ptr, col, val, term_in, term_out, c, b, order, rtol,
                                                              partials, ctl, ignore_stop, tot_out, expect_out, 0);
    }
}

void taylor_launch_defer(int grid, int sm_count, cudaStream_t stream, uint32_t n, const uint32_t* row_ptr,
                         const int32_t* col, const double* val, const double2* term_in, double2* term_out, double b,
                         int order, double* partials, TaylorCtl* ctl, int max_row, const TaylorCodes* codes) {
    if (g_use_tiles && max_row > 0 &&
        tile::launch<tile::DEFER>(sm_count, stream, n, row_ptr, col, val, codes, term_in, term_out, nullptr, b, order, 0.0,
                                  max_row, partials, ctl, 0, nullptr, nullptr))
        return;
    taylor_defer_kernel<<<grid, NT, 0, stream>>>(n, row_ptr, col, val, term_in, term_out, b, order, partials, ctl);
}

void taylor_launch_catchup(int grid, int sm_count, cudaStream_t stream, uint32_t n, const uint32_t* row_ptr,
                           const int32_t* col, const double* val, const double2* term_in, double2* term_out, double2* c,
                           double b, int order, double rtol, double* partials, TaylorCtl* ctl, int max_row,
                           const TaylorCodes* codes) {
    if (g_use_tiles && max_row > 0 &&
        tile::launch<tile::CATCHUP>(sm_count, stream, n, row_ptr, col, val, codes, term_in, term_out, c, b, order, rtol,
                                    max_row, partials, ctl, 0, nullptr, nullptr))
        return;
    static const int per_sm = resident_ctas(taylor_catchup_kernel, 4);
    taylor_catchup_kernel<<<std::min(grid, sm_count * per_sm), NT, 0, stream>>>(n, row_ptr, col, val, term_in, term_out,
                                                                               c, b, order, rtol, partials, ctl);
}

}  // namespace pb
