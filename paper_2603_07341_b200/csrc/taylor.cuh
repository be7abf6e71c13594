// taylor.cuh -- K4, the fused Taylor-order kernels of expmv (propagator.hpp:52-92): control block and launchers.
// The kernels live in their own translation unit (taylor.cu): they are latency-bound and need exact register budgets
// (32 / 40), and inside the large unity module (-split-compile) ptxas was seen to give the same source 40 registers or
// spills depending on unrelated code.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace pb {

struct TaylorCtl {
    int done;        // stop rule satisfied: later launches of this substep return immediately
    int streak;      // consecutive small terms (propagator.hpp:80)
    int order_used;  // max over substeps (propagator.hpp:78)
    int last_order;  // order of the most recent launch that did work
    double last_term_norm;
    double last_c_norm;
    unsigned ticket;
    int pending;         // the previous order ran deferred: its term is not in c yet, its stop rule not applied
    double pending_tn2;  // |term|^2 of that order
    int bail;            // a deferred launch found streak != 0 at this order and did nothing: the host relaunches it SINGLE
    unsigned deferred;   // launches that ran deferred (statistics)
};

/// Value codes of a model-built H_eff (Engine::encode_values): the matrix holds only a few hundred distinct elements
/// (bond amplitudes, g*sqrt(k), omega*N), so the tile kernels can stream a 2-byte code per entry instead of the 8-byte
/// value -- 6 of the 12 bytes per non-zero -- and look the double up in a shared-memory copy of the table: the very
/// same operand bits, hence the very same products and sums.  CODE_DIAG marks the diagonal entry of a row when the
/// model's diagonal elements are not tabulated (disordered omega / eps): its value comes from diag[row].
constexpr uint32_t CODE_DIAG = 0xffffu;
constexpr uint32_t CODE_FAIL = 0xfffeu;  // encode: value not in the table (the space then keeps using `val`)
constexpr int TAYLOR_VT_MAX = 2048;      // table entries the kernels copy into shared memory
struct TaylorCodes {
    const uint16_t* code;  // [nnz]
    const double* diag;    // [n] or nullptr (diagonal elements are in the table)
    const double* vtab;    // [vt_n] distinct matrix elements, ascending bit patterns
    int vt_n;
};

/// max_row: upper bound on the entries of a row (0 = unknown).  With a bound <= 15 the launch uses the TMA tile kernels
/// (taylor.cu, namespace tile); otherwise -- arbitrary uploaded CSR matrices -- the thread-per-row kernels.
/// PB200_TAYLOR_ROWS=1 forces the row kernels (A/B measurements).
/// first_from_x (first order of a step, expect = true): the state vector is only in term_in so far; the launch uses it
/// as the old c as well and only WRITES c -- no copy of the state into the term buffer, no read of c.
/// Launch modes (see taylor.cu).  `grid` is the caller's row grid (8 CTAs per SM); the first-order and catch-up
/// kernels clamp it to one resident wave.  All launches are asynchronous on `stream`; errors surface in the caller's
/// cudaGetLastError check.
void taylor_launch_single(bool expect, int grid, int sm_count, cudaStream_t stream, uint32_t n, const uint32_t* row_ptr,
                          const int32_t* col, const double* val, const double2* term_in, double2* term_out, double2* c,
                          double b, int order, double rtol, double* partials, TaylorCtl* ctl, int ignore_stop,
                          double* tot_out, double* expect_out, int max_row, const TaylorCodes* codes = nullptr,
                          int first_from_x = 0);
void taylor_launch_defer(int grid, int sm_count, cudaStream_t stream, uint32_t n, const uint32_t* row_ptr,
                         const int32_t* col, const double* val, const double2* term_in, double2* term_out, double b,
                         int order, double* partials, TaylorCtl* ctl, int max_row, const TaylorCodes* codes = nullptr);
void taylor_launch_catchup(int grid, int sm_count, cudaStream_t stream, uint32_t n, const uint32_t* row_ptr,
                           const int32_t* col, const double* val, const double2* term_in, double2* term_out, double2* c,
                           double b, int order, double rtol, double* partials, TaylorCtl* ctl, int max_row,
                           const TaylorCodes* codes = nullptr);

/// Sharded SpMV (taylor.cu, row-list form): mode 0 = SINGLE, 2 = DEFER, 3 = CATCHUP; the launch covers rows[0..nrows)
/// and deposits its partial sums in tot_out[0..3].
constexpr int TAYLOR_ROWS_SINGLE = 0, TAYLOR_ROWS_DEFER = 2, TAYLOR_ROWS_CATCHUP = 3;
void taylor_launch_rows(int mode, int grid, cudaStream_t stream, uint32_t nrows, const uint32_t* rows,
                        const uint32_t* row_ptr, const int32_t* col, const double* val, const double2* term_in,
                        double2* term_out, double2* c, double b, int order, double* partials, TaylorCtl* ctl,
                        double* tot_out);


/// Sharded SpMV, tile form (the kernels of the single-GPU path with a row filter): part 1 = the rows without halo
/// columns, 2 = the rows with halo columns, 0 = all rows; modes and deposits as taylor_launch_rows, plus mode 1 = FIRST
/// (the first order of a step: <x|H|x>, |x|^2 and the non-finite count of the part's rows go to expect_out[0..2], and
/// with first_from_x the input vector doubles as the old c).  Returns false when the tile kernels cannot take the
/// matrix (row-length bound unknown or > 9): the caller uses the row lists.
constexpr int TAYLOR_ROWS_FIRST = 1;
bool taylor_tiles_usable(int max_row);
bool taylor_launch_tile_shard(int mode, int part, int sm_count, cudaStream_t stream, uint32_t n, const uint32_t* row_ptr,
                              const int32_t* col, const double* val, const TaylorCodes* codes, const double2* term_in,
                              double2* term_out, double2* c, double b, int order, int max_row, double* partials,
                              TaylorCtl* ctl, double* tot_out, double* expect_out = nullptr, int first_from_x = 0);

}  // namespace pb
