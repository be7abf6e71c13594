/*
 * paces_b200.h -- C ABI of the B200-native paces adapt-evolve-truncate timestep.
 *
 * This is the drop-in boundary.  The reference (arxiv 2603.07341, "paces") has no FFI layer: its
 * operator API is the set of inline C++ free functions in namespace paces that run()/step() and the
 * reference tests call.  Every entry point below names the reference function it replaces
 * (file:line relative to /root/reference/proj/include/paces/).  include/paces_b200.hpp re-creates the
 * reference's C++ signatures on top of this header; paper_2603_07341_b200/ binds it with ctypes.
 *
 * Conventions
 *   - Every function returns 0 on success.  Nonzero: PB200_ERR_PACES means the reference would have
 *     thrown paces::Error (common.hpp:21-24) and pb200_last_error() holds the same text (tests grep
 *     "memory cap", "reduce dt", ...); PB200_ERR_CUDA is a CUDA runtime failure; PB200_ERR_ARG is a
 *     misuse of this ABI (null pointer, call out of order).
 *   - Layouts are the reference's: keys are row-major rows x Omega uint32 words, lexicographically
 *     sorted, no duplicates (basis_codec.hpp:206-238); coefficients are interleaved (re, im) doubles
 *     (std::complex<double>); CSR is int64 row_ptr[n+1] / int32 col[nnz] ascending per row /
 *     double val[nnz] (subspace.hpp:25-32).  All pointers are HOST pointers owned by the caller; the
 *     context owns every device allocation; no allocation crosses the ABI.
 *   - A context drives one GPU on one stream and is not re-entrant; independent contexts may run
 *     concurrently.  There is no CPU fallback: pb200_ctx_create fails when no sm_100
 *     device is visible.
 */
#ifndef PACES_B200_H
#define PACES_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PB200_OK 0
#define PB200_ERR_PACES 1
#define PB200_ERR_CUDA 2
#define PB200_ERR_ARG 3

typedef struct pb200_ctx pb200_ctx;

/* RunConfig (engine.hpp:34-64) flattened; identical field meaning. */
typedef struct pb200_run_cfg {
    int32_t init_kind;  /* InitialStateSpec::Kind: 0 localized, 1 optical, 2 explicit list (engine.hpp:25-32) */
    int64_t init_site;  /* localized: lattice site, -1 = centre (engine.hpp:173-178) */
    int32_t m_init;
    int32_t m;
    uint64_t q_nom;
    double dt;
    double rtol;
    int32_t max_order;
    int32_t substeps;
    double t_max;
    uint64_t seed;
    uint64_t cadence;
    uint64_t n_entries;        /* explicit list: n_entries occupation vectors of layout-site length */
    const uint32_t* entry_occ; /* n_entries x layout_sites */
    const double* entry_amp;   /* n_entries x (re, im) */
} pb200_run_cfg;

/* DiagnosticsRecord (engine.hpp:67-77). */
typedef struct pb200_diag {
    uint64_t step;
    double t;
    double norm_pre;
    double norm_post;
    double discarded_weight;
    double delta_norm_expmv;
    double energy;
    uint64_t q_true;
    int32_t taylor_order;
    int32_t pad_;
} pb200_diag;

/* Device-time breakdown of the resident step (CUDA events on the context's stream), cumulative
 * since pb200_run_begin; the phases are those of SURVEY 3.5. */
typedef struct pb200_phase_times {
    double select_ms, grow_ms, assemble_ms, remap_ms, expectation_ms, expmv_ms, total_ms;
    uint64_t spmv_nnz;      /* sum over Taylor orders of nnz(H_eff) */
    uint64_t taylor_orders; /* number of fused Taylor-order launches */
    uint64_t kernel_launches;
    uint64_t steps;
    uint64_t taylor_deferred; /* of taylor_orders: launches that ran deferred (c untouched: 12z + 40n bytes) */
    uint64_t taylor_rows;          /* sum over Taylor-order launches of the rows they covered */
    uint64_t taylor_deferred_rows; /* same, deferred launches only */
    uint64_t rows_sum, nnz_sum;    /* sum over steps of q_true and nnz(H_eff) of the space the step evolved on */
    uint64_t rows_old_sum;         /* sum over steps of the rows of the state the step started from */
    uint64_t kept_sum;             /* sum over steps of the keys truncate_select kept */
    uint64_t spmv_nnz_coded;       /* of spmv_nnz: non-zeros streamed as 2-byte value codes (6 instead of 12 bytes each) */
    /* assemble_ms, remap_ms and expectation_ms stay ~0 in the resident single-GPU step: assembly and remap are
     * part of the incremental adapt phase (inside grow_ms), <H> rides on the first Taylor order (inside expmv_ms) */
} pb200_phase_times;

/* ---- context ------------------------------------------------------------------------------- */
int pb200_ctx_create(int device, pb200_ctx** out);
void pb200_ctx_destroy(pb200_ctx* ctx);
/* Message of the last failing call on ctx (ctx == NULL: of the last failing pb200_ctx_create). */
const char* pb200_last_error(const pb200_ctx* ctx);
const char* pb200_version(void);
/* Optional externally owned CUDA stream (cudaStream_t as void*); default: a stream the ctx creates. */
int pb200_ctx_set_stream(pb200_ctx* ctx, void* cuda_stream);
/* Number of kernels this context has launched so far. */
uint64_t pb200_kernel_launches(const pb200_ctx* ctx);
/* common.hpp:76-81 (host-side splitmix64; the per-step tie-break seed of engine.hpp:275). */
uint64_t pb200_mix_seed(uint64_t x);

/* ---- multi-GPU: one process (and one context) per GPU; the table is sharded by hash of the phonon part of the
 * basis key.  The collectives come either from NCCL inside the library (pb200_ctx_set_comm_nccl,
 * below -- the production path) or from the host through this table (any other transport; tests).  Device
 * variants receive DEVICE pointers on the context's device plus the context's stream; they must be complete or
 * stream-ordered on that stream when they return.  Host variants are small blocking collectives on host memory.
 * All ranks call every pb200_* function collectively and in the same order.  Every callback returns 0 on success. */
typedef struct pb200_comm_ops {
    void* user;
    int (*allreduce_f64_host)(void* user, double* buf, uint64_t n);          /* sum, in place */
    int (*allreduce_u64_host)(void* user, uint64_t* buf, uint64_t n);        /* sum, in place */
    /* one value per peer.  Not called any more: the per-peer counts of a routed exchange travel on the device
     * (alltoallv_dev with one 4-byte element per peer) and come back in one read-back; the slot stays for ABI
     * compatibility and must still be non-NULL. */
    int (*alltoall_u64_host)(void* user, const uint64_t* send, uint64_t* recv);
    int (*allgather_host)(void* user, const void* send, uint64_t nbytes, void* recv); /* recv: world * nbytes */
    /* buckets are contiguous and in rank order on both sides; counts are in elements of elem_bytes bytes (1 for the BFS
     * distances of the halo rows, 4 for counts and look-up replies, 4 * words for keys, 16 for complex128 halos);
     * the device pointers need no alignment beyond elem_bytes */
    int (*alltoallv_dev)(void* user, const void* send, const uint64_t* send_counts, void* recv,
                         const uint64_t* recv_counts, uint64_t elem_bytes, void* stream);
    int (*allreduce_f64_dev)(void* user, double* buf, uint64_t n, void* stream);   /* sum, in place */
    int (*allreduce_u32_dev)(void* user, uint32_t* buf, uint64_t n, void* stream); /* sum, in place */
    /* Optional (may be NULL): alltoallv_dev on an INDEPENDENT channel that is allowed to run concurrently with the
     * other collectives (the halo exchange of a Taylor order, issued on its own stream beside the interior rows of
     * the SpMV).  NULL: the halo exchange is ordered on the context's stream like everything else. */
    int (*alltoallv_dev2)(void* user, const void* send, const uint64_t* send_counts, void* recv,
                          const uint64_t* recv_counts, uint64_t elem_bytes, void* stream);
} pb200_comm_ops;
/* Must be called before pb200_model_set; world == 1 (or never calling it) is the single-GPU path. */
int pb200_ctx_set_comm(pb200_ctx* ctx, int rank, int world, const pb200_comm_ops* ops);
/* The production transport: NCCL inside the library (NVLink 5 / NVSwitch on a B200 box; libnccl.so.2 is resolved at
 * run time).  Rank 0 calls pb200_nccl_unique_id and hands the PB200_NCCL_ID_BYTES bytes to every rank (MPI, a file,
 * torch.distributed, ... -- the only thing the host has to move); then every rank calls pb200_ctx_set_comm_nccl
 * (collective: it creates the communicators) before pb200_model_set.  The callback table above stays available for
 * other transports and for tests (several ranks on one GPU, which NCCL refuses). */
#define PB200_NCCL_ID_BYTES 256
int pb200_nccl_unique_id(uint8_t* id);
int pb200_ctx_set_comm_nccl(pb200_ctx* ctx, int rank, int world, const uint8_t* id);
/* One line about the context's transport (NCCL version, rank, collectives issued so far); "" without one. */
const char* pb200_comm_describe(pb200_ctx* ctx);
/* Shard owner of a key (host-side restatement of the device rule), and this context's rank/world. */
int pb200_owner_of(const pb200_ctx* ctx, const uint32_t* key, uint32_t world, uint32_t* owner);

/* ---- model: build_model (lattice_models.hpp:140-189) ---------------------------------------------
 * kind: 0 tight_binding, 1 holstein.  eps/hop/omega/g hold 0, 1 or n values (broadcast rule of
 * lattice_models.hpp:129-136; hop is per bond in LatticeGeometry::bonds() order, :54-65).  The
 * spin-lattice kind is rejected exactly as initialize() rejects it (engine.hpp:238-239). */
int pb200_model_set(pb200_ctx* ctx, int kind, int ndim, const uint32_t* extents, const double* eps,
                    int n_eps, const double* hop, int n_hop, const double* omega, int n_omega,
                    const double* g, int n_g, uint32_t d_pho);
int pb200_model_info(const pb200_ctx* ctx, uint32_t* layout_sites, uint32_t* words_per_row,
                     uint32_t* lattice_sites, uint32_t* n_terms, uint32_t* total_bits);
/* pack_state / unpack_state (basis_codec.hpp:131-172), host-side. */
int pb200_pack(const pb200_ctx* ctx, const uint32_t* occ, uint32_t* words);
int pb200_unpack(const pb200_ctx* ctx, const uint32_t* words, uint32_t* occ);
/* apply_terms (lattice_models.hpp:212-267) for n_keys keys on the device: per key up to `cap`
 * (neighbour key, amplitude) pairs in CANONICAL (ascending key) order -- the reference emits them in term order;
 * as sorted sets the two are identical (tests/test_gpu_parity.py) -- count[i] of them. */
int pb200_apply_terms(pb200_ctx* ctx, const uint32_t* keys, uint64_t n_keys, uint32_t* out_keys,
                      double* out_amps, int cap, int* count);

/* ---- stand-alone operators: host buffers in, host buffers out ---------------------------------
 * Each uploads its inputs, runs the same kernels as the resident step and downloads the result. */

/* grow_subspace (subspace.hpp:195-249) incl. assemble_effective_hamiltonian (:142-187).  The grown
 * space stays resident as the context's current space; read it with pb200_space_info/_get. */
int pb200_grow(pb200_ctx* ctx, const uint32_t* seeds, uint64_t rows, int order, uint64_t* q_true,
               uint64_t* nnz);
int pb200_space_info(const pb200_ctx* ctx, uint64_t* q_true, uint64_t* nnz, uint64_t* q_nom);
int pb200_space_get(pb200_ctx* ctx, uint32_t* words, int64_t* row_ptr, int32_t* col, double* val);

/* truncate_select (engine.hpp:107-156): out_words has room for min(rows, q_nom) rows. */
int pb200_truncate_select(pb200_ctx* ctx, const uint32_t* words, const double* coeff, uint64_t rows,
                          uint64_t q_nom, uint64_t seed, uint32_t* out_words, uint64_t* kept);
/* remap_state (subspace.hpp:281-305). */
int pb200_remap(pb200_ctx* ctx, const uint32_t* src_words, const double* src_coeff,
                uint64_t src_rows, const uint32_t* dst_words, uint64_t dst_rows, double* out_coeff,
                double* discarded);
/* csr_matvec (subspace.hpp:35-43), csr_expectation (:46-55), expmv (propagator.hpp:52-92). */
int pb200_csr_matvec(pb200_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* col,
                     const double* val, const double* x, double* y);
int pb200_csr_expectation(pb200_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* col,
                          const double* val, const double* x, double* out);
int pb200_expmv(pb200_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* col,
                const double* val, double* c, double dt, double rtol, int max_order, int substeps,
                int* order_used, double* last_term_norm);
/* state_norm (subspace.hpp:91-95), exciton_density (observables.hpp:26-37), dipole_amplitude
 * (observables.hpp:99-112), phonon_numbers (observables.hpp:84-95). */
int pb200_state_norm(pb200_ctx* ctx, const double* coeff, uint64_t rows, double* out);
int pb200_exciton_density(pb200_ctx* ctx, const uint32_t* words, const double* coeff, uint64_t rows,
                          double* p);
int pb200_dipole_amplitude(pb200_ctx* ctx, const uint32_t* words, const double* coeff,
                           uint64_t rows, double* amp);
int pb200_phonon_numbers(pb200_ctx* ctx, const uint32_t* words, const double* coeff, uint64_t rows,
                         double* n_out);

/* weight_histogram (observables.hpp:114-176): descending |c|^2 curve of the non-zero
 * coefficients, the counts reaching 50 / 90 / 99 / 99.99 % of the total weight, the log-log tail slope, and the
 * curve sampled at `bins` ranks (0 = every rank).  Everything runs on the GPU (stable LSD radix sort of the
 * weights' bit patterns, prefix sums for the marks, a grid reduction for the slope); only min(cap, *npts) curve
 * points and a 64-byte result block are downloaded.  support, the sampled ranks and weights are exact; the marks
 * use fixed-tree prefix sums instead of the reference's serial running sum (they can differ only when a running
 * sum lies within rounding distance of a threshold); tail_exponent agrees to 1e-10 relative.
 * pb200_run_weight_histogram works on the resident state. */
typedef struct {
    uint64_t support, q50, q90, q99, q9999;
    double tail_exponent;
} pb200_weight_hist;
int pb200_weight_histogram(pb200_ctx* ctx, const double* coeff, uint64_t rows, uint64_t bins,
                           pb200_weight_hist* out, uint64_t* rank, double* weight, uint64_t cap,
                           uint64_t* npts);
int pb200_run_weight_histogram(pb200_ctx* ctx, uint64_t bins, pb200_weight_hist* out, uint64_t* rank,
                               double* weight, uint64_t cap, uint64_t* npts);

/* ---- device-resident trajectory: initialize / step / run (engine.hpp:235-291, 318-375) ----------
 * pb200_run_begin = initialize(): seed state, grow to m_init, remap.  pb200_run_step advances one
 * timestep exactly as run() does: step 1 evolves on the m_init space (engine.hpp:335-352), steps >= 2
 * are step() (engine.hpp:268-291).  State and space stay in HBM between steps; a failing step leaves
 * the last good state current (engine.hpp:263-267) and reports the reference's message. */
int pb200_run_begin(pb200_ctx* ctx, const pb200_run_cfg* cfg);
int pb200_run_step(pb200_ctx* ctx, pb200_diag* out);
int pb200_run_info(const pb200_ctx* ctx, uint64_t* rows, uint64_t* nnz, double* t,
                   uint64_t* steps_done);
/* Sharded runs: pb200_run_info/_state/_csr describe THIS rank's shard; the job-wide sizes are here. */
int pb200_run_global(const pb200_ctx* ctx, uint64_t* rows_global, uint64_t* nnz_global);
/* Canonical-order download: keys ascending, coefficients aligned (checkpoint order, io.hpp:77-99). */
int pb200_run_state(pb200_ctx* ctx, uint32_t* words, double* coeff);
int pb200_run_csr(pb200_ctx* ctx, int64_t* row_ptr, int32_t* col, double* val);
/* Replaces the resident state/space by a host-supplied pair (checkpoint resume, io.hpp:101-144 read side):
 * the sorted table is taken as is and H_eff is assembled over it (grow_subspace with m = 0). */
int pb200_run_load_state(pb200_ctx* ctx, const pb200_run_cfg* cfg, const uint32_t* words,
                         const double* coeff, uint64_t rows, double t, uint64_t steps_done);
/* step() (engine.hpp:268-291) as a stand-alone operator on HOST buffers: uploads the caller's SparseState
 * (sorted table + coefficients at time t), runs select -> grow -> remap -> expectation -> expmv for
 * step_index >= 2 (the index only feeds the tie-break seed, engine.hpp:275) and leaves the new
 * (state, space) resident; rows_out/nnz_out size the buffers for pb200_run_state / pb200_run_csr, which
 * download StepOutput.state and StepOutput.space. */
int pb200_step(pb200_ctx* ctx, const pb200_run_cfg* cfg, uint64_t step_index, const uint32_t* words,
               const double* coeff, uint64_t rows, double t, pb200_diag* out, uint64_t* rows_out,
               uint64_t* nnz_out);
/* Same operator with the transfers overlapped with the step: the key upload runs beside the weight/selection
 * kernels (which only need the coefficients), the download of the new table runs beside remap + <H> + expmv, and only
 * the new coefficients cross PCIe after the last Taylor order.  out_words/out_coeff must hold out_cap_rows rows
 * (pinned host memory for full PCIe speed); fails with PB200_ERR_ARG if the new state has more rows.
 * The context keeps its last result resident.  When a call is the next step of that result (same step index, time
 * and run parameters), the uploaded coefficients and keys are compared on the device with the resident ones -- on
 * their own stream, beside the step -- and, when they are bit-identical, the step works on the resident table and
 * H_eff (the caller's EffectiveSpace, engine.hpp:268) and takes the incremental adapt path; nothing is committed
 * before both comparisons agree.  Any difference, and the step is redone from the caller's buffers.
 * The input buffers are read while the outputs are written: words/coeff must not overlap out_words/out_coeff
 * (PB200_ERR_ARG otherwise) -- alternate between two buffer sets. */
int pb200_step_io(pb200_ctx* ctx, const pb200_run_cfg* cfg, uint64_t step_index, const uint32_t* words,
                  const double* coeff, uint64_t rows, double t, uint32_t* out_words, double* out_coeff,
                  uint64_t out_cap_rows, pb200_diag* out, uint64_t* rows_out, uint64_t* nnz_out);
/* detail::observe (engine.hpp:299-311): ObservablesRow of the resident state; density has
 * lattice_sites entries, amp is (re, im). */
int pb200_run_observe(pb200_ctx* ctx, double* norm, double* energy, double* rmsd, double* xbar,
                      double* amp, double* density);
int pb200_run_times(const pb200_ctx* ctx, pb200_phase_times* out);
/* How the resident steps grew their subspace: steps taken by the incremental adapt path (old-index-space BFS over
 * the previous H_eff, incremental.cuh), steps that fell back to the full expansion, and how much key-based work the
 * incremental steps still needed (old rows re-expanded, keys that entered from outside the previous table). */
typedef struct {
    uint64_t incremental_steps, fallbacks, expanded_rows, side_keys;
} pb200_adapt_stats;
int pb200_run_adapt_stats(const pb200_ctx* ctx, pb200_adapt_stats* out);
int pb200_run_reset_times(pb200_ctx* ctx);

/* ---- measurement helpers (bench.py) -----------------------------------------------------------
 * Runs `orders` fused Taylor-order launches (SpMV + scale + axpy + two norms, propagator.hpp:68-77)
 * on the resident space with the stop rule disabled, timing them with CUDA events on the context's
 * stream; the resident state is restored afterwards.  flush_l2 != 0 overwrites a buffer larger than
 * L2 between launches (outside the timed intervals). */
int pb200_bench_taylor(pb200_ctx* ctx, int orders, int flush_l2, double dt, double* ms_per_order,
                       uint64_t* nnz, uint64_t* rows);
/* Same for the plain SpMV y = H x (subspace.hpp:35-43). */
int pb200_bench_spmv(pb200_ctx* ctx, int reps, int flush_l2, double* ms_per_spmv);

#ifdef __cplusplus
}
#endif
#endif
