/*
 * oracle_abi.h -- C ABI shared by the two CPU checkers of the paces hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is product code: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load these libraries, and only as the checker / the
 * timed CPU baseline -- never as a fallback for the CUDA path.
 *
 * Two shared objects export exactly this symbol set:
 *
 *   oracle/_ref/libpaces_ref.so   built from oracle/ref_shim.cpp, a thin
 *                                 adapter over the UNMODIFIED reference
 *                                 headers compiled where they lie
 *                                 (/root/reference/proj/include/paces/...).
 *   oracle/libpaces_oracle.so     built from oracle/paces_oracle.cpp, an
 *                                 independent restatement of the same
 *                                 algorithm that needs no reference files.
 *
 * Layouts are the reference's: keys are row-major rows x Omega uint32 words
 * (basis_codec.hpp:206-238), coefficients are interleaved (re, im) doubles
 * (std::complex<double>), CSR is int64 row_ptr / int32 col / double val
 * (subspace.hpp:25-32).
 *
 * Every function returns 0 on success, nonzero on error; po_last_error()
 * returns the message of the last failing call on the calling thread (the
 * text of the reference's paces::Error where one was thrown).
 */
#ifndef PACES_ORACLE_ABI_H
#define PACES_ORACLE_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct po_model po_model; /* HamiltonianTermSet + ModelSpec */
typedef struct po_space po_space; /* EffectiveSpace: sorted table + CSR */
typedef struct po_run po_run;     /* (state, space) pair advanced step by step */

/* RunConfig (engine.hpp:34-64) flattened. */
typedef struct po_run_cfg {
    int32_t init_kind;  /* 0 localized, 1 optical, 2 explicit list */
    int64_t init_site;  /* localized: lattice site, -1 = centre */
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
    /* explicit list (init_kind == 2): n_entries occupation vectors of
     * layout-site length, amplitudes interleaved (re, im) */
    uint64_t n_entries;
    const uint32_t* entry_occ;
    const double* entry_amp;
} po_run_cfg;

/* DiagnosticsRecord (engine.hpp:67-77). */
typedef struct po_diag {
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
} po_diag;

const char* po_last_error(void);
const char* po_impl_name(void); /* "reference" or "port" */
void po_set_threads(int n);     /* common.hpp:55-61 */
int po_get_threads(void);
uint64_t po_mix_seed(uint64_t x); /* common.hpp:76-81 */

/* ---- model (lattice_models.hpp:140-189) -------------------------------- */
/* kind: 0 tight_binding, 1 holstein.  eps/hop/omega/g: 0, 1 or n values
 * (broadcast rule of lattice_models.hpp:129-136). */
int po_model_create(int kind, int ndim, const uint32_t* extents, const double* eps, int n_eps,
                    const double* hop, int n_hop, const double* omega, int n_omega,
                    const double* g, int n_g, uint32_t d_pho, po_model** out);
void po_model_destroy(po_model* m);
int po_model_info(const po_model* m, uint32_t* layout_sites, uint32_t* words_per_row,
                  uint32_t* lattice_sites, uint32_t* n_terms, uint32_t* total_bits);
int po_model_dims(const po_model* m, uint32_t* dims);

/* ---- codec (basis_codec.hpp:131-172) ----------------------------------- */
int po_pack(const po_model* m, const uint32_t* occ, uint32_t* words);
int po_unpack(const po_model* m, const uint32_t* words, uint32_t* occ);

/* ---- term application (lattice_models.hpp:212-267) --------------------- */
int po_apply_terms(const po_model* m, const uint32_t* key, uint32_t* out_keys, double* out_amps,
                   int cap, int* count);

/* ---- subspace growth + assembly (subspace.hpp:142-249) ----------------- */
int po_grow(const po_model* m, const uint32_t* seeds, uint64_t rows, int order, po_space** out);
int po_space_info(const po_space* s, uint64_t* q_true, uint64_t* nnz, uint64_t* q_nom);
int po_space_get(const po_space* s, uint32_t* words, int64_t* row_ptr, int32_t* col, double* val);
void po_space_destroy(po_space* s);

/* ---- selection / remap (engine.hpp:107-156, subspace.hpp:281-305) ------ */
int po_truncate_select(const po_model* m, const uint32_t* words, const double* coeff, uint64_t rows,
                       uint64_t q_nom, uint64_t seed, uint32_t* out_words, uint64_t* kept);
int po_remap(const po_model* m, const uint32_t* src_words, const double* src_coeff,
             uint64_t src_rows, const uint32_t* dst_words, uint64_t dst_rows, double* out_coeff,
             double* discarded);

/* ---- sparse kernels (subspace.hpp:35-55, propagator.hpp:52-92) --------- */
int po_csr_matvec(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                  const double* x, double* y);
int po_csr_expectation(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                       const double* x, double* out);
int po_expmv(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val, double* c,
             double dt, double rtol, int max_order, int substeps, int* order_used,
             double* last_term_norm);

/* ---- reductions (subspace.hpp:91-95, observables.hpp:26-37,99-112) ----- */
int po_state_norm(const double* coeff, uint64_t rows, double* out);
int po_exciton_density(const po_model* m, const uint32_t* words, const double* coeff, uint64_t rows,
                       double* p);
int po_dipole_amplitude(const po_model* m, const uint32_t* words, const double* coeff,
                        uint64_t rows, double* amp);
/* "next" row (observables.hpp:84-95) */
int po_phonon_numbers(const po_model* m, const uint32_t* words, const double* coeff, uint64_t rows,
                      double* n_out);

/* "next" row (observables.hpp:114-176): sorted |c|^2 curve, cumulative-weight quantiles, tail slope.
 * rank/weight receive min(cap, npts) sampled points; npts = support when bins == 0 or support <= bins. */
typedef struct {
    uint64_t support, q50, q90, q99, q9999;
    double tail_exponent;
} po_weight_hist;
int po_weight_histogram(const double* coeff, uint64_t rows, uint64_t bins, po_weight_hist* out,
                        uint64_t* rank, double* weight, uint64_t cap, uint64_t* npts);

/* ---- stepping (engine.hpp:235-291, 318-375) ---------------------------- */
/* po_run_begin = initialize(); po_run_step advances one timestep exactly as
 * run() does (step 1 evolves on the m_init space, steps >= 2 call step()). */
int po_run_begin(const po_model* m, const po_run_cfg* cfg, po_run** out);
int po_run_step(po_run* r, po_diag* out);
int po_run_info(const po_run* r, uint64_t* rows, uint64_t* nnz, double* t, uint64_t* steps_done);
int po_run_state(const po_run* r, uint32_t* words, double* coeff);
int po_run_csr(const po_run* r, int64_t* row_ptr, int32_t* col, double* val);
/* ObservablesRow (engine.hpp:79-87, 299-311): density has lattice_sites entries */
int po_run_observe(const po_run* r, double* norm, double* energy, double* rmsd, double* xbar,
                   double* amp, double* density);
void po_run_destroy(po_run* r);

/* Whole trajectory through the implementation's own run() loop: n_diag
 * records are written (capacity cap); err receives the run's error string
 * ("" if none).  Final state via the returned po_run. */
int po_run_all(const po_model* m, const po_run_cfg* cfg, po_diag* diag, uint64_t cap,
               uint64_t* n_diag, po_run** final_out);

/* Phase timer for the CPU baseline: seconds spent in po_run_step split the
 * way SURVEY 3.5 splits them (only filled by implementations that can). */
typedef struct po_phase_times {
    double select, grow, remap, expectation, expmv, total;
    uint64_t spmv_nnz; /* sum over Taylor orders of nnz */
} po_phase_times;
int po_run_times(const po_run* r, po_phase_times* out); /* cumulative since begin */

#ifdef __cplusplus
}
#endif
#endif
