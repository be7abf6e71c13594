// engine.cuh -- host-side orchestration of the device-resident paces step: context, pooled device
// buffers, and one method per reference function on the hot path.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "../../include/paces_b200.h"
#include "host_model.hpp"
#include "kernels.cuh"
#include "window.cuh"
#include "incremental.cuh"
#include "sharded.cuh"
#include "taylor.cuh"
#include "nccl_comm.hpp"

namespace pb {

struct CudaFail : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ArgError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define PB_CUDA(call)                                                                                      \
    do {                                                                                                   \
        cudaError_t e_ = (call);                                                                           \
        if (e_ != cudaSuccess)                                                                             \
            throw pb::CudaFail(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + __FILE__ + ":" + \
                               std::to_string(__LINE__) + " (" #call ")");                                 \
    } while (0)

/// PACES_MAX_MEMORY_BYTES (common.hpp:30-49): 0 = unlimited; read on every call.
inline uint64_t memory_cap_bytes() {
    const char* env = std::getenv("PACES_MAX_MEMORY_BYTES");
    if (env == nullptr || *env == '\0') return 0;
    char* end = nullptr;
    unsigned long long v = std::strtoull(env, &end, 10);
    if (end == env) throw PacesError("PACES_MAX_MEMORY_BYTES is not a number: " + std::string(env));
    return uint64_t(v);
}
inline void require_memory(uint64_t bytes, const char* what) {
    const uint64_t cap = memory_cap_bytes();
    if (cap != 0 && bytes > cap)
        throw PacesError(std::string("memory cap exceeded: ") + what + " needs " + std::to_string(bytes) +
                         " bytes, PACES_MAX_MEMORY_BYTES=" + std::to_string(cap));
}

/// Grow-only device allocation; steady-state steps never call cudaMalloc.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    /// Contents are NOT preserved when the buffer grows.
    void ensure(size_t bytes) {
        if (bytes <= cap) return;
        size_t want = bytes + bytes / 4 + 256;
        if (p) cudaFree(p);  // implicit device synchronisation: nothing in flight still uses it
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, want);
        if (e != cudaSuccess) {
            cudaGetLastError();
            want = bytes;
            e = cudaMalloc(&p, want);
        }
        if (e != cudaSuccess) {
            p = nullptr;
            throw CudaFail(std::string("CUDA error: out of device memory allocating ") + std::to_string(bytes) +
                           " bytes: " + cudaGetErrorString(e));
        }
        cap = want;
    }
    /// Grows while preserving the first keep_bytes bytes.
    void ensure_keep(size_t bytes, size_t keep_bytes) {
        if (bytes <= cap) return;
        DevBuf bigger;
        bigger.ensure(bytes);
        if (p && keep_bytes) cudaMemcpy(bigger.p, p, keep_bytes, cudaMemcpyDeviceToDevice);
        swap(bigger);
    }
    void swap(DevBuf& o) {
        std::swap(p, o.p);
        std::swap(cap, o.cap);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

/// Slack behind row_ptr / col / val: the Taylor tile kernels fetch 16-byte-aligned slices with bulk copies, which may
/// read up to 15 bytes past the last element.
constexpr size_t CSR_PAD = 64;
constexpr int MAX_PEERS = 64;  // per-peer counters live in 64-entry shared-memory tables (sharded.cuh)

/// EffectiveSpace (subspace.hpp:76-82) on the device: sorted key table + CSR H_eff.
struct Space {
    DevBuf words;  // n x W uint32, canonical order
    uint32_t n = 0;
    DevBuf row_ptr;  // uint32[n+1]
    DevBuf col;      // int32[nnz] ascending per row
    DevBuf val;      // double[nnz]
    // value codes of a model-built H_eff (taylor.cuh, TaylorCodes; Engine::encode_values)
    DevBuf code;     // uint16[nnz]
    DevBuf diag;     // double[n], only when the model's diagonal elements are not tabulated
    bool has_code = false;
    // false: `val` was left behind by an incremental adapt step that carried the codes only (the Taylor tile kernels
    // do not read it); Engine::ensure_val() rebuilds it from the codes for whoever asks.  !val_valid implies has_code.
    bool val_valid = true;
    uint64_t nnz = 0;
    int max_row = 0;  // upper bound on the entries of a row (0 = unknown): selects the Taylor tile kernels
    uint64_t q_nom = 0;
    int order = 0;
    bool has_h = false;
    DevBuf full;  // uint8[n]: 1 = the row's whole neighbourhood is in the table (it was expanded), 0 = final frontier
    bool has_full = false;
    // sharded runs: columns >= n index the halo (values received from other ranks every SpMV)
    uint32_t halo_n = 0;
    uint32_t send_total = 0;
    DevBuf send_idx;                          // local rows to pack, grouped by destination rank
    std::vector<uint64_t> halo_send, halo_recv;  // per-peer element counts
    uint64_t n_global = 0, nnz_global = 0;
    // rows without / with halo columns (sharded SpMV: the former run while the halo is in flight)
    // (row-list form only -- row_lists; the tile kernels decide per row from the columns)
    uint32_t n_interior = 0, n_boundary = 0;
    DevBuf rows_int, rows_bnd;
    bool row_lists = false;
    // sharded assembly: the neighbour generator's move id of every CSR entry (the hint of the next step's assembly)
    DevBuf move;
    bool has_move = false;
};

struct Engine {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = true;
    std::string err;
    uint64_t launches = 0;

    bool has_model = false;
    HostModel hm;
    ModelDev md{};
    DevBuf d_eps, d_omega, d_g, d_nbs, d_nba, d_omega_n, d_diag_masks, d_vtab;
    bool use_codes = std::getenv("PB200_NO_VALUE_CODES") == nullptr && std::getenv("PB200_TAYLOR_ROWS") == nullptr;
    bool drop_val = std::getenv("PB200_KEEP_VALUES") == nullptr;  // coded spaces carry no 8-byte values between steps
    /// Makes sp.val current (decodes it from the value codes when an incremental step left it behind).
    void ensure_val(const Space& sp);
    int row_width = 1;  // max entries of an H_eff row for this model

    // resident trajectory
    Space space[2];
    int cur = 0;
    DevBuf coeff[2];
    int ccur = 0;
    bool has_state = false;
    double t = 0;
    uint64_t steps_done = 0;
    pb200_run_cfg cfg{};
    std::vector<uint32_t> cfg_occ;
    std::vector<double> cfg_amp;
    bool has_cfg = false;
    int last_order = 0;
    pb200_phase_times times{};

    // scratch
    DevBuf seeds;  // kept keys
    uint32_t n_seeds = 0;
    DevBuf tab_tmp, frontier[2], cand_keys, cand_gap, perm, seg_rank, gap, scan_tiles;
    DevBuf tmp_col, tmp_val, row_len;
    DevBuf weights, flag_keep, flag_tie, pos_a, idx_tmp, hist, sel_list, sort_out, sort_tmp;
    DevBuf term[2], partials, ctl;  // ctl: small device control block
    DevBuf aux_words, aux_coeff, aux2_words, aux2_coeff, aux_vec;  // staging for the host-buffer operators
    DevBuf flush;
    void* pinned = nullptr;  // 4 KiB pinned host scratch for read-backs
    void* mapped = nullptr;      // 4 KiB mapped pinned memory: [0] sequence flag, [64..] payload (read_back)
    void* mapped_dev = nullptr;  // its device address
    uint32_t rb_seq = 0;
    cudaEvent_t ev[10]{};
    // host-buffer step with overlapped transfers (pb200_step_io)
    cudaStream_t copy_stream = nullptr;
    cudaStream_t io_stream = nullptr;  // uploads + comparisons of a cached host-buffer step (beside everything else)
    cudaEvent_t ev_words = nullptr, ev_table = nullptr;
    bool pending_words = false;   // the key upload of the current step is still in flight on copy_stream
    struct StepIO {
        uint32_t* out_words = nullptr;
        double* out_coeff = nullptr;
        uint64_t out_cap_rows = 0;
        // The caller handed in the very state this context produced last (verified on the device, bit for bit):
        // the resident table, H_eff and expansion flags are used, so the step can take the incremental adapt path.
        // The comparison of the keys runs beside the step on the copy stream and is checked before the commit.
        bool cached = false;
        const uint32_t* mismatch = nullptr;  // two device flags written by the comparisons (coefficients, keys)
        // Enqueues the verification uploads + comparisons.  run_step calls it once the adapt phase is enqueued: that
        // phase is ~40 short kernels whose launches (command fetches over PCIe) crawl while 100 MB of upload
        // saturate the same link direction; the Taylor kernels behind it are long and enqueued ahead.
        mutable std::function<void()> start_upload;
        // Enqueues the two comparison kernels behind the uploads; run_step calls it with the event that marks the end
        // of the Taylor phase (they run while the coefficients travel to the host, on an otherwise idle GPU).
        mutable std::function<void(cudaEvent_t)> start_compare;
    };
    /// thrown by run_step when the deferred key comparison of a cached host-buffer step fails
    struct CacheMiss {};
    DevBuf io_flags;  // [0] coefficients differ, [1] keys differ
    const StepIO* io = nullptr;

    // multi-GPU (one context per rank); world == 1 is the single-GPU path
    int rank = 0, world = 1;
    bool sharded = false;          // the sharded algorithms are in use (world > 1, or a one-rank NCCL communicator)
    pb200_comm_ops ops{};
    NcclTransport* nccl = nullptr;  // owned: the in-library transport (pb200_ctx_set_comm_nccl)
    std::string comm_info;
    cudaStream_t halo_stream = nullptr;  // halo exchange beside the interior rows (ops.alltoallv_dev2)
    cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
    DevBuf row_class, scan_aligned;
    DevBuf out_keys, out_dest, route_pos, route_ctr, sendbuf, recvbuf, req_keys, req_dest, req_pos, reply, answer,
        found, halo_flag, tmp_cnt, tmp_move, halo_stage, sel_keys, sel_stage, asm_info;
    std::vector<uint64_t> h_send, h_recv;

    explicit Engine(int dev);
    ~Engine();

    // ---- collectives (thin wrappers over ops with error translation)
    void comm_check(int rc, const char* what) const {
        if (rc != 0) throw CudaFail(std::string("collective failed: ") + what);
    }
    double allreduce_host(double v) {
        comm_check(ops.allreduce_f64_host(ops.user, &v, 1), "allreduce_f64_host");
        return v;
    }
    uint64_t allreduce_host_u64(uint64_t v) {
        comm_check(ops.allreduce_u64_host(ops.user, &v, 1), "allreduce_u64_host");
        return v;
    }
    /// Routed exchange, device-side sizes.  route_async enqueues the bucketing of dest[0 .. *cnt_ptr) (a counter inside
    /// the route block's ShardCounters, clamped to cnt_bound) and the all-to-all of the per-peer counts; nothing returns
    /// to the host.  The caller scatters its payload by pos[] (same device count), then route_finish() is the ONE
    /// read-back of the exchange: shard counters + per-peer send / receive counts (-> h_send, h_recv), and
    /// exchange_known() moves the payload.  No blocking host collective, no stream synchronisation in between.
    RouteBlock* route_block();
    void route_async(const uint32_t* dest, const uint32_t* cnt_ptr, uint32_t cnt_bound, uint32_t* pos);
    ShardCounters route_finish();
    /// all-to-all-v of a bucketed device buffer with the per-peer counts in h_send / h_recv; returns the elements received
    uint64_t exchange_known(const void* send, DevBuf& recv, uint64_t elem_bytes);
    void halo_exchange(const Space& sp, double2* x);
    /// pack on the context's stream, exchange on the halo stream (when the transport has an independent channel);
    /// halo_wait() makes the context's stream wait for the arrival
    void halo_start(const Space& sp, double2* x);
    void halo_wait();
    void classify_rows(Space& sp);
    void grow_sharded(const uint32_t* d_seeds, uint32_t ns, int order, Space& out);
    /// hint != nullptr: the table grew incrementally from the previous space (sharded.cuh, AsmHint)
    void assemble_sharded(Space& sp, const AsmHint* hint = nullptr);
    /// incremental table growth on shards (sharded.cu); collective, false on every rank = take the full path
    /// (the coefficients are remapped into c_new on the way, discarded weight -> Ctl::out[0])
    bool grow_incremental_sharded(const Space& old, const double2* c_old, uint64_t kept_global, int m, Space& next,
                                  DevBuf& c_new);
    uint64_t last_kept_global = 0;  // rows select_sharded kept over all ranks
    /// compact = false: only the keep flags (flag_keep) are produced and 0 is returned; compact_kept_counted() gathers
    /// the kept keys later if the full expansion needs them
    uint32_t select_sharded(const uint32_t* d_words, const double2* d_c, uint32_t n, uint64_t q_nom, uint64_t seed,
                            double* norm2_out, bool compact = true);
    uint32_t compact_kept_counted(const uint32_t* d_words, uint32_t n);
    /// fuse_first (tile kernels only): the first order also yields <x|H|x>, |x|^2 and the non-finite count of the input
    /// state (*exp_out, *norm2_out; a non-finite coefficient throws) and takes that state from term[0], writing c only
    void expmv_sharded(const Space& sp, double2* c, double dt, double rtol, int max_order, int substeps,
                       int* order_used, double* last_term_norm, double* last_c_norm, bool fuse_first = false,
                       double* exp_out = nullptr, double* norm2_out = nullptr, double* discarded_out = nullptr);
    /// the sharded Taylor orders of sp run on the tile kernels (else: row lists)
    bool shard_tiles(const Space& sp) const { return taylor_tiles_usable(sp.max_row) && !sp.row_lists; }

    // ---- helpers
    int grid_for(uint64_t n) const {
        uint64_t g = (n + NT - 1) / NT;
        const uint64_t cap = uint64_t(sm_count) * 8;
        if (g > cap) g = cap;
        if (g < 1) g = 1;
        return int(g);
    }
    /// Rows per thread for the cursor kernels: long enough to amortise the first full search, short enough
    /// to keep ~3/4 of the machine's thread slots busy.
    uint32_t chunk_for(uint64_t n) const {
        const uint64_t slots = uint64_t(sm_count) * 1536;
        uint32_t c = 16;
        while (c > 2 && n / c < slots) c >>= 1;
        return c;
    }
    int grid_chunked(uint64_t n, uint32_t chunk) const {
        const uint64_t threads = (n + chunk - 1) / chunk;
        const uint64_t g = (threads + NT - 1) / NT;
        return int(g < 1 ? 1 : g);
    }
    void sync() { PB_CUDA(cudaStreamSynchronize(stream)); }
    void check_launch() {
        ++launches;
        PB_CUDA(cudaGetLastError());
    }
    /// Small device -> host read-back, stream-ordered.  A one-CTA kernel writes the words straight into mapped
    /// pinned host memory and raises a sequence flag behind a system-scope fence; the host spins on the flag.  No
    /// copy engine and no stream synchronisation: ~8 us instead of ~22 us idle, and it does not queue behind the
    /// large transfers of pb200_step_io (57-70 us, or the whole table download) -- tools/readback_probe.py.
    /// PB200_READBACK_MEMCPY=1 restores cudaMemcpyAsync + synchronize.
    template <class T>
    T read_back(const void* dptr) {
        static_assert(sizeof(T) % 4 == 0 && sizeof(T) <= 3584, "read_back: word-sized payloads up to 3.5 KiB");
        T v;
        if (!mapped) {
            PB_CUDA(cudaMemcpyAsync(pinned, dptr, sizeof(T), cudaMemcpyDeviceToHost, stream));
            sync();
            std::memcpy(&v, pinned, sizeof(T));
            return v;
        }
        publish(dptr, sizeof(T) / 4);
        std::memcpy(&v, static_cast<const char*>(mapped) + 64, sizeof(T));
        return v;
    }
    void publish(const void* dptr, uint32_t nwords);  // engine.cu
    void exclusive_scan(uint32_t* data, uint64_t n);  // in place over n elements
    bool rows_sorted_on_device(const uint32_t* table, uint32_t n);
    void require_model() const {
        if (!has_model) throw ArgError("no model set: call pb200_model_set first");
    }

    // ---- control block layout (device)
    struct Ctl {
        GrowCounters grow;
        TaylorCtl taylor;
        SelectCtl select;
        unsigned ticket;  // generic reduction ticket
        unsigned pad[3];
        double out[8];  // reduction outputs: [0] remap (discarded weight), [1..3] expectation, [4..] scratch
        uint32_t nnz;   // row_ptr[n] of the last assembly (read with the step's final read-back)
        uint32_t n_new; // unique new keys of the last merge (read together with the expansion counters)
        uint32_t code_fail;  // encode_csr_kernel met a value outside the model's table
        uint32_t pad2[1];
        // sharded Taylor orders: [0..3] / [4..7] deposits of the two launches of an order (rows without / with halo
        // columns), [8..10] / [11..13] the first order's <x|H|x>, |x|^2, #non-finite; all-reduced in place
        double tsum[16];
    };
    /// Snapshot of the control block taken by the last read-back of expmv(): the step's deferred scalars
    /// (discarded weight, <H>, norm, nnz) ride along instead of costing a stream synchronisation each.
    Ctl last_ctl{};
    // paired Taylor orders (kernels.cuh, TAYLOR_DEFER / TAYLOR_CATCHUP); PB200_NO_TAYLOR_DEFER=1 runs every order SINGLE
    bool taylor_defer = std::getenv("PB200_NO_TAYLOR_DEFER") == nullptr;
    bool defer_reads = false;  // run_step on one GPU: leave scalars on the device until the final read-back
    Ctl* dctl() const { return ctl.as<Ctl>(); }

    // ---- model
    void set_model(const HostModel& m);

    // ---- operators on device data
    void grow(const uint32_t* d_seeds, uint32_t n_seeds_, int order, Space& out);
    /// dedup + merge of the nc candidates of one BFS order into out.words (n rows); returns the number of new keys
    /// nc_bound >= the candidate count (which the kernels read from Ctl::grow.n_cand).  deferred: no read-back until
    /// the scatter is queued; the counters of the expansion come back through *counters.
    uint32_t merge_level(Space& out, uint32_t n, uint32_t nc_bound, int& fcur, bool deferred = false,
                         GrowCounters* counters = nullptr);
    void dedup_candidates_async(uint32_t n, uint32_t nc_bound);
    uint32_t dedup_candidates(uint32_t n, uint32_t nc_bound);  // returns the number of unique new keys
    void assemble(Space& sp);
    /// Enqueues the value-code pass over sp's CSR (n_ptr: row count on the device, or nullptr -> sp.n); a value outside
    /// the model's table raises *fail.  The caller sets sp.has_code once it has seen the flag.
    bool encode_values_async(Space& sp, uint64_t n_bound, uint64_t nnz_bound, const uint32_t* n_ptr, uint32_t* fail);
    /// the codes of sp for the Taylor launchers, or nullptr
    const TaylorCodes* codes_of(const Space& sp, TaylorCodes& tmp) const {
        if (!sp.has_code) return nullptr;
        tmp.code = sp.code.as<uint16_t>();
        tmp.diag = md.vt_diag ? nullptr : sp.diag.as<double>();
        tmp.vtab = md.vtab;
        tmp.vt_n = md.vt_n;
        return &tmp;
    }
    /// returns kept count; result in this->seeds
    uint32_t select(const uint32_t* d_words, const double2* d_c, uint32_t n, uint64_t q_nom, uint64_t seed,
                    double* norm2_out, bool compact = true);
    /// gathers the rows flagged in flag_keep into this->seeds (second half of select)
    void compact_kept(const uint32_t* d_words, uint32_t n, uint32_t kept);
    /// Incremental adapt (incremental.cuh): grows `next` from the previous space and the keep flags of select(),
    /// remaps the coefficients into c_new (discarded weight -> Ctl::out[0]).  Returns false when it had to bail out
    /// (a buffer bound was hit): the caller then runs the full path.
    bool grow_incremental(const Space& old, const double2* c_old, uint32_t kept, int m, Space& next, DevBuf& c_new);
    DevBuf inc_dist, inc_elist, inc_side_keys[2], inc_side_gap[2], inc_side_dist[2], inc_new_keys, inc_new_gap,
        inc_newidx, inc_inv, inc_side_newidx, inc_s_col, inc_s_val, inc_has_extra, inc_ctr, inc_simple, inc_buckets,
        inc_tile_disc, inc_tile_jlo, inc_xlist, inc_x_slot, inc_x_ref, inc_x_val, inc_s_code, inc_x_code, inc_row_len;
    uint64_t inc_steps = 0, inc_fallbacks = 0, inc_side_keys_total = 0, inc_expanded_total = 0;
    double remap(const uint32_t* src_words, const double2* src_c, uint32_t ns, const uint32_t* dst_words,
                 uint32_t nd, double2* dst_c);
    /// launches only: the discarded weight lands in Ctl::out[0]
    void remap_async(const uint32_t* src_words, const double2* src_c, uint32_t ns, const uint32_t* dst_words,
                     uint32_t nd, double2* dst_c);
    /// launches only: <x|H|x>, |x|^2, #non-finite land in Ctl::out[1..3]
    void expectation_async(const Space& sp, const double2* x);
    /// out: <x|H|x>, |x|^2; throws on non-finite input when check_finite
    void expectation(const Space& sp, const double2* x, double* exp_out, double* norm2_out, bool check_finite);
    /// fuse_expectation: the first order also writes <x|H|x>, |x|^2, #non-finite of the INPUT vector to Ctl::out[1..3]
    /// state_in_term0: the input state is in term[0] (not in c, which is then output only)
    void expmv(const Space& sp, double2* c, double dt, double rtol, int max_order, int substeps, int* order_used,
               double* last_term_norm, double* last_c_norm, bool fuse_expectation = false, bool state_in_term0 = false);
    void spmv(const Space& sp, const double2* x, double2* y);
    void upload_csr(Space& sp, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val);
    void observe(const uint32_t* words, const double2* c, uint32_t n, double* density, double* amp, double* phonons);

    /// weight_histogram (observables.hpp:123-176), entirely on the device (histogram.cuh); only the sampled curve and
    /// a 64-byte result block are downloaded
    DevBuf hist_counts, hist_tiles, hist_res, hist_curve;
    void weight_histogram(const double2* c, uint32_t n, uint64_t bins, pb200_weight_hist* out, uint64_t* rank,
                          double* weight, uint64_t cap, uint64_t* npts);

    // ---- resident trajectory
    void run_begin(const pb200_run_cfg& c);
    void run_step(pb200_diag* out);
};

}  // namespace pb
