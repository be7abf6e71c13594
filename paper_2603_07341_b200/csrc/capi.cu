// capi.cu -- the extern "C" surface declared in include/paces_b200.h.
#include <cmath>

#include "engine.cuh"

using namespace pb;

struct pb200_ctx {
    Engine eng;
    explicit pb200_ctx(int dev) : eng(dev) {}
};

namespace {
thread_local std::string g_create_err;

template <class F>
int guarded(pb200_ctx* ctx, F&& f) {
    if (ctx == nullptr) {
        g_create_err = "null context";
        return PB200_ERR_ARG;
    }
    try {
        cudaSetDevice(ctx->eng.device);
        f(ctx->eng);
        return PB200_OK;
    } catch (const PacesError& e) {
        ctx->eng.err = e.what();
        return PB200_ERR_PACES;
    } catch (const CudaFail& e) {
        ctx->eng.err = e.what();
        return PB200_ERR_CUDA;
    } catch (const ArgError& e) {
        ctx->eng.err = e.what();
        return PB200_ERR_ARG;
    } catch (const std::exception& e) {
        ctx->eng.err = e.what();
        return PB200_ERR_ARG;
    }
}

void need(bool ok, const char* what) {
    if (!ok) throw ArgError(what);
}

/// Uploads a sorted key table + coefficients into staging buffers.
void upload_state(Engine& e, DevBuf& dw, DevBuf& dc, const uint32_t* words, const double* coeff, uint64_t rows) {
    const size_t W = e.hm.W;
    need(rows <= 0x7fffffffull, "too many rows");
    dw.ensure(rows * W * 4 + 4);
    if (rows && words) PB_CUDA(cudaMemcpyAsync(dw.p, words, rows * W * 4, cudaMemcpyHostToDevice, e.stream));
    if (coeff) {
        dc.ensure(rows * 16 + 16);
        if (rows) PB_CUDA(cudaMemcpyAsync(dc.p, coeff, rows * 16, cudaMemcpyHostToDevice, e.stream));
    }
    e.sync();
}

void download_csr(Engine& e, const Space& sp, int64_t* row_ptr, int32_t* col, double* val) {
    need(sp.has_h, "no assembled H_eff resident");
    if (row_ptr) {
        std::vector<uint32_t> rp(size_t(sp.n) + 1);
        PB_CUDA(cudaMemcpyAsync(rp.data(), sp.row_ptr.p, rp.size() * 4, cudaMemcpyDeviceToHost, e.stream));
        e.sync();
        for (size_t i = 0; i < rp.size(); ++i) row_ptr[i] = int64_t(rp[i]);
    }
    if (col && sp.nnz) PB_CUDA(cudaMemcpyAsync(col, sp.col.p, sp.nnz * 4, cudaMemcpyDeviceToHost, e.stream));
    if (val && sp.nnz) {
        e.ensure_val(sp);
        PB_CUDA(cudaMemcpyAsync(val, sp.val.p, sp.nnz * 8, cudaMemcpyDeviceToHost, e.stream));
    }
    e.sync();
}
}  // namespace

extern "C" {

int pb200_ctx_create(int device, pb200_ctx** out) {
    if (!out) {
        g_create_err = "null output pointer";
        return PB200_ERR_ARG;
    }
    *out = nullptr;
    try {
        *out = new pb200_ctx(device);
        return PB200_OK;
    } catch (const CudaFail& e) {
        g_create_err = e.what();
        return PB200_ERR_CUDA;
    } catch (const std::exception& e) {
        g_create_err = e.what();
        return PB200_ERR_ARG;
    }
}

void pb200_ctx_destroy(pb200_ctx* ctx) { delete ctx; }

const char* pb200_last_error(const pb200_ctx* ctx) { return ctx ? ctx->eng.err.c_str() : g_create_err.c_str(); }

const char* pb200_version(void) { return "paces_b200 0.1 (sm_100a)"; }

int pb200_ctx_set_stream(pb200_ctx* ctx, void* cuda_stream) {
    return guarded(ctx, [&](Engine& e) {
        e.sync();
        if (e.own_stream && e.stream) cudaStreamDestroy(e.stream);
        e.stream = static_cast<cudaStream_t>(cuda_stream);
        e.own_stream = false;
    });
}

uint64_t pb200_kernel_launches(const pb200_ctx* ctx) { return ctx ? ctx->eng.launches : 0; }

uint64_t pb200_mix_seed(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

int pb200_ctx_set_comm(pb200_ctx* ctx, int rank, int world, const pb200_comm_ops* ops) {
    return guarded(ctx, [&](Engine& e) {
        // the routing kernels keep per-peer counters in 64-entry shared-memory tables (sharded.cuh)
        need(world >= 1 && world <= MAX_PEERS && rank >= 0 && rank < world, "set_comm: bad rank/world (world <= 64)");
        if (e.nccl) {
            e.sync();
            nccl_transport_destroy(e.nccl);
            e.nccl = nullptr;
        }
        if (world > 1) {
            need(ops && ops->allreduce_f64_host && ops->allreduce_u64_host && ops->alltoall_u64_host &&
                     ops->allgather_host && ops->alltoallv_dev && ops->allreduce_f64_dev && ops->allreduce_u32_dev,
                 "set_comm: every collective must be supplied when world > 1");
            e.ops = *ops;
        }
        e.rank = rank;
        e.world = world;
        e.sharded = world > 1;
        e.has_state = false;
    });
}

int pb200_nccl_unique_id(uint8_t* id) {
    if (!id) return PB200_ERR_ARG;
    try {
        nccl_make_unique_id(id);
        return PB200_OK;
    } catch (const std::exception& e) {
        g_create_err = e.what();
        return PB200_ERR_CUDA;
    }
}

int pb200_ctx_set_comm_nccl(pb200_ctx* ctx, int rank, int world, const uint8_t* id) {
    return guarded(ctx, [&](Engine& e) {
        need(id != nullptr, "set_comm_nccl: null id");
        need(world >= 1 && world <= MAX_PEERS && rank >= 0 && rank < world, "set_comm_nccl: bad rank/world (world <= 64)");
        e.sync();
        if (e.nccl) {
            nccl_transport_destroy(e.nccl);
            e.nccl = nullptr;
        }
        try {
            e.nccl = nccl_transport_create(e.device, rank, world, id, &e.stream);
        } catch (const std::exception& ex) {
            throw CudaFail(ex.what());
        }
        e.ops = nccl_transport_ops(e.nccl);
        e.rank = rank;
        e.world = world;
        // a one-rank communicator still runs the sharded algorithms (every exchange is a self-exchange): the
        // transport's self-test on a single GPU
        e.sharded = true;
        e.has_state = false;
    });
}

const char* pb200_comm_describe(pb200_ctx* ctx) {
    if (!ctx) return "";
    Engine& e = ctx->eng;
    e.comm_info = e.nccl ? nccl_transport_describe(e.nccl) : (e.sharded ? std::string("host-supplied callbacks") : std::string());
    return e.comm_info.c_str();
}

int pb200_owner_of(const pb200_ctx* ctx, const uint32_t* key, uint32_t world, uint32_t* owner) {
    if (!ctx || !ctx->eng.has_model || !key || !owner || world == 0) return PB200_ERR_ARG;
    *owner = host_owner(ctx->eng.hm, key, world);
    return PB200_OK;
}

// ---- model ---------------------------------------------------------------------------------------
int pb200_model_set(pb200_ctx* ctx, int kind, int ndim, const uint32_t* extents, const double* eps, int n_eps,
                    const double* hop, int n_hop, const double* omega, int n_omega, const double* g, int n_g,
                    uint32_t d_pho) {
    return guarded(ctx, [&](Engine& e) {
        HostModel m = build_host_model(kind, ndim, extents, eps, n_eps, hop, n_hop, omega, n_omega, g, n_g, d_pho);
        e.set_model(m);
    });
}

int pb200_model_info(const pb200_ctx* ctx, uint32_t* layout_sites, uint32_t* words_per_row, uint32_t* lattice_sites,
                     uint32_t* n_terms, uint32_t* total_bits) {
    if (!ctx || !ctx->eng.has_model) return PB200_ERR_ARG;
    const HostModel& m = ctx->eng.hm;
    if (layout_sites) *layout_sites = uint32_t(m.layout_sites());
    if (words_per_row) *words_per_row = m.W;
    if (lattice_sites) *lattice_sites = m.L;
    if (n_terms) *n_terms = m.n_terms;
    if (total_bits) *total_bits = m.total_bits;
    return PB200_OK;
}

int pb200_pack(const pb200_ctx* ctx, const uint32_t* occ, uint32_t* words) {
    return guarded(const_cast<pb200_ctx*>(ctx), [&](Engine& e) {
        e.require_model();
        host_pack(e.hm, occ, e.hm.layout_sites(), words);
    });
}

int pb200_unpack(const pb200_ctx* ctx, const uint32_t* words, uint32_t* occ) {
    return guarded(const_cast<pb200_ctx*>(ctx), [&](Engine& e) {
        e.require_model();
        host_unpack(e.hm, words, occ);
    });
}

int pb200_apply_terms(pb200_ctx* ctx, const uint32_t* keys, uint64_t n_keys, uint32_t* out_keys, double* out_amps,
                      int cap, int* count) {
    return guarded(ctx, [&](Engine& e) {
        e.require_model();
        need(keys && out_keys && out_amps && count && cap > 0, "apply_terms: bad arguments");
        const size_t W = e.hm.W;
        std::vector<uint32_t> occ(e.hm.layout_sites());
        for (uint64_t i = 0; i < n_keys; ++i) host_unpack(e.hm, keys + i * W, occ.data());  // validates the keys
        upload_state(e, e.aux_words, e.aux_coeff, keys, nullptr, n_keys);
        e.aux2_words.ensure(n_keys * cap * W * 4 + 4);
        e.aux2_coeff.ensure(n_keys * cap * 8 + 8);
        e.aux_vec.ensure(n_keys * 4 + 4);
        const int Wv = int(W);
        switch (Wv) {
#define PB_CASE(N)                                                                                                   \
    case N:                                                                                                          \
        apply_terms_kernel<N><<<e.grid_for(n_keys), NT, 0, e.stream>>>(e.md, e.aux_words.as<uint32_t>(),              \
                                                                       uint32_t(n_keys), cap,                        \
                                                                       e.aux2_words.as<uint32_t>(),                  \
                                                                       e.aux2_coeff.as<double>(), e.aux_vec.as<int>()); \
        break;
            PB_CASE(1) PB_CASE(2) PB_CASE(3) PB_CASE(4) PB_CASE(5) PB_CASE(6) PB_CASE(7) PB_CASE(8) PB_CASE(9)
            PB_CASE(10) PB_CASE(11) PB_CASE(12) PB_CASE(13) PB_CASE(14) PB_CASE(15) PB_CASE(16)
#undef PB_CASE
            default:
                throw PacesError("basis keys wider than 16 words are not supported by this build");
        }
        e.check_launch();
        PB_CUDA(cudaMemcpyAsync(out_keys, e.aux2_words.p, n_keys * cap * W * 4, cudaMemcpyDeviceToHost, e.stream));
        PB_CUDA(cudaMemcpyAsync(out_amps, e.aux2_coeff.p, n_keys * cap * 8, cudaMemcpyDeviceToHost, e.stream));
        PB_CUDA(cudaMemcpyAsync(count, e.aux_vec.p, n_keys * 4, cudaMemcpyDeviceToHost, e.stream));
        e.sync();
    });
}

// ---- stand-alone operators -----------------------------------------------------------------------
int pb200_grow(pb200_ctx* ctx, const uint32_t* seeds, uint64_t rows, int order, uint64_t* q_true, uint64_t* nnz) {
    return guarded(ctx, [&](Engine& e) {
        e.require_model();
        if (rows == 0) throw PacesError("grow_subspace: empty seed set");
        need(seeds != nullptr, "grow: null seeds");
        if (!host_rows_sorted(seeds, rows, e.hm.W)) throw PacesError("grow_subspace: seed keys must be sorted");
        if (order < 0) throw PacesError("grow_subspace: neighbor order must be >= 0");
        upload_state(e, e.aux_words, e.aux_coeff, seeds, nullptr, rows);
        e.has_state = false;  // the resident state no longer matches the current space
        Space& sp = e.space[e.cur];
        sp.has_h = false;
        sp.has_code = false;
        sp.val_valid = true;
        sp.has_full = false;
        e.grow(e.aux_words.as<uint32_t>(), uint32_t(rows), order, sp);
        e.sync();
        if (q_true) *q_true = sp.n;
        if (nnz) *nnz = sp.nnz;
    });
}

int pb200_space_info(const pb200_ctx* ctx, uint64_t* q_true, uint64_t* nnz, uint64_t* q_nom) {
    if (!ctx) return PB200_ERR_ARG;
    const Space& sp = ctx->eng.space[ctx->eng.cur];
    if (q_true) *q_true = sp.n;
    if (nnz) *nnz = sp.nnz;
    if (q_nom) *q_nom = sp.q_nom;
    return PB200_OK;
}

int pb200_space_get(pb200_ctx* ctx, uint32_t* words, int64_t* row_ptr, int32_t* col, double* val) {
    return guarded(ctx, [&](Engine& e) {
        const Space& sp = e.space[e.cur];
        if (words && sp.n)
            PB_CUDA(cudaMemcpyAsync(words, sp.words.p, size_t(sp.n) * e.hm.W * 4, cudaMemcpyDeviceToHost, e.stream));
        e.sync();
        download_csr(e, sp, row_ptr, col, val);
    });
}

int pb200_truncate_select(pb200_ctx* ctx, const uint32_t* words, const double* coeff, uint64_t rows, uint64_t q_nom,
                          uint64_t seed, uint32_t* out_words, uint64_t* kept) {
    return guarded(ctx, [&](Engine& e) {
        e.require_model();
        if (q_nom < 1) throw PacesError("truncate_select: q_nom must be >= 1");
        need(words && coeff && out_words, "truncate_select: null pointer");
        if (!host_rows_sorted(words, rows, e.hm.W)) throw PacesError("truncate_select: state table must be sorted");
        if (rows == 0) throw PacesError("truncate_select: state has no support");
        upload_state(e, e.aux_words, e.aux_coeff, words, coeff, rows);
        const uint32_t k = e.select(e.aux_words.as<uint32_t>(), e.aux_coeff.as<double2>(), uint32_t(rows), q_nom,
                                    seed, nullptr);
        if (k) PB_CUDA(cudaMemcpyAsync(out_words, e.seeds.p, size_t(k) * e.hm.W * 4, cudaMemcpyDeviceToHost, e.stream));
        e.sync();
        if (kept) *kept = k;
    });
}

int pb200_remap(pb200_ctx* ctx, const uint32_t* src_words, const double* src_coeff, uint64_t src_rows,
                const uint32_t* dst_words, uint64_t dst_rows, double* out_coeff, double* discarded) {
    return guarded(ctx, [&](Engine& e) {
        e.require_model();
        need(out_coeff != nullptr, "remap: null output");
        if (!host_rows_sorted(src_words, src_rows, e.hm.W)) throw PacesError("remap: state table must be sorted");
        upload_state(e, e.aux_words, e.aux_coeff, src_words, src_coeff, src_rows);
        upload_state(e, e.aux2_words, e.aux2_coeff, dst_words, nullptr, dst_rows);
        e.aux2_coeff.ensure(dst_rows * 16 + 16);
        const double d = e.remap(e.aux_words.as<uint32_t>(), e.aux_coeff.as<double2>(), uint32_t(src_rows),
                                 e.aux2_words.as<uint32_t>(), uint32_t(dst_rows), e.aux2_coeff.as<double2>());
        if (dst_rows) PB_CUDA(cudaMemcpyAsync(out_coeff, e.aux2_coeff.p, dst_rows * 16, cudaMemcpyDeviceToHost, e.stream));
        e.sync();
        if (discarded) *discarded = d;
    });
}

int pb200_csr_matvec(pb200_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                     const double* x, double* y) {
    return guarded(ctx, [&](Engine& e) {
        need(row_ptr && x && y, "csr_matvec: null pointer");
        Space tmp;
        e.upload_csr(tmp, n, row_ptr, col, val);
        e.aux_coeff.ensure(size_t(n) * 16 + 16);
        e.aux2_coeff.ensure(size_t(n) * 16 + 16);
        if (n) PB_CUDA(cudaMemcpyAsync(e.aux_coeff.p, x, size_t(n) * 16, cudaMemcpyHostToDevice, e.stream));
        e.spmv(tmp, e.aux_coeff.as<double2>(), e.aux2_coeff.as<double2>());
        if (n) PB_CUDA(cudaMemcpyAsync(y, e.aux2_coeff.p, size_t(n) * 16, cudaMemcpyDeviceToHost, e.stream));
        e.sync();
    });
}

int pb200_csr_expectation(pb200_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                          const double* x, double* out) {
    return guarded(ctx, [&](Engine& e) {
        need(row_ptr && x && out, "csr_expectation: null pointer");
        Space tmp;
        e.upload_csr(tmp, n, row_ptr, col, val);
        e.aux_coeff.ensure(size_t(n) * 16 + 16);
        if (n) PB_CUDA(cudaMemcpyAsync(e.aux_coeff.p, x, size_t(n) * 16, cudaMemcpyHostToDevice, e.stream));
        e.expectation(tmp, e.aux_coeff.as<double2>(), out, nullptr, false);
    });
}

int pb200_expmv(pb200_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val, double* c,
                double dt, double rtol, int max_order, int substeps, int* order_used, double* last_term_norm) {
    return guarded(ctx, [&](Engine& e) {
        need(row_ptr && c, "expmv: null pointer");
        // propagator.hpp:53-57: validate, dimension, finiteness
        if (!(dt > 0)) throw PacesError("propagator: dt must be > 0");
        if (!(rtol > 0) || !(rtol < 1)) throw PacesError("propagator: rtol must be in (0, 1)");
        if (max_order < 1) throw PacesError("propagator: max_order must be >= 1");
        if (substeps < 1) throw PacesError("propagator: substeps must be >= 1");
        for (int64_t i = 0; i < 2 * n; ++i)
            if (!std::isfinite(c[i])) throw PacesError("expmv: non-finite input coefficient");
        Space tmp;
        e.upload_csr(tmp, n, row_ptr, col, val);
        e.aux_coeff.ensure(size_t(n) * 16 + 16);
        if (n) PB_CUDA(cudaMemcpyAsync(e.aux_coeff.p, c, size_t(n) * 16, cudaMemcpyHostToDevice, e.stream));
        // a stand-alone operator must not disturb a resident run's batching heuristics, deferred scalars or counters
        struct Restore {
            Engine& e;
            int last_order;
            Engine::Ctl last_ctl;
            pb200_phase_times times;
            ~Restore() {
                e.last_order = last_order;
                e.last_ctl = last_ctl;
                e.times = times;
            }
        } restore{e, e.last_order, e.last_ctl, e.times};
        e.last_order = 0;
        e.expmv(tmp, e.aux_coeff.as<double2>(), dt, rtol, max_order, substeps, order_used, last_term_norm, nullptr);
        if (n) PB_CUDA(cudaMemcpyAsync(c, e.aux_coeff.p, size_t(n) * 16, cudaMemcpyDeviceToHost, e.stream));
        e.sync();
    });
}

int pb200_state_norm(pb200_ctx* ctx, const double* coeff, uint64_t rows, double* out) {
    return guarded(ctx, [&](Engine& e) {
        need(out != nullptr, "state_norm: null output");
        e.aux_coeff.ensure(rows * 16 + 16);
        e.weights.ensure(rows * 8 + 8);
        if (rows) PB_CUDA(cudaMemcpyAsync(e.aux_coeff.p, coeff, rows * 16, cudaMemcpyHostToDevice, e.stream));
        Engine::Ctl* c = e.dctl();
        PB_CUDA(cudaMemsetAsync(&c->select, 0, sizeof(SelectCtl), e.stream));
        weights_kernel<<<e.grid_for(rows), NT, 0, e.stream>>>(e.aux_coeff.as<double2>(), uint32_t(rows),
                                                              e.weights.as<double>(), e.partials.as<double>(),
                                                              &c->select);
        e.check_launch();
        SelectCtl sc = e.read_back<SelectCtl>(&c->select);
        *out = std::sqrt(sc.norm2);
    });
}

int pb200_exciton_density(pb200_ctx* ctx, const uint32_t* words, const double* coeff, uint64_t rows, double* p) {
    return guarded(ctx, [&](Engine& e) {
        e.require_model();
        upload_state(e, e.aux_words, e.aux_coeff, words, coeff, rows);
        e.observe(e.aux_words.as<uint32_t>(), e.aux_coeff.as<double2>(), uint32_t(rows), p, nullptr, nullptr);
    });
}

int pb200_dipole_amplitude(pb200_ctx* ctx, const uint32_t* words, const double* coeff, uint64_t rows, double* amp) {
    return guarded(ctx, [&](Engine& e) {
        e.require_model();
        upload_state(e, e.aux_words, e.aux_coeff, words, coeff, rows);
        e.observe(e.aux_words.as<uint32_t>(), e.aux_coeff.as<double2>(), uint32_t(rows), nullptr, amp, nullptr);
    });
}

int pb200_phonon_numbers(pb200_ctx* ctx, const uint32_t* words, const double* coeff, uint64_t rows, double* n_out) {
    return guarded(ctx, [&](Engine& e) {
        e.require_model();
        upload_state(e, e.aux_words, e.aux_coeff, words, coeff, rows);
        e.observe(e.aux_words.as<uint32_t>(), e.aux_coeff.as<double2>(), uint32_t(rows), nullptr, nullptr, n_out);
    });
}

int pb200_weight_histogram(pb200_ctx* ctx, const double* coeff, uint64_t rows, uint64_t bins, pb200_weight_hist* out,
                           uint64_t* rank, double* weight, uint64_t cap, uint64_t* npts) {
    return guarded(ctx, [&](Engine& e) {
        need(coeff && out, "weight_histogram: null pointer");
        if (rows == 0) throw PacesError("weight histogram: empty state");
        if (rows > 0x7fffffffull) throw ArgError("weight_histogram: too many rows");
        e.aux_coeff.ensure(rows * 16 + 16);
        PB_CUDA(cudaMemcpyAsync(e.aux_coeff.p, coeff, rows * 16, cudaMemcpyHostToDevice, e.stream));
        e.weight_histogram(e.aux_coeff.as<double2>(), uint32_t(rows), bins, out, rank, weight, cap, npts);
    });
}

int pb200_run_weight_histogram(pb200_ctx* ctx, uint64_t bins, pb200_weight_hist* out, uint64_t* rank, double* weight,
                               uint64_t cap, uint64_t* npts) {
    return guarded(ctx, [&](Engine& e) {
        need(out != nullptr, "run_weight_histogram: null pointer");
        if (!e.has_state) throw ArgError("no resident run: call pb200_run_begin first");
        if (e.sharded) throw ArgError("run_weight_histogram: gather the shards first (single-GPU operator)");
        e.weight_histogram(e.coeff[e.ccur].as<double2>(), e.space[e.cur].n, bins, out, rank, weight, cap, npts);
    });
}

// ---- resident trajectory -------------------------------------------------------------------------
int pb200_run_begin(pb200_ctx* ctx, const pb200_run_cfg* cfg) {
    return guarded(ctx, [&](Engine& e) {
        need(cfg != nullptr, "run_begin: null config");
        e.run_begin(*cfg);
    });
}

int pb200_run_step(pb200_ctx* ctx, pb200_diag* out) {
    return guarded(ctx, [&](Engine& e) { e.run_step(out); });
}

int pb200_run_info(const pb200_ctx* ctx, uint64_t* rows, uint64_t* nnz, double* t, uint64_t* steps_done) {
    if (!ctx || !ctx->eng.has_state) return PB200_ERR_ARG;
    const Engine& e = ctx->eng;
    const Space& sp = e.space[e.cur];
    if (rows) *rows = sp.n;
    if (nnz) *nnz = sp.nnz;
    if (t) *t = e.t;
    if (steps_done) *steps_done = e.steps_done;
    return PB200_OK;
}

int pb200_run_global(const pb200_ctx* ctx, uint64_t* rows_global, uint64_t* nnz_global) {
    if (!ctx || !ctx->eng.has_state) return PB200_ERR_ARG;
    const Engine& e = ctx->eng;
    const Space& sp = e.space[e.cur];
    if (rows_global) *rows_global = e.sharded ? sp.n_global : sp.n;
    if (nnz_global) *nnz_global = e.sharded ? sp.nnz_global : sp.nnz;
    return PB200_OK;
}

int pb200_run_state(pb200_ctx* ctx, uint32_t* words, double* coeff) {
    return guarded(ctx, [&](Engine& e) {
        need(e.has_state, "no resident state");
        const Space& sp = e.space[e.cur];
        if (words && sp.n)
            PB_CUDA(cudaMemcpyAsync(words, sp.words.p, size_t(sp.n) * e.hm.W * 4, cudaMemcpyDeviceToHost, e.stream));
        if (coeff && sp.n)
            PB_CUDA(cudaMemcpyAsync(coeff, e.coeff[e.ccur].p, size_t(sp.n) * 16, cudaMemcpyDeviceToHost, e.stream));
        e.sync();
    });
}

int pb200_run_csr(pb200_ctx* ctx, int64_t* row_ptr, int32_t* col, double* val) {
    return guarded(ctx, [&](Engine& e) {
        need(e.has_state, "no resident state");
        // sharded: this is the rank-local CSR block; columns >= local rows index the halo
        download_csr(e, e.space[e.cur], row_ptr, col, val);
    });
}

int pb200_run_load_state(pb200_ctx* ctx, const pb200_run_cfg* cfg, const uint32_t* words, const double* coeff,
                         uint64_t rows, double t, uint64_t steps_done) {
    return guarded(ctx, [&](Engine& e) {
        e.require_model();
        need(cfg && words && coeff && rows > 0, "run_load_state: bad arguments");
        if (!host_rows_sorted(words, rows, e.hm.W)) throw PacesError("load_state: state table must be sorted");
        pb200_run_cfg c = *cfg;
        c.init_kind = 0;  // the seed description is irrelevant from here on
        c.n_entries = 0;
        c.entry_occ = nullptr;
        c.entry_amp = nullptr;
        e.cfg = c;
        e.has_cfg = true;
        e.has_state = false;
        upload_state(e, e.aux_words, e.aux_coeff, words, coeff, rows);
        Space& sp = e.space[e.cur];
        e.grow(e.aux_words.as<uint32_t>(), uint32_t(rows), 0, sp);  // table as is; H_eff over it
        e.coeff[e.ccur].ensure(rows * 16 + 16);
        PB_CUDA(cudaMemcpyAsync(e.coeff[e.ccur].p, e.aux_coeff.p, rows * 16, cudaMemcpyDeviceToDevice, e.stream));
        e.sync();
        e.t = t;
        e.steps_done = steps_done;
        e.last_order = 0;
        e.has_state = true;
        e.times = pb200_phase_times{};
    });
}

int pb200_step(pb200_ctx* ctx, const pb200_run_cfg* cfg, uint64_t step_index, const uint32_t* words,
               const double* coeff, uint64_t rows, double t, pb200_diag* out, uint64_t* rows_out, uint64_t* nnz_out) {
    return guarded(ctx, [&](Engine& e) {
        e.require_model();
        need(cfg && words && coeff, "step: null pointer");
        need(step_index >= 2, "step: step_index must be >= 2 (step 1 evolves on the initial space, use pb200_run_*)");
        if (rows == 0) throw PacesError("truncate_select: state has no support");
        need(rows <= 0x7fffffffull, "too many rows");
        pb200_run_cfg c = *cfg;
        c.init_kind = 0;
        c.n_entries = 0;
        c.entry_occ = nullptr;
        c.entry_amp = nullptr;
        e.cfg = c;
        e.has_cfg = true;
        e.has_state = false;
        Space& sp = e.space[e.cur];
        const size_t W = e.hm.W;
        sp.words.ensure(rows * W * 4 + 4);
        e.coeff[e.ccur].ensure(rows * 16 + 16);
        PB_CUDA(cudaMemcpyAsync(sp.words.p, words, rows * W * 4, cudaMemcpyHostToDevice, e.stream));
        PB_CUDA(cudaMemcpyAsync(e.coeff[e.ccur].p, coeff, rows * 16, cudaMemcpyHostToDevice, e.stream));
        sp.n = uint32_t(rows);
        sp.nnz = 0;
        sp.has_h = false;
        sp.has_code = false;
        sp.val_valid = true;
        sp.has_full = false;
        // engine.hpp:110: the caller's table must be sorted -- checked on the device copy (one streaming kernel)
        if (!e.rows_sorted_on_device(sp.words.as<uint32_t>(), sp.n))
            throw PacesError("truncate_select: state table must be sorted");
        e.t = t;
        e.steps_done = step_index - 1;
        e.has_state = true;
        e.run_step(out);
        const Space& nsp = e.space[e.cur];
        if (rows_out) *rows_out = nsp.n;
        if (nnz_out) *nnz_out = nsp.nnz;
    });
}

int pb200_step_io(pb200_ctx* ctx, const pb200_run_cfg* cfg, uint64_t step_index, const uint32_t* words,
                  const double* coeff, uint64_t rows, double t, uint32_t* out_words, double* out_coeff,
                  uint64_t out_cap_rows, pb200_diag* out, uint64_t* rows_out, uint64_t* nnz_out) {
    return guarded(ctx, [&](Engine& e) {
        e.require_model();
        need(cfg && words && coeff && out_words && out_coeff, "step_io: null pointer");
        need(step_index >= 2, "step: step_index must be >= 2 (step 1 evolves on the initial space, use pb200_run_*)");
        if (rows == 0) throw PacesError("truncate_select: state has no support");
        need(rows <= 0x7fffffffull, "too many rows");
        pb200_run_cfg c = *cfg;
        c.init_kind = 0;
        c.n_entries = 0;
        c.entry_occ = nullptr;
        c.entry_amp = nullptr;
        const size_t W = e.hm.W;
        {
            // The input buffers are still being read (verification uploads, a redo after a cache miss) while the
            // outputs are written: in-place calls are not supported.
            auto overlap = [](const void* a, size_t na, const void* b, size_t nb) {
                const char* pa = static_cast<const char*>(a);
                const char* pb_ = static_cast<const char*>(b);
                return na != 0 && nb != 0 && pa < pb_ + nb && pb_ < pa + na;
            };
            const size_t in_w = rows * W * 4, in_c = rows * 16, out_w = out_cap_rows * W * 4, out_c = out_cap_rows * 16;
            need(!overlap(words, in_w, out_words, out_w) && !overlap(words, in_w, out_coeff, out_c) &&
                     !overlap(coeff, in_c, out_words, out_w) && !overlap(coeff, in_c, out_coeff, out_c),
                 "step_io: input and output buffers must not overlap (use two buffer sets and alternate)");
        }
        Engine::StepIO io;
        io.out_words = out_words;
        io.out_coeff = out_coeff;
        io.out_cap_rows = out_cap_rows;
        struct Guard {
            Engine& e;
            ~Guard() {
                e.io = nullptr;
                e.pending_words = false;
                cudaStreamSynchronize(e.copy_stream);  // never leave a transfer into caller memory in flight
                cudaStreamSynchronize(e.io_stream);
            }
        } guard{e};

        // ---- Is this the state the context produced last?  Same step, same time, same run parameters and (checked on
        // the device, bit for bit) the same coefficients and keys: then the resident table, H_eff and expansion flags
        // are exactly the caller's EffectiveSpace and the step takes the incremental adapt path.  Everything is still
        // uploaded -- the comparison needs it -- but the keys no longer sit on the critical path: their upload and
        // comparison run on the copy stream beside the step and are checked before anything is committed.
        const Space& res = e.space[e.cur];
        const bool candidate = !e.sharded && e.has_state && e.has_cfg && res.has_h && res.has_full && res.n == rows &&
                               e.steps_done + 1 == step_index && e.t == t && e.cfg.m == c.m && e.cfg.q_nom == c.q_nom &&
                               e.cfg.dt == c.dt && e.cfg.rtol == c.rtol && e.cfg.max_order == c.max_order &&
                               e.cfg.substeps == c.substeps && e.cfg.seed == c.seed &&
                               std::getenv("PB200_NO_STEP_CACHE") == nullptr;
        if (candidate) {
            e.io_flags.ensure(16);
            uint32_t* flags = e.io_flags.as<uint32_t>();
            e.aux_coeff.ensure(rows * 16 + 16);
            e.aux_words.ensure(rows * W * 4 + 16);
            // both uploads and comparisons on their own stream: the step itself starts at once on the resident data
            e.sync();  // the resident buffers they read are final
            // uploads first, both on the io stream; the two comparison kernels follow once the Taylor phase is enqueued
            // and wait for its end: the GPU is idle then (the coefficient download is the critical path), while beside
            // the Taylor launches they would take SM slots from the persistent tile kernels
            // PB200_EARLY_COEFF_UPLOAD=1: both uploads beside the step (the round-2 v1 behaviour); default: only the keys
            // travel beside the step, the coefficients go up while the result's coefficients come down (the link is full
            // duplex and the GPU idle), so the Taylor phase shares the device with less DMA traffic
            static const bool early_coeff = std::getenv("PB200_EARLY_COEFF_UPLOAD") != nullptr;
            auto upload = [&e, flags, coeff, words, rows, W]() {
                PB_CUDA(cudaMemsetAsync(flags, 0, 8, e.io_stream));
                if (early_coeff)
                    PB_CUDA(cudaMemcpyAsync(e.aux_coeff.p, coeff, rows * 16, cudaMemcpyHostToDevice, e.io_stream));
                PB_CUDA(cudaMemcpyAsync(e.aux_words.p, words, rows * W * 4, cudaMemcpyHostToDevice, e.io_stream));
            };
            const uint32_t* res_words = res.words.as<uint32_t>();
            const uint32_t* res_coeff = e.coeff[e.ccur].as<uint32_t>();
            auto compare = [&e, flags, coeff, rows, W, res_words, res_coeff](cudaEvent_t after) {
                if (after) PB_CUDA(cudaStreamWaitEvent(e.io_stream, after, 0));
                if (!early_coeff)
                    PB_CUDA(cudaMemcpyAsync(e.aux_coeff.p, coeff, rows * 16, cudaMemcpyHostToDevice, e.io_stream));
                words_differ_kernel<<<e.grid_for(rows * 4), NT, 0, e.io_stream>>>(e.aux_coeff.as<uint32_t>(), res_coeff,
                                                                                  rows * 4, flags);
                e.check_launch();
                words_differ_kernel<<<e.grid_for(rows * W), NT, 0, e.io_stream>>>(e.aux_words.as<uint32_t>(), res_words,
                                                                                  rows * W, flags + 1);
                e.check_launch();
            };
            if (std::getenv("PB200_EAGER_UPLOAD")) {
                upload();
                compare(nullptr);
            } else {
                io.start_upload = upload;
                io.start_compare = compare;
            }
            {
                const pb200_run_cfg saved = e.cfg;
                e.cfg = c;
                io.cached = true;
                io.mismatch = flags;
                e.io = &io;
                try {
                    e.run_step(out);
                    const Space& nsp = e.space[e.cur];
                    if (rows_out) *rows_out = nsp.n;
                    if (nnz_out) *nnz_out = nsp.nnz;
                    return;
                } catch (const Engine::CacheMiss&) {
                    // not the resident state after all: redo the step from the caller's buffers
                } catch (...) {
                    cudaStreamSynchronize(e.io_stream);
                    e.cfg = saved;
                    throw;
                }
                e.cfg = saved;
                e.io = nullptr;
                io.cached = false;
                io.mismatch = nullptr;
            }
            PB_CUDA(cudaStreamSynchronize(e.io_stream));
            PB_CUDA(cudaStreamSynchronize(e.copy_stream));
        }

        e.cfg = c;
        e.has_cfg = true;
        e.has_state = false;
        Space& sp = e.space[e.cur];
        sp.words.ensure(rows * W * 4 + 4);
        e.coeff[e.ccur].ensure(rows * 16 + 16);
        // coefficients first on the compute stream (the weight / selection kernels need only them); the keys travel
        // on the copy stream and are awaited right before the compaction of the kept rows
        PB_CUDA(cudaMemcpyAsync(e.coeff[e.ccur].p, coeff, rows * 16, cudaMemcpyHostToDevice, e.stream));
        // both uploads share one PCIe direction: let the coefficients through first, then the keys
        PB_CUDA(cudaEventRecord(e.ev_table, e.stream));
        PB_CUDA(cudaStreamWaitEvent(e.copy_stream, e.ev_table, 0));
        PB_CUDA(cudaMemcpyAsync(sp.words.p, words, rows * W * 4, cudaMemcpyHostToDevice, e.copy_stream));
        PB_CUDA(cudaEventRecord(e.ev_words, e.copy_stream));
        e.pending_words = true;
        sp.n = uint32_t(rows);
        sp.nnz = 0;
        sp.has_h = false;
        sp.has_code = false;
        sp.val_valid = true;
        sp.has_full = false;
        e.t = t;
        e.steps_done = step_index - 1;
        e.has_state = true;
        e.io = &io;
        e.run_step(out);
        const Space& nsp = e.space[e.cur];
        if (rows_out) *rows_out = nsp.n;
        if (nnz_out) *nnz_out = nsp.nnz;
    });
}

int pb200_run_observe(pb200_ctx* ctx, double* norm, double* energy, double* rmsd, double* xbar, double* amp,
                      double* density) {
    return guarded(ctx, [&](Engine& e) {
        need(e.has_state, "no resident state");
        const Space& sp = e.space[e.cur];
        const HostModel& m = e.hm;
        const double2* c = e.coeff[e.ccur].as<double2>();
        double ex = 0, n2 = 0;
        e.expectation(sp, c, &ex, &n2, false);
        const double nrm = std::sqrt(n2);
        if (norm) *norm = nrm;
        // energy(): <psi|H|psi> / pow(norm, 2) (observables.hpp:75-81)
        const double nn = std::pow(nrm, 2);
        if (nn == 0.0) throw PacesError("energy: zero-norm state");
        if (energy) *energy = ex / nn;
        std::vector<double> p(m.L, 0.0);
        double a[2] = {0, 0};
        e.observe(sp.words.as<uint32_t>(), c, sp.n, p.data(), a, nullptr);
        if (density) std::copy(p.begin(), p.end(), density);
        if (amp) {
            amp[0] = a[0];
            amp[1] = a[1];
        }
        // mean_position / rmsd (observables.hpp:41-70): O(L) host post-processing of the density
        if (xbar) {
            double acc = 0;
            for (size_t i = 0; i < p.size(); ++i) acc += double(i) * p[i];
            *xbar = acc;
        }
        if (rmsd) {
            double wsum = 0;
            double mean[3] = {0, 0, 0};
            auto coords = [&](uint32_t idx, uint32_t* cc) {
                cc[0] = idx % m.extents[0];
                cc[1] = (idx / m.extents[0]) % m.extents[1];
                cc[2] = idx / (m.extents[0] * m.extents[1]);
            };
            for (uint32_t i = 0; i < p.size(); ++i) {
                uint32_t cc[3];
                coords(i, cc);
                wsum += p[i];
                for (int k = 0; k < 3; ++k) mean[k] += p[i] * double(cc[k]);
            }
            if (wsum <= 0) throw PacesError("rmsd: zero-norm state");
            for (int k = 0; k < 3; ++k) mean[k] /= wsum;
            double var = 0;
            for (uint32_t i = 0; i < p.size(); ++i) {
                uint32_t cc[3];
                coords(i, cc);
                double r2 = 0;
                for (int k = 0; k < 3; ++k) {
                    const double dx = double(cc[k]) - mean[k];
                    r2 += dx * dx;
                }
                var += (p[i] / wsum) * r2;
            }
            *rmsd = std::sqrt(var);
        }
    });
}

int pb200_run_times(const pb200_ctx* ctx, pb200_phase_times* out) {
    if (!ctx || !out) return PB200_ERR_ARG;
    *out = ctx->eng.times;
    return PB200_OK;
}

int pb200_run_adapt_stats(const pb200_ctx* ctx, pb200_adapt_stats* out) {
    if (!ctx || !out) return PB200_ERR_ARG;
    const Engine& e = ctx->eng;
    out->incremental_steps = e.inc_steps;
    out->fallbacks = e.inc_fallbacks;
    out->expanded_rows = e.inc_expanded_total;
    out->side_keys = e.inc_side_keys_total;
    return PB200_OK;
}

int pb200_run_reset_times(pb200_ctx* ctx) {
    if (!ctx) return PB200_ERR_ARG;
    ctx->eng.times = pb200_phase_times{};
    return PB200_OK;
}

// ---- measurement helpers -------------------------------------------------------------------------
static void flush_l2(Engine& e) {
    const size_t bytes = size_t(256) << 20;  // 256 MiB > 126 MB L2
    e.flush.ensure(bytes);
    flush_kernel<<<e.sm_count * 8, 256, 0, e.stream>>>(e.flush.as<double>(), bytes / 8);
    e.check_launch();
}

int pb200_bench_taylor(pb200_ctx* ctx, int orders, int flush, double dt, double* ms_per_order, uint64_t* nnz,
                       uint64_t* rows) {
    return guarded(ctx, [&](Engine& e) {
        need(e.has_state && orders > 0, "bench_taylor: no resident state");
        need(!e.sharded, "bench_taylor: single-GPU spaces only (a shard's gathers need the halo)");
        const Space& sp = e.space[e.cur];
        const uint32_t n = sp.n;
        Engine::Ctl* c = e.dctl();
        e.term[0].ensure(size_t(n) * 16 + 16);
        e.term[1].ensure(size_t(n) * 16 + 16);
        e.aux_coeff.ensure(size_t(n) * 16 + 16);
        // work on a copy so the resident state is untouched
        PB_CUDA(cudaMemcpyAsync(e.aux_coeff.p, e.coeff[e.ccur].p, size_t(n) * 16, cudaMemcpyDeviceToDevice, e.stream));
        PB_CUDA(cudaMemcpyAsync(e.term[0].p, e.coeff[e.ccur].p, size_t(n) * 16, cudaMemcpyDeviceToDevice, e.stream));
        PB_CUDA(cudaMemsetAsync(&c->taylor, 0, sizeof(TaylorCtl), e.stream));
        double total = 0;
        TaylorCodes codes_tmp;
        const TaylorCodes* cd = e.codes_of(sp, codes_tmp);
        for (int o = 1; o <= orders; ++o) {
            if (flush) flush_l2(e);
            PB_CUDA(cudaEventRecord(e.ev[8], e.stream));
            taylor_launch_single(false, e.grid_for(n), e.sm_count, e.stream, n, sp.row_ptr.as<uint32_t>(),
                                 sp.col.as<int32_t>(), sp.val.as<double>(), e.term[(o - 1) & 1].as<double2>(),
                                 e.term[o & 1].as<double2>(), e.aux_coeff.as<double2>(), -dt / double(o), o, 1e-15,
                                 e.partials.as<double>(), &c->taylor, 1, nullptr, nullptr, sp.max_row, cd);
            e.check_launch();
            PB_CUDA(cudaEventRecord(e.ev[9], e.stream));
            e.sync();
            float ms = 0;
            PB_CUDA(cudaEventElapsedTime(&ms, e.ev[8], e.ev[9]));
            total += ms;
        }
        if (ms_per_order) *ms_per_order = total / orders;
        if (nnz) *nnz = sp.nnz;
        if (rows) *rows = n;
    });
}

int pb200_bench_spmv(pb200_ctx* ctx, int reps, int flush, double* ms_per_spmv) {
    return guarded(ctx, [&](Engine& e) {
        need(e.has_state && reps > 0, "bench_spmv: no resident state");
        need(!e.sharded, "bench_spmv: single-GPU spaces only (a shard's gathers need the halo)");
        const Space& sp = e.space[e.cur];
        const uint32_t n = sp.n;
        e.aux_coeff.ensure(size_t(n) * 16 + 16);
        double total = 0;
        for (int r = 0; r < reps; ++r) {
            if (flush) flush_l2(e);
            PB_CUDA(cudaEventRecord(e.ev[8], e.stream));
            e.spmv(sp, e.coeff[e.ccur].as<double2>(), e.aux_coeff.as<double2>());
            PB_CUDA(cudaEventRecord(e.ev[9], e.stream));
            e.sync();
            float ms = 0;
            PB_CUDA(cudaEventElapsedTime(&ms, e.ev[8], e.ev[9]));
            total += ms;
        }
        if (ms_per_spmv) *ms_per_spmv = total / reps;
    });
}

}  // extern "C"
