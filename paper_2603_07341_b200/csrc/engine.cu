// engine.cu -- implementation of the device-resident paces step (see engine.cuh, kernels.cuh).
#include <atomic>
#include <chrono>
#include "engine.cuh"

#include <cmath>

namespace pb {

#ifdef PB_ONLY_W  // development / profiling builds: one key width, small module, fast compile
#define PB_DISPATCH_W(Wv, ...)                                  \
    switch (Wv) {                                               \
        case PB_ONLY_W: { constexpr int W = PB_ONLY_W; __VA_ARGS__; } break; \
        default: throw PacesError("this development build only supports one key width (PB_ONLY_W)"); \
    }
#else
#define PB_DISPATCH_W(Wv, ...)                                  \
    switch (Wv) {                                               \
        case 1: { constexpr int W = 1; __VA_ARGS__; } break;    \
        case 2: { constexpr int W = 2; __VA_ARGS__; } break;    \
        case 3: { constexpr int W = 3; __VA_ARGS__; } break;    \
        case 4: { constexpr int W = 4; __VA_ARGS__; } break;    \
        case 5: { constexpr int W = 5; __VA_ARGS__; } break;    \
        case 6: { constexpr int W = 6; __VA_ARGS__; } break;    \
        case 7: { constexpr int W = 7; __VA_ARGS__; } break;    \
        case 8: { constexpr int W = 8; __VA_ARGS__; } break;    \
        case 9: { constexpr int W = 9; __VA_ARGS__; } break;    \
        case 10: { constexpr int W = 10; __VA_ARGS__; } break;  \
        case 11: { constexpr int W = 11; __VA_ARGS__; } break;  \
        case 12: { constexpr int W = 12; __VA_ARGS__; } break;  \
        case 13: { constexpr int W = 13; __VA_ARGS__; } break;  \
        case 14: { constexpr int W = 14; __VA_ARGS__; } break;  \
        case 15: { constexpr int W = 15; __VA_ARGS__; } break;  \
        case 16: { constexpr int W = 16; __VA_ARGS__; } break;  \
        default: throw PacesError("basis keys wider than 16 words (512 bits) are not supported by this build"); \
    }
#endif

// ------------------------------------------------------------------------------------------------
Engine::Engine(int dev) : device(dev) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        throw CudaFail(std::string("no CUDA device visible (") + cudaGetErrorString(e) +
                       "); paces_b200 has no CPU fallback");
    if (dev < 0 || dev >= count) throw ArgError("device index out of range");
    PB_CUDA(cudaSetDevice(dev));
    cudaDeviceProp prop{};
    PB_CUDA(cudaGetDeviceProperties(&prop, dev));
    if (prop.major < 10)
        throw CudaFail(std::string("device ") + prop.name + " is sm_" + std::to_string(prop.major) +
                       std::to_string(prop.minor) + "; this library is built for sm_100a (B200) only");
    sm_count = prop.multiProcessorCount;
    PB_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    PB_CUDA(cudaMallocHost(&pinned, 4096));
    if (std::getenv("PB200_READBACK_MEMCPY") == nullptr) {
        PB_CUDA(cudaHostAlloc(&mapped, 4096, cudaHostAllocMapped));
        std::memset(mapped, 0, 4096);
        PB_CUDA(cudaHostGetDevicePointer(&mapped_dev, mapped, 0));
    }
    for (auto& x : ev) PB_CUDA(cudaEventCreate(&x));
    PB_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    PB_CUDA(cudaStreamCreateWithFlags(&io_stream, cudaStreamNonBlocking));
    {
        // highest priority: the transport's kernels of a halo exchange must get SM slots beside the Taylor launch that
        // is meant to hide them, not behind it
        int prio_lo = 0, prio_hi = 0;
        PB_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        PB_CUDA(cudaStreamCreateWithPriority(&halo_stream, cudaStreamNonBlocking, prio_hi));
    }
    PB_CUDA(cudaEventCreateWithFlags(&ev_pack, cudaEventDisableTiming));
    PB_CUDA(cudaEventCreateWithFlags(&ev_halo, cudaEventDisableTiming));
    PB_CUDA(cudaEventCreateWithFlags(&ev_words, cudaEventDisableTiming));
    PB_CUDA(cudaEventCreateWithFlags(&ev_table, cudaEventDisableTiming));
    ctl.ensure(sizeof(Ctl));
    PB_CUDA(cudaMemsetAsync(ctl.p, 0, sizeof(Ctl), stream));
    partials.ensure(sizeof(double) * 8 * size_t(sm_count) * 8);
    hist.ensure(SEL_BINS * sizeof(uint32_t));
    PB_CUDA(cudaMemsetAsync(hist.p, 0, SEL_BINS * sizeof(uint32_t), stream));
    sync();
}

Engine::~Engine() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (auto& x : ev)
        if (x) cudaEventDestroy(x);
    if (copy_stream) {
        cudaStreamSynchronize(copy_stream);
        cudaStreamDestroy(copy_stream);
    }
    if (io_stream) {
        cudaStreamSynchronize(io_stream);
        cudaStreamDestroy(io_stream);
    }
    if (halo_stream) {
        cudaStreamSynchronize(halo_stream);
        cudaStreamDestroy(halo_stream);
    }
    if (nccl) nccl_transport_destroy(nccl);
    if (ev_pack) cudaEventDestroy(ev_pack);
    if (ev_halo) cudaEventDestroy(ev_halo);
    if (ev_words) cudaEventDestroy(ev_words);
    if (ev_table) cudaEventDestroy(ev_table);
    if (pinned) cudaFreeHost(pinned);
    if (mapped) cudaFreeHost(mapped);
    if (own_stream && stream) cudaStreamDestroy(stream);
}

/// read_back's device side: payload words into mapped host memory, then the sequence flag.
__global__ void publish_kernel(const uint32_t* __restrict__ src, uint32_t* dst, uint32_t nwords, uint32_t* flag,
                               uint32_t seq) {
    for (uint32_t i = threadIdx.x; i < nwords; i += blockDim.x) dst[i] = __ldcg(src + i);
    __syncthreads();  // every thread's payload stores happen-before thread 0's fence ...
    if (threadIdx.x == 0) {
        __threadfence_system();  // ... which orders them (cumulativity) before the flag at system scope
        *(volatile uint32_t*)flag = seq;
    }
}

void Engine::publish(const void* dptr, uint32_t nwords) {
    const uint32_t want = ++rb_seq;
    uint32_t* base = static_cast<uint32_t*>(mapped_dev);
    publish_kernel<<<1, 128, 0, stream>>>(static_cast<const uint32_t*>(dptr), base + 16, nwords, base, want);
    check_launch();
    volatile uint32_t* flag = static_cast<volatile uint32_t*>(mapped);
    // A failed kernel never raises the flag: look at the stream now and then; a kernel that neither finishes nor
    // fails (a wedged device) ends the wait after PB200_READBACK_TIMEOUT_S seconds (default 120) instead of spinning
    // for ever.
    static const double timeout_s = [] {
        const char* e = std::getenv("PB200_READBACK_TIMEOUT_S");
        const double v = e ? std::atof(e) : 120.0;
        return v > 0 ? v : 120.0;
    }();
    std::chrono::steady_clock::time_point t0{};
    bool timing = false;
    for (uint64_t spins = 1; *flag != want; ++spins) {
        if ((spins & 0x3fff) == 0) {
            const cudaError_t q = cudaStreamQuery(stream);
            if (q == cudaSuccess) {
                if (*flag == want) break;
                throw CudaFail("internal error: read-back flag missing after the stream drained");
            }
            if (q != cudaErrorNotReady) PB_CUDA(q);
            if (!timing) {
                t0 = std::chrono::steady_clock::now();
                timing = true;
            } else if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
                throw CudaFail("read-back timed out after " + std::to_string(int(timeout_s)) +
                               " s: a kernel on the context's stream neither finished nor failed");
            }
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
}

void Engine::exclusive_scan(uint32_t* data, uint64_t n) {
    if (n == 0) return;
    const uint64_t ntiles = (n + LB_TILE - 1) / LB_TILE;
    // [ticket (8 bytes)] [status: one 64-bit word per tile]
    scan_tiles.ensure((ntiles + 1) * 8);
    PB_CUDA(cudaMemsetAsync(scan_tiles.p, 0, (ntiles + 1) * 8, stream));
    unsigned long long* st = scan_tiles.as<unsigned long long>();
    scan_lookback_kernel<<<unsigned(ntiles), NT, 0, stream>>>(data, n, data, st + 1, reinterpret_cast<unsigned*>(st));
    check_launch();
}

bool Engine::rows_sorted_on_device(const uint32_t* table, uint32_t n) {
    Ctl* c = dctl();
    uint32_t* bad = reinterpret_cast<uint32_t*>(&c->pad[0]);
    PB_CUDA(cudaMemsetAsync(bad, 0, 4, stream));
    PB_DISPATCH_W(md.W, check_sorted_kernel<W><<<grid_for(n), NT, 0, stream>>>(table, n, bad));
    check_launch();
    return read_back<uint32_t>(bad) == 0;
}

// ------------------------------------------------------------------------------------------------
void Engine::set_model(const HostModel& m) {
    hm = m;
    const size_t L = m.L;
    std::vector<int> nbs(L * MAX_NB, -1);
    std::vector<double> nba(L * MAX_NB, 0.0);
    std::vector<int> deg(L, 0);
    std::vector<std::vector<std::pair<uint32_t, double>>> adj(L);
    for (size_t b = 0; b < m.bonds.size(); ++b) {
        if (m.hop[b] == 0.0) continue;  // zero parameters produce no term (lattice_models.hpp:163)
        adj[m.bonds[b].first].push_back({m.bonds[b].second, m.hop[b]});
        adj[m.bonds[b].second].push_back({m.bonds[b].first, m.hop[b]});
    }
    int max_deg = 0;
    for (size_t s = 0; s < L; ++s) {
        std::sort(adj[s].begin(), adj[s].end());
        if (adj[s].size() > size_t(MAX_NB)) throw PacesError("lattice site with more than 6 bonds");
        for (size_t d = 0; d < adj[s].size(); ++d) {
            nbs[s * MAX_NB + d] = int(adj[s][d].first);
            nba[s * MAX_NB + d] = adj[s][d].second;
        }
        max_deg = std::max(max_deg, int(adj[s].size()));
    }
    std::vector<double> om = m.omega, gg = m.g;
    if (om.empty()) om.assign(L, 0.0);
    if (gg.empty()) gg.assign(L, 0.0);
    d_eps.ensure(L * 8);
    d_omega.ensure(L * 8);
    d_g.ensure(L * 8);
    d_nbs.ensure(L * MAX_NB * 4);
    d_nba.ensure(L * MAX_NB * 8);
    PB_CUDA(cudaMemcpyAsync(d_eps.p, m.eps.data(), L * 8, cudaMemcpyHostToDevice, stream));
    PB_CUDA(cudaMemcpyAsync(d_omega.p, om.data(), L * 8, cudaMemcpyHostToDevice, stream));
    PB_CUDA(cudaMemcpyAsync(d_g.p, gg.data(), L * 8, cudaMemcpyHostToDevice, stream));
    PB_CUDA(cudaMemcpyAsync(d_nbs.p, nbs.data(), L * MAX_NB * 4, cudaMemcpyHostToDevice, stream));
    PB_CUDA(cudaMemcpyAsync(d_nba.p, nba.data(), L * MAX_NB * 8, cudaMemcpyHostToDevice, stream));
    sync();
    md.kind = m.kind;
    md.L = int(L);
    md.nph = (m.kind == 1) ? int(L) : 0;
    md.b0 = m.b0;
    md.bp = m.bp;
    md.W = int(m.W);
    md.d_pho = m.d_pho;
    md.max_deg = max_deg;
    md.eps = d_eps.as<double>();
    md.omega = d_omega.as<double>();
    md.g = d_g.as<double>();
    md.nb_site = d_nbs.as<int>();
    md.nb_amp = d_nba.as<double>();
    for (int w = 0; w <= 16; ++w) {
        // first phonon register whose leading bit (offset b0 + j*bp) is at or beyond bit 32*w
        int j = 0;
        if (md.bp > 0 && 32 * w > md.b0) j = (32 * w - md.b0 + md.bp - 1) / md.bp;
        md.wfirst[w] = std::min(j, md.nph);
    }
    {
        // omega[j] * double(n): the products the diagonal sums, tabulated once (same IEEE multiply as
        // lattice_models.hpp:234; the host compiler contracts no FMA)
        const int nph = (m.kind == 1) ? int(L) : 0;
        const size_t per = size_t(1) << m.bp;
        std::vector<double> tab(std::max<size_t>(1, size_t(nph) * per), 0.0);
        for (int j = 0; j < nph; ++j)
            for (size_t q = 0; q < per; ++q) tab[size_t(j) * per + q] = om[size_t(j)] * double(q);
        d_omega_n.ensure(tab.size() * 8);
        PB_CUDA(cudaMemcpy(d_omega_n.p, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice));
        md.omega_n = d_omega_n.as<double>();
        // exact uniform-omega shortcut of the diagonal (see ModelDev::diag_uniform)
        bool uniform = nph > 0 && m.bp > 0;
        for (size_t s2 = 0; s2 < L && uniform; ++s2) uniform = (m.eps[s2] == 0.0);
        const double w0 = nph > 0 ? om[0] : 0.0;
        for (int j = 0; j < nph && uniform; ++j) uniform = (om[size_t(j)] == w0);
        uniform = uniform && w0 == std::floor(w0) && std::fabs(w0) * double(nph) * double(per) < 9.0e15;
        std::vector<uint32_t> masks(std::max<size_t>(1, size_t(m.bp) * m.W), 0u);
        for (int j = 0; j < nph; ++j)
            for (int b = 0; b < m.bp; ++b) {
                // bit b (value 2^b) of register j sits at bit offset b0 + j*bp + (bp-1-b) from the top of word 0
                const int off = m.b0 + j * m.bp + (m.bp - 1 - b);
                masks[size_t(b) * m.W + size_t(off >> 5)] |= 1u << (31 - (off & 31));
            }
        d_diag_masks.ensure(masks.size() * 4);
        PB_CUDA(cudaMemcpy(d_diag_masks.p, masks.data(), masks.size() * 4, cudaMemcpyHostToDevice));
        md.diag_masks = d_diag_masks.as<uint32_t>();
        md.diag_uniform = uniform ? 1 : 0;
        md.omega_u = w0;
    }
    {
        // value table: every matrix element for_each_neighbor() can emit -- bond amplitudes, g*sqrt(double(k)) (same
        // IEEE operations as the device generator: correctly rounded sqrt, one multiply) and, for diag_uniform models,
        // omega_u * double(N).  Anything it misses only costs the codes (encode raises `fail`), never a wrong value.
        std::vector<double> vt;
        for (double a : nba)
            if (a != 0.0) vt.push_back(a);
        if (m.kind == 1)
            for (size_t s2 = 0; s2 < L; ++s2)
                if (gg[s2] != 0.0)
                    for (uint32_t k = 1; k < m.d_pho; ++k) vt.push_back(gg[s2] * std::sqrt(double(k)));
        if (md.diag_uniform) {
            const uint64_t top = uint64_t(L) * (m.d_pho > 0 ? m.d_pho - 1 : 0);
            for (uint64_t N = 1; N <= top && vt.size() <= size_t(TAYLOR_VT_MAX) + 1; ++N) vt.push_back(md.omega_u * double(N));
        }
        auto bits = [](double v) {
            uint64_t b;
            std::memcpy(&b, &v, 8);
            return b;
        };
        std::sort(vt.begin(), vt.end(), [&](double a, double b) { return bits(a) < bits(b); });
        vt.erase(std::unique(vt.begin(), vt.end(), [&](double a, double b) { return bits(a) == bits(b); }), vt.end());
        md.vtab = nullptr;
        md.vt_n = 0;
        md.vt_diag = md.diag_uniform;
        if (!vt.empty() && vt.size() <= size_t(TAYLOR_VT_MAX)) {
            d_vtab.ensure(vt.size() * 8);
            PB_CUDA(cudaMemcpy(d_vtab.p, vt.data(), vt.size() * 8, cudaMemcpyHostToDevice));
            md.vtab = d_vtab.as<double>();
            md.vt_n = int(vt.size());
        }
    }
    row_width = max_deg + (m.kind == 1 ? 2 : 0) + 1;
    space[0].has_code = space[1].has_code = false;
    has_model = true;
    has_state = false;
    has_cfg = false;
    space[0].n = space[1].n = 0;
    space[0].has_h = space[1].has_h = false;
    space[0].has_full = space[1].has_full = false;
    space[0].has_move = space[1].has_move = false;
    if (m.W > 16) throw PacesError("basis keys wider than 16 words (512 bits) are not supported by this build");
}

// ------------------------------------------------------------------------------------------------
// K2: counting sort of the candidates by insertion gap, exact dedup + rank inside each gap segment, and the
// scatter that writes the merged sorted table plus the next (sorted) frontier.  Expects gap[] (n+2 counters)
// filled by the expansion kernel; the new frontier ends up in frontier[fcur] (fcur is flipped).
// ------------------------------------------------------------------------------------------------
/// Counting sort of the candidates by insertion gap, exact dedup + rank inside each gap segment, and the scan of
/// the survivor counts: afterwards row_len[g] = unique new keys in gaps < g, row_len[n+1] = their total.
void Engine::dedup_candidates_async(uint32_t n, uint32_t nc_bound) {
    const int W = md.W;
    Ctl* c = dctl();
    const uint32_t* nc_ptr = &c->grow.n_cand;  // exact candidate count, on the device
    const int gc_grid = grid_for(nc_bound);
    // counting sort by insertion gap: gap[] (counts) -> segment starts; row_len[] is the per-gap cursor
    // during placement and then the per-gap survivor count
    exclusive_scan(gap.as<uint32_t>(), uint64_t(n) + 2);
    perm.ensure(size_t(nc_bound) * 4 + 4);
    seg_rank.ensure(size_t(nc_bound) * 4 + 4);
    row_len.ensure((size_t(n) + 2) * 4);
    PB_CUDA(cudaMemsetAsync(row_len.p, 0, (size_t(n) + 2) * 4, stream));
    place_candidates_kernel<<<gc_grid, NT, 0, stream>>>(cand_gap.as<uint32_t>(), nc_ptr, nc_bound, 0, gap.as<uint32_t>(),
                                                        row_len.as<uint32_t>(), perm.as<uint32_t>());
    check_launch();
    PB_CUDA(cudaMemsetAsync(row_len.p, 0, (size_t(n) + 2) * 4, stream));
    PB_DISPATCH_W(W, segment_dedup_kernel<W><<<gc_grid, NT, 0, stream>>>(
                         cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), perm.as<uint32_t>(), nc_ptr, nc_bound, 0,
                         gap.as<uint32_t>(), seg_rank.as<uint32_t>(), row_len.as<uint32_t>(), &c->grow));
    check_launch();
    PB_DISPATCH_W(W, segment_rank_kernel<W><<<gc_grid, NT, 0, stream>>>(
                         cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), perm.as<uint32_t>(), nc_ptr, nc_bound, 0,
                         gap.as<uint32_t>(), seg_rank.as<uint32_t>()));
    check_launch();
    // kept_before[g] = number of new keys in gaps < g; kept_before[n+1] = total
    exclusive_scan(row_len.as<uint32_t>(), uint64_t(n) + 2);
}

uint32_t Engine::dedup_candidates(uint32_t n, uint32_t nc_bound) {
    dedup_candidates_async(n, nc_bound);
    return read_back<uint32_t>(row_len.as<uint32_t>() + (size_t(n) + 1));
}

uint32_t Engine::merge_level(Space& out, uint32_t n, uint32_t nc_bound, int& fcur, bool deferred,
                             GrowCounters* counters) {
    const int W = md.W;
    Ctl* c = dctl();
    const uint32_t* nc_ptr = &c->grow.n_cand;  // exact candidate count, on the device
    const int gc_grid = grid_for(nc_bound);
    dedup_candidates_async(n, nc_bound);
    uint32_t n_new = 0;
    uint64_t rows_bound;
    if (deferred) {
        // size the merged table by the bound n + nc_bound and read the counts back once, after the scatter
        PB_CUDA(cudaMemcpyAsync(&c->n_new, row_len.as<uint32_t>() + (size_t(n) + 1), 4, cudaMemcpyDeviceToDevice,
                                stream));
        rows_bound = uint64_t(n) + nc_bound;
        frontier[fcur ^ 1].ensure(size_t(nc_bound) * 4 + 4);
    } else {
        n_new = read_back<uint32_t>(row_len.as<uint32_t>() + (size_t(n) + 1));
        rows_bound = uint64_t(n) + n_new;
        frontier[fcur ^ 1].ensure(size_t(n_new) * 4 + 4);
    }
    if (rows_bound > 0x7fffffffull && !deferred)
        throw PacesError("subspace growth: table exceeds 2^31 rows (CSR columns are int32)");
    tab_tmp.ensure(size_t(rows_bound) * W * 4);
    PB_DISPATCH_W(W, merge_old_rows_kernel<W><<<grid_for(n), NT, 0, stream>>>(
                         out.words.as<uint32_t>(), n, row_len.as<uint32_t>(), tab_tmp.as<uint32_t>()));
    check_launch();
    PB_DISPATCH_W(W, merge_new_rows_kernel<W><<<gc_grid, NT, 0, stream>>>(
                         cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), perm.as<uint32_t>(),
                         seg_rank.as<uint32_t>(), nc_ptr, row_len.as<uint32_t>(), tab_tmp.as<uint32_t>(),
                         frontier[fcur ^ 1].as<uint32_t>()));
    check_launch();
    if (deferred) {
        const Ctl snap = read_back<Ctl>(c);
        if (counters) *counters = snap.grow;
        n_new = snap.n_new;
        if (uint64_t(n) + n_new > 0x7fffffffull)
            throw PacesError("subspace growth: table exceeds 2^31 rows (CSR columns are int32)");
    }
    out.words.swap(tab_tmp);
    fcur ^= 1;
    return n_new;
}

// ------------------------------------------------------------------------------------------------
// grow_subspace (subspace.hpp:195-249)
// ------------------------------------------------------------------------------------------------
void Engine::grow(const uint32_t* d_seeds, uint32_t ns, int order, Space& out) {
    require_model();
    if (ns == 0) throw PacesError("grow_subspace: empty seed set");
    if (order < 0) throw PacesError("grow_subspace: neighbor order must be >= 0");
    const int W = md.W;
    const int nmoves = md.max_deg + (md.kind == 1 ? 2 : 0);  // off-diagonal moves per key
    const int count_emitted = memory_cap_bytes() != 0;  // transcript sizes only matter for the cap check

    out.words.ensure(size_t(ns) * W * 4);
    PB_CUDA(cudaMemcpyAsync(out.words.p, d_seeds, size_t(ns) * W * 4, cudaMemcpyDeviceToDevice, stream));
    uint32_t n = ns;
    uint32_t nf = ns;
    bool identity_frontier = true;
    int fcur = 0;
    uint64_t emitted_total = 0;
    Ctl* c = dctl();

    int levels_done = 0;
    for (int k = 0; k < order && nf > 0; ++k, ++levels_done) {
        const uint64_t cand_cap64 = uint64_t(nf) * uint64_t(nmoves);
        if (cand_cap64 == 0) {
            nf = 0;
            break;
        }
        if (cand_cap64 > 0xfffffff0ull) throw PacesError("subspace growth: candidate count exceeds 32-bit indexing");
        const uint32_t cand_cap = uint32_t(cand_cap64);
        cand_keys.ensure(size_t(cand_cap) * W * 4);
        cand_gap.ensure(size_t(cand_cap) * 4);
        gap.ensure((size_t(n) + 2) * 4);
        PB_CUDA(cudaMemsetAsync(gap.p, 0, (size_t(n) + 2) * 4, stream));
        PB_CUDA(cudaMemsetAsync(&c->grow, 0, sizeof(GrowCounters), stream));
        const uint32_t* fr = identity_frontier ? nullptr : frontier[fcur].as<uint32_t>();
        const uint32_t xchunk = chunk_for(nf);
        PB_DISPATCH_W(W, expand_window_kernel<W><<<grid_chunked(nf, xchunk), NT, 0, stream>>>(
                             md, out.words.as<uint32_t>(), n, fr, nf, xchunk, cand_keys.as<uint32_t>(),
                             cand_gap.as<uint32_t>(), cand_cap, gap.as<uint32_t>(), &c->grow, count_emitted));
        check_launch();
        // dedup + merge run on the device-side candidate count; ONE read-back per BFS order brings the counters
        GrowCounters gc{};
        const uint32_t n_new = merge_level(out, n, cand_cap, fcur, true, &gc);
        if (gc.overflow) throw CudaFail("internal error: candidate buffer overflow during expansion");
        if (std::getenv("PB200_DEBUG_GROW"))
            std::fprintf(stderr, "[grow] level %d: n=%u nf=%u candidates=%u new=%u longest gap segment=%u\n", k, n, nf,
                         gc.n_cand, n_new, gc.max_seg);
        emitted_total += gc.emitted;
        identity_frontier = false;
        n += n_new;
        nf = n_new;  // 0 when nothing new was found: the loop ends, the (re-copied) table is unchanged
        require_memory((uint64_t(n) * W + emitted_total * W * 2) * 4 + emitted_total * 8, "subspace growth");
    }
    out.n = n;
    out.q_nom = ns;
    out.order = order;
    // which rows had their neighbourhood generated: all but the last frontier (incremental.cuh needs it next step)
    out.full.ensure(size_t(n) + 1);
    PB_CUDA(cudaMemsetAsync(out.full.p, order == 0 ? 0 : 1, n, stream));
    if (order > 0 && levels_done == order && nf > 0 && !identity_frontier) {
        inc_clear_full_kernel<<<grid_for(nf), NT, 0, stream>>>(frontier[fcur].as<uint32_t>(), nf, out.full.as<uint8_t>());
        check_launch();
    }
    out.has_full = true;
    PB_CUDA(cudaEventRecord(ev[2], stream));
    assemble(out);
}

// ------------------------------------------------------------------------------------------------
// assemble_effective_hamiltonian (subspace.hpp:142-187), row-wise
// ------------------------------------------------------------------------------------------------
void Engine::assemble(Space& sp) {
    const int W = md.W;
    const uint32_t n = sp.n;
    const int width = row_width;
    tmp_col.ensure(size_t(n) * width * 4);
    tmp_val.ensure(size_t(n) * width * 8);
    sp.row_ptr.ensure((size_t(n) + 1) * 4 + CSR_PAD);
    const uint32_t achunk = chunk_for(n);
    PB_DISPATCH_W(W, assemble_window_kernel<W><<<grid_chunked(n, achunk), NT, 0, stream>>>(
                         md, sp.words.as<uint32_t>(), n, achunk, width, tmp_col.as<uint32_t>(), tmp_val.as<double>(),
                         sp.row_ptr.as<uint32_t>()));
    check_launch();
    PB_CUDA(cudaMemsetAsync(sp.row_ptr.as<uint32_t>() + n, 0, 4, stream));
    exclusive_scan(sp.row_ptr.as<uint32_t>(), uint64_t(n) + 1);
    uint32_t nnz = 0;
    if (defer_reads) {
        // resident step: size col/val by the row-width bound and pick nnz up with the step's final read-back
        PB_CUDA(cudaMemcpyAsync(&dctl()->nnz, sp.row_ptr.as<uint32_t>() + n, 4, cudaMemcpyDeviceToDevice, stream));
        sp.col.ensure(size_t(n) * width * 4 + CSR_PAD);
        sp.val.ensure(size_t(n) * width * 8 + CSR_PAD);
    } else {
        nnz = read_back<uint32_t>(sp.row_ptr.as<uint32_t>() + n);
        // the reference's assembly buffer check: 2 entries of 16 bytes per transcript element (subspace.hpp:152)
        require_memory(uint64_t(nnz) * 2 * 16, "matrix assembly buffer");
        sp.col.ensure(size_t(nnz) * 4 + CSR_PAD);
        sp.val.ensure(size_t(nnz) * 8 + CSR_PAD);
    }
    assemble_compact_kernel<<<grid_for(n), NT, 0, stream>>>(n, width, tmp_col.as<uint32_t>(), tmp_val.as<double>(),
                                                            sp.row_ptr.as<uint32_t>(), sp.col.as<int32_t>(),
                                                            sp.val.as<double>());
    check_launch();
    sp.nnz = nnz;
    sp.max_row = width;
    sp.has_h = true;
    sp.val_valid = true;
    // value codes for the Taylor tile kernels (single GPU): one more pass over the finished CSR
    sp.has_code = false;
    if (!sharded) {
        uint32_t* fail = &dctl()->code_fail;
        if (encode_values_async(sp, n, defer_reads ? uint64_t(n) * width : nnz, nullptr, fail))
            sp.has_code = read_back<uint32_t>(fail) == 0;
    }
}

void Engine::ensure_val(const Space& csp) {
    if (csp.val_valid) return;
    Space& sp = const_cast<Space&>(csp);
    if (!sp.has_code) throw CudaFail("internal error: H_eff has neither values nor value codes");
    const uint64_t zb = sp.nnz ? sp.nnz : uint64_t(sp.n) * uint64_t(std::max(sp.max_row, 1));
    sp.val.ensure(size_t(zb) * 8 + CSR_PAD);
    decode_csr_kernel<<<grid_for(sp.n), NT, 0, stream>>>(sp.n, sp.row_ptr.as<uint32_t>(), sp.code.as<uint16_t>(),
                                                        sp.diag.as<double>(), md.vtab, sp.val.as<double>());
    check_launch();
    sp.val_valid = true;
}

bool Engine::encode_values_async(Space& sp, uint64_t n_bound, uint64_t nnz_bound, const uint32_t* n_ptr, uint32_t* fail) {
    if (!use_codes || md.vt_n <= 0 || sp.max_row < 1 || sp.max_row > 9) return false;
    sp.code.ensure(size_t(nnz_bound) * 2 + CSR_PAD);
    if (!md.vt_diag) sp.diag.ensure(size_t(n_bound) * 8 + CSR_PAD);
    PB_CUDA(cudaMemsetAsync(fail, 0, 4, stream));
    encode_csr_kernel<<<grid_for(n_bound), NT, 0, stream>>>(uint32_t(n_bound), n_ptr, sp.row_ptr.as<uint32_t>(),
                                                             sp.col.as<int32_t>(), sp.val.as<double>(), md.vtab, md.vt_n,
                                                             md.vt_diag, sp.code.as<uint16_t>(), sp.diag.as<double>(),
                                                             fail);
    check_launch();
    return true;
}

// ------------------------------------------------------------------------------------------------
// truncate_select (engine.hpp:107-156)
// ------------------------------------------------------------------------------------------------
uint32_t Engine::select(const uint32_t* d_words, const double2* d_c, uint32_t n, uint64_t q_nom, uint64_t seed,
                        double* norm2_out, bool compact) {
    require_model();
    if (q_nom < 1) throw PacesError("truncate_select: q_nom must be >= 1");
    const int W = md.W;
    Ctl* c = dctl();
    weights.ensure(size_t(n) * 8 + 8);
    PB_CUDA(cudaMemsetAsync(hist.p, 0, SEL_BINS * sizeof(uint32_t), stream));
    flag_keep.ensure((size_t(n) + 1) * 4);
    const int g = grid_for(n);
    SelectCtl init{};
    init.k = q_nom;
    std::memcpy(pinned, &init, sizeof(init));
    PB_CUDA(cudaMemcpyAsync(&c->select, pinned, sizeof(SelectCtl), cudaMemcpyHostToDevice, stream));
    // pass 1 (weights + top digit) -> pass 2 -> gather the surviving group -> single-CTA tail; ONE read-back
    sel_list.ensure(size_t(SEL_LIST_CAP) * 8);
    weights_hist_kernel<<<g, NT, 0, stream>>>(d_c, n, weights.as<double>(), partials.as<double>(), &c->select,
                                              hist.as<uint32_t>());
    check_launch();
    select_pass_kernel<<<g, NT, 0, stream>>>(weights.as<double>(), n, 42, 11, &c->select, hist.as<uint32_t>(), 2);
    check_launch();
    select_gather_kernel<<<g, NT, 0, stream>>>(weights.as<double>(), n, 42, &c->select,
                                               sel_list.as<unsigned long long>());
    check_launch();
    select_tail_kernel<<<1, NT, 0, stream>>>(sel_list.as<unsigned long long>(), &c->select);
    check_launch();
    SelectCtl sc = read_back<SelectCtl>(&c->select);
    if (norm2_out) *norm2_out = sc.norm2;
    if (sc.support == 0) {
        if (pending_words) {  // the reference checks sortedness first (engine.hpp:110-112)
            PB_CUDA(cudaStreamWaitEvent(stream, ev_words, 0));
            pending_words = false;
            if (!rows_sorted_on_device(d_words, n)) throw PacesError("truncate_select: state table must be sorted");
        }
        throw PacesError("truncate_select: state has no support");
    }

    // compact: uint32 keep flags for the compaction of the kept keys (full expansion); otherwise the kept rows are
    // marked as BFS distance 0 for the incremental adapt phase (incremental.cuh), which never materialises them
    uint32_t* keep = compact ? flag_keep.as<uint32_t>() : nullptr;
    uint8_t* dist0 = nullptr;
    if (!compact) {
        inc_dist.ensure(size_t(n) + 16);
        dist0 = inc_dist.as<uint8_t>();
    }
    uint64_t kept64 = sc.support;
    if (sc.support <= q_nom) {
        select_flags_kernel<<<g, NT, 0, stream>>>(weights.as<double>(), n, 0, &c->select, 1, keep, nullptr, dist0);
        check_launch();
    } else {
        kept64 = q_nom;
        if (!sc.tail_done) {
            // the group sharing the first 22 bits did not fit the list (massive exact ties): full passes
            static const int shifts[4] = {31, 20, 9, 0};
            static const int widths[4] = {11, 11, 11, 9};
            for (int p = 0; p < 4; ++p) {
                select_pass_kernel<<<g, NT, 0, stream>>>(weights.as<double>(), n, shifts[p], widths[p], &c->select,
                                                         hist.as<uint32_t>(), 1);
                check_launch();
            }
            sc = read_back<SelectCtl>(&c->select);
        }
        const uint64_t need = q_nom - sc.count_gt;  // 1 <= need <= count_eq
        if (need >= sc.count_eq) {
            // every tie is admitted: the shuffle loop of engine.hpp:138-141 does not run
            select_flags_kernel<<<g, NT, 0, stream>>>(weights.as<double>(), n, 1, &c->select, 1, keep, nullptr, dist0);
            check_launch();
        } else {
            // ties in ascending table index -> host -> seeded Fisher-Yates exactly as engine.hpp:137-142
            flag_tie.ensure((size_t(n) + 1) * 4);
            pos_a.ensure((size_t(n) + 1) * 4);
            select_flags_kernel<<<g, NT, 0, stream>>>(weights.as<double>(), n, 1, &c->select, 0, keep,
                                                      flag_tie.as<uint32_t>(), dist0);
            check_launch();
            PB_CUDA(cudaMemcpyAsync(pos_a.p, flag_tie.p, (size_t(n) + 1) * 4, cudaMemcpyDeviceToDevice, stream));
            exclusive_scan(pos_a.as<uint32_t>(), uint64_t(n) + 1);
            const uint32_t nt = uint32_t(sc.count_eq);
            idx_tmp.ensure(size_t(nt) * 4 + 4);
            compact_index_kernel<<<g, NT, 0, stream>>>(flag_tie.as<uint32_t>(), pos_a.as<uint32_t>(), n,
                                                       idx_tmp.as<uint32_t>());
            check_launch();
            std::vector<uint32_t> ties(nt);
            PB_CUDA(cudaMemcpyAsync(ties.data(), idx_tmp.p, size_t(nt) * 4, cudaMemcpyDeviceToHost, stream));
            sync();
            std::mt19937_64 rng(seed);
            for (size_t i = ties.size(); i > 1 && need < ties.size(); --i) {
                const size_t j = size_t(rng() % i);
                std::swap(ties[i - 1], ties[j]);
            }
            PB_CUDA(cudaMemcpyAsync(idx_tmp.p, ties.data(), size_t(need) * 4, cudaMemcpyHostToDevice, stream));
            set_flags_kernel<<<grid_for(need), NT, 0, stream>>>(idx_tmp.as<uint32_t>(), uint32_t(need), keep, dist0);
            check_launch();
            sync();  // `ties` must outlive the copy
        }
    }
    const uint32_t kept = uint32_t(kept64);  // = popcount of keep[]: support when nothing is cut, else q_nom
    if (compact) compact_kept(d_words, n, kept);
    return kept;
}

void Engine::compact_kept(const uint32_t* d_words, uint32_t n, uint32_t kept) {
    const int W = md.W;
    const int g = grid_for(n);
    uint32_t* keep = flag_keep.as<uint32_t>();
    pos_a.ensure((size_t(n) + 1) * 4);
    PB_CUDA(cudaMemcpyAsync(pos_a.p, keep, (size_t(n) + 1) * 4, cudaMemcpyDeviceToDevice, stream));
    exclusive_scan(pos_a.as<uint32_t>(), uint64_t(n) + 1);
    if (pending_words) {
        // pb200_step_io: the keys were uploaded beside the kernels above; from here on they are needed
        PB_CUDA(cudaStreamWaitEvent(stream, ev_words, 0));
        pending_words = false;
        if (!rows_sorted_on_device(d_words, n)) throw PacesError("truncate_select: state table must be sorted");
    }
    seeds.ensure(size_t(kept) * W * 4 + 4);
    PB_DISPATCH_W(W, compact_rows_kernel<W><<<g, NT, 0, stream>>>(d_words, keep, pos_a.as<uint32_t>(), n,
                                                                  seeds.as<uint32_t>()));
    check_launch();
    n_seeds = kept;
}

// ------------------------------------------------------------------------------------------------
// remap_state (subspace.hpp:281-305)
// ------------------------------------------------------------------------------------------------
void Engine::remap_async(const uint32_t* src_words, const double2* src_c, uint32_t ns, const uint32_t* dst_words,
                         uint32_t nd, double2* dst_c) {
    const int W = md.W;
    Ctl* c = dctl();
    PB_CUDA(cudaMemsetAsync(dst_c, 0, size_t(nd) * 16, stream));
    const uint32_t rchunk = chunk_for(ns);
    const int rgrid = std::min(grid_chunked(ns, rchunk), sm_count * 8);  // grid_sum partials: <= 8 CTAs per SM
    if (size_t(rgrid) * 8 > partials.cap) throw CudaFail("internal error: reduction scratch too small for the grid");
    PB_DISPATCH_W(W, remap_window_kernel<W><<<rgrid, NT, 0, stream>>>(src_words, src_c, ns, dst_words, nd, rchunk, dst_c,
                                                                      partials.as<double>(), &c->ticket, c->out));
    check_launch();
}

double Engine::remap(const uint32_t* src_words, const double2* src_c, uint32_t ns, const uint32_t* dst_words,
                     uint32_t nd, double2* dst_c) {
    remap_async(src_words, src_c, ns, dst_words, nd, dst_c);
    const double d = read_back<double>(dctl()->out);
    return sharded ? allreduce_host(d) : d;
}

// ------------------------------------------------------------------------------------------------
void Engine::expectation_async(const Space& sp, const double2* x) {
    Ctl* c = dctl();
    ensure_val(sp);
    expectation_kernel<<<grid_for(sp.n), NT, 0, stream>>>(sp.n, sp.row_ptr.as<uint32_t>(), sp.col.as<int32_t>(),
                                                          sp.val.as<double>(), x, partials.as<double>(), &c->ticket,
                                                          c->out + 1);
    check_launch();
}

void Engine::expectation(const Space& sp, const double2* x, double* exp_out, double* norm2_out, bool check_finite) {
    Ctl* c = dctl();
    if (sharded) {
        // the SpMV reads halo columns: stage x next to its halo
        term[0].ensure((size_t(sp.n) + sp.halo_n) * 16 + 16);
        PB_CUDA(cudaMemcpyAsync(term[0].p, x, size_t(sp.n) * 16, cudaMemcpyDeviceToDevice, stream));
        halo_exchange(sp, term[0].as<double2>());
        x = term[0].as<double2>();
    }
    expectation_async(sp, x);
    struct R {
        double v[3];
    };
    R r = read_back<R>(c->out + 1);
    if (sharded) comm_check(ops.allreduce_f64_host(ops.user, r.v, 3), "allreduce_f64_host");
    if (exp_out) *exp_out = r.v[0];
    if (norm2_out) *norm2_out = r.v[1];
    if (check_finite && r.v[2] != 0.0) throw PacesError("expmv: non-finite input coefficient");
}

void Engine::spmv(const Space& sp, const double2* x, double2* y) {
    ensure_val(sp);
    spmv_kernel<<<grid_for(sp.n), NT, 0, stream>>>(sp.n, sp.row_ptr.as<uint32_t>(), sp.col.as<int32_t>(),
                                                   sp.val.as<double>(), x, y);
    check_launch();
}

// ------------------------------------------------------------------------------------------------
// expmv (propagator.hpp:52-92)
// ------------------------------------------------------------------------------------------------
void Engine::expmv(const Space& sp, double2* c_vec, double dt, double rtol, int max_order, int substeps,
                   int* order_used, double* last_term_norm, double* last_c_norm, bool fuse_expectation,
                   bool state_in_term0) {
    if (!(dt > 0)) throw PacesError("propagator: dt must be > 0");
    if (!(rtol > 0) || !(rtol < 1)) throw PacesError("propagator: rtol must be in (0, 1)");
    if (max_order < 1) throw PacesError("propagator: max_order must be >= 1");
    if (substeps < 1) throw PacesError("propagator: substeps must be >= 1");
    const uint32_t n = sp.n;
    Ctl* c = dctl();
    term[0].ensure(size_t(n) * 16 + 16);
    term[1].ensure(size_t(n) * 16 + 16);
    const double dt_sub = dt / substeps;
    const int g = grid_for(n);
    TaylorCtl tc{};
    PB_CUDA(cudaMemsetAsync(&c->taylor, 0, sizeof(TaylorCtl), stream));
    // state_in_term0 (resident step after an incremental adapt phase, which remaps the coefficients straight into
    // term[0]): the first order takes the state from there and only writes c_vec -- no copy, no read of c_vec
    const bool from_x = state_in_term0 && fuse_expectation;
    if (state_in_term0 && !from_x)
        PB_CUDA(cudaMemcpyAsync(c_vec, term[0].p, size_t(n) * 16, cudaMemcpyDeviceToDevice, stream));
    for (int s = 0; s < substeps; ++s) {
        if (!(from_x && s == 0))
            PB_CUDA(cudaMemcpyAsync(term[0].p, c_vec, size_t(n) * 16, cudaMemcpyDeviceToDevice, stream));
        if (s > 0) {
            // new substep: streak and done restart, order_used keeps its running maximum
            tc.done = 0;
            tc.streak = 0;
            tc.ticket = 0;
            std::memcpy(pinned, &tc, sizeof(tc));
            PB_CUDA(cudaMemcpyAsync(&c->taylor, pinned, sizeof(TaylorCtl), cudaMemcpyHostToDevice, stream));
        }
        int order = 1;
        bool converged = false;
        // Paired orders (kernels.cuh): DEFER/CATCHUP pairs from order k0 on, placed so that the order the previous
        // expmv stopped at is the second of a pair; a DEFER launch that meets streak != 0 raises `bail` instead.
        bool singles = !taylor_defer;
        const int k0 = (last_order > 2 && (last_order & 1) == 0) ? 3 : 2;
        // launch in batches; the stop rule runs on the device and turns the tail of a batch into no-ops
        int batch = last_order > 2 ? last_order : 8;
        while (order <= max_order) {
            const int end = std::min(max_order, order + batch - 1);
            for (; order <= end; ++order) {
                const double b = -dt_sub / double(order);
                const double2* tin = term[(order - 1) & 1].as<double2>();
                double2* tout = term[order & 1].as<double2>();
                const uint32_t* rp = sp.row_ptr.as<uint32_t>();
                const int32_t* cl = sp.col.as<int32_t>();
                const double* vl = sp.val.as<double>();
                double* pt = partials.as<double>();
                TaylorCodes codes_tmp;
                const TaylorCodes* cd = codes_of(sp, codes_tmp);
                if (fuse_expectation && s == 0 && order == 1) {
                    // the first order's row sums are H x: <x|H|x>, |x|^2 and the finiteness check ride along
                    // (Ctl::out[1..3], read with the final read-back)
                    taylor_launch_single(true, g, sm_count, stream, n, rp, cl, vl, tin, tout, c_vec, b, order, rtol, pt,
                                         &c->taylor, 0, nullptr, c->out + 1, sp.max_row, cd, from_x ? 1 : 0);
                } else if (!singles && order >= k0 && ((order - k0) & 1)) {
                    taylor_launch_catchup(g, sm_count, stream, n, rp, cl, vl, tin, tout, c_vec, b, order, rtol, pt,
                                          &c->taylor, sp.max_row, cd);
                } else if (!singles && order >= k0 && order < max_order) {
                    taylor_launch_defer(g, sm_count, stream, n, rp, cl, vl, tin, tout, b, order, pt, &c->taylor,
                                        sp.max_row, cd);
                } else {
                    taylor_launch_single(false, g, sm_count, stream, n, rp, cl, vl, tin, tout, c_vec, b, order, rtol, pt,
                                         &c->taylor, 0, nullptr, nullptr, sp.max_row, cd);
                }
                check_launch();
            }
            last_ctl = read_back<Ctl>(c);  // one read-back carries the stop flag AND the step's deferred scalars
            tc = last_ctl.taylor;
            if (tc.done) {
                converged = true;
                break;
            }
            if (tc.bail) {  // order tc.bail has to run SINGLE (everything launched after it returned at once)
                order = tc.bail;
                singles = true;
                tc.bail = 0;
                PB_CUDA(cudaMemsetAsync(&c->taylor.bail, 0, sizeof(int), stream));
            }
            batch = 2;
        }
        times.taylor_orders += uint64_t(tc.last_order);
        times.taylor_rows += uint64_t(tc.last_order) * n;
        if (!converged)
            throw PacesError("expmv: Taylor series did not converge within max_order=" + std::to_string(max_order) +
                             "; reduce dt or increase substeps");
    }
    times.taylor_deferred += uint64_t(tc.deferred);
    times.taylor_deferred_rows += uint64_t(tc.deferred) * n;
    last_order = tc.order_used;
    if (order_used) *order_used = tc.order_used;
    if (last_term_norm) *last_term_norm = tc.last_term_norm;
    if (last_c_norm) *last_c_norm = tc.last_c_norm;
}

void Engine::upload_csr(Space& sp, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val) {
    if (n < 0 || n > 0x7fffffffLL) throw ArgError("csr: n out of range");
    const int64_t nnz = row_ptr[n];
    if (nnz < 0 || nnz > 0xfffffff0LL) throw ArgError("csr: nnz out of range");
    std::vector<uint32_t> rp(size_t(n) + 1);
    int64_t longest = 0;
    for (int64_t i = 0; i <= n; ++i) {
        rp[size_t(i)] = uint32_t(row_ptr[i]);
        if (i > 0) longest = std::max<int64_t>(longest, row_ptr[i] - row_ptr[i - 1]);
    }
    sp.max_row = longest <= 15 ? int(std::max<int64_t>(longest, 1)) : 0;
    sp.row_ptr.ensure((size_t(n) + 1) * 4 + CSR_PAD);
    sp.col.ensure(size_t(nnz) * 4 + CSR_PAD);
    sp.val.ensure(size_t(nnz) * 8 + CSR_PAD);
    PB_CUDA(cudaMemcpyAsync(sp.row_ptr.p, rp.data(), (size_t(n) + 1) * 4, cudaMemcpyHostToDevice, stream));
    if (nnz) {
        PB_CUDA(cudaMemcpyAsync(sp.col.p, col, size_t(nnz) * 4, cudaMemcpyHostToDevice, stream));
        PB_CUDA(cudaMemcpyAsync(sp.val.p, val, size_t(nnz) * 8, cudaMemcpyHostToDevice, stream));
    }
    sync();
    sp.n = uint32_t(n);
    sp.nnz = uint64_t(nnz);
    sp.has_h = true;
    sp.has_code = false;  // arbitrary values: the Taylor kernels read `val`
    sp.val_valid = true;
}

// ------------------------------------------------------------------------------------------------
// observables (observables.hpp:26-37, 84-95, 99-112)
// ------------------------------------------------------------------------------------------------
void Engine::observe(const uint32_t* words, const double2* cvec, uint32_t n, double* density, double* amp,
                     double* phonons) {
    require_model();
    const int W = md.W;
    const int L = md.L;
    const uint32_t rows_per_block = 4096;
    const uint32_t nb = (n + rows_per_block - 1) / rows_per_block;
    aux_vec.ensure((size_t(nb) * L + size_t(L) * 3 + 8) * 8);
    // layout: [found: L double2 (16-byte aligned)] [out: L doubles] [per-CTA partials: nb * L doubles]
    double2* d_found = aux_vec.as<double2>();
    double* d_out = reinterpret_cast<double*>(d_found + L);
    double* block_part = d_out + L;
    if (density) {
        PB_CUDA(cudaMemsetAsync(block_part, 0, size_t(nb) * L * 8, stream));
        if (nb) {
            PB_DISPATCH_W(W, density_kernel<W><<<nb, NT, 0, stream>>>(md, words, cvec, n, rows_per_block, block_part));
            check_launch();
        }
        density_finish_kernel<<<(L + 127) / 128, 128, 0, stream>>>(block_part, nb, L, d_out);
        check_launch();
        PB_CUDA(cudaMemcpyAsync(density, d_out, size_t(L) * 8, cudaMemcpyDeviceToHost, stream));
        sync();
        if (sharded) comm_check(ops.allreduce_f64_host(ops.user, density, uint64_t(L)), "allreduce_f64_host");
    }
    if (phonons) {
        if (md.kind != 1) throw PacesError("phonon numbers: not a Holstein model");
        PB_CUDA(cudaMemsetAsync(block_part, 0, size_t(nb) * L * 8, stream));
        if (nb) {
            PB_DISPATCH_W(W, phonon_numbers_kernel<W><<<nb, NT, 0, stream>>>(md, words, cvec, n, rows_per_block,
                                                                            block_part));
            check_launch();
        }
        density_finish_kernel<<<(L + 127) / 128, 128, 0, stream>>>(block_part, nb, L, d_out);
        check_launch();
        PB_CUDA(cudaMemcpyAsync(phonons, d_out, size_t(L) * 8, cudaMemcpyDeviceToHost, stream));
        sync();
        if (sharded) comm_check(ops.allreduce_f64_host(ops.user, phonons, uint64_t(L)), "allreduce_f64_host");
    }
    if (amp) {
        PB_DISPATCH_W(W, dipole_kernel<W><<<1, 256, 0, stream>>>(md, words, cvec, n, d_found, d_out));
        check_launch();
        PB_CUDA(cudaMemcpyAsync(amp, d_out, 16, cudaMemcpyDeviceToHost, stream));
        sync();
        if (sharded) {
            // the L vacuum keys share one phonon configuration, hence one owner; the others contribute zeros,
            // but the 1/sqrt(L) factor was applied per rank, which is exact for the single non-zero term
            comm_check(ops.allreduce_f64_host(ops.user, amp, 2), "allreduce_f64_host");
        }
    }
}

// ------------------------------------------------------------------------------------------------
// initialize (engine.hpp:235-251) and the per-step driver (engine.hpp:268-291, 333-368)
// ------------------------------------------------------------------------------------------------
static void validate_cfg(const pb200_run_cfg& c) {
    if (c.m < 0 || c.m_init < c.m) throw PacesError("run: need m_init >= m >= 0");
    if (c.q_nom < 1) throw PacesError("run: q_nom must be >= 1");
    if (c.t_max < 0) throw PacesError("run: t_max must be >= 0");
    if (c.cadence < 1) throw PacesError("run: cadence must be >= 1");
    if (!(c.dt > 0)) throw PacesError("propagator: dt must be > 0");
    if (!(c.rtol > 0) || !(c.rtol < 1)) throw PacesError("propagator: rtol must be in (0, 1)");
    if (c.max_order < 1) throw PacesError("propagator: max_order must be >= 1");
    if (c.substeps < 1) throw PacesError("propagator: substeps must be >= 1");
}

void Engine::run_begin(const pb200_run_cfg& c) {
    require_model();
    validate_cfg(c);
    cfg = c;
    cfg_occ.clear();
    cfg_amp.clear();
    if (c.init_kind == 2 && c.n_entries && c.entry_occ && c.entry_amp) {
        cfg_occ.assign(c.entry_occ, c.entry_occ + c.n_entries * hm.layout_sites());
        cfg_amp.assign(c.entry_amp, c.entry_amp + 2 * c.n_entries);
        cfg.entry_occ = cfg_occ.data();
        cfg.entry_amp = cfg_amp.data();
    }
    has_cfg = true;
    has_state = false;
    std::vector<uint32_t> words;
    std::vector<cplx> amps;
    build_seed_state(hm, c.init_kind, c.init_site, c.n_entries, c.entry_occ, c.entry_amp, words, amps);
    const int W = md.W;
    if (sharded) {
        // every rank builds the same normalised seed list and keeps the keys it owns
        std::vector<uint32_t> w2;
        std::vector<cplx> a2;
        for (size_t k = 0; k < amps.size(); ++k)
            if (host_owner(hm, words.data() + k * W, uint32_t(world)) == uint32_t(rank)) {
                w2.insert(w2.end(), words.begin() + k * W, words.begin() + (k + 1) * W);
                a2.push_back(amps[k]);
            }
        words.swap(w2);
        amps.swap(a2);
    }
    const uint32_t ns = uint32_t(amps.size());
    aux_words.ensure(words.size() * 4 + 16);
    aux_coeff.ensure(amps.size() * 16 + 16);
    PB_CUDA(cudaMemcpyAsync(aux_words.p, words.data(), words.size() * 4, cudaMemcpyHostToDevice, stream));
    PB_CUDA(cudaMemcpyAsync(aux_coeff.p, amps.data(), amps.size() * 16, cudaMemcpyHostToDevice, stream));
    sync();
    Space& sp = space[cur];
    if (sharded)
        grow_sharded(aux_words.as<uint32_t>(), ns, c.m_init, sp);
    else
        grow(aux_words.as<uint32_t>(), ns, c.m_init, sp);
    coeff[ccur].ensure(size_t(sp.n) * 16 + 16);
    const double discarded = remap(aux_words.as<uint32_t>(), aux_coeff.as<double2>(), ns, sp.words.as<uint32_t>(),
                                   sp.n, coeff[ccur].as<double2>());
    if (discarded != 0) throw PacesError("initialize: seed keys lost during growth");
    t = 0;
    steps_done = 0;
    last_order = 0;
    has_state = true;
    times = pb200_phase_times{};
}

void Engine::run_step(pb200_diag* out) {
    if (!has_state || !has_cfg) throw ArgError("no resident run: call pb200_run_begin first");
    const uint64_t s = steps_done + 1;
    pb200_diag rec{};
    rec.step = s;
    const uint64_t launches0 = launches;
    Space& old = space[cur];
    double2* c_old = coeff[ccur].as<double2>();
    PB_CUDA(cudaEventRecord(ev[0], stream));
    if (s == 1) {
        // engine.hpp:335-352: the m_init space is the effective space of the first evolution
        double e = 0, n2 = 0;
        expectation(old, c_old, &e, &n2, true);
        PB_CUDA(cudaEventRecord(ev[5], stream));
        rec.norm_pre = std::sqrt(n2);
        rec.norm_post = rec.norm_pre;
        rec.q_true = sharded ? old.n_global : old.n;
        rec.energy = e;
        coeff[ccur ^ 1].ensure(size_t(old.n) * 16 + 16);
        double2* psi = coeff[ccur ^ 1].as<double2>();
        PB_CUDA(cudaMemcpyAsync(psi, c_old, size_t(old.n) * 16, cudaMemcpyDeviceToDevice, stream));
        int order = 0;
        double ltn = 0, lcn = 0;
        if (sharded)
            expmv_sharded(old, psi, cfg.dt, cfg.rtol, cfg.max_order, cfg.substeps, &order, &ltn, &lcn);
        else
            expmv(old, psi, cfg.dt, cfg.rtol, cfg.max_order, cfg.substeps, &order, &ltn, &lcn);
        PB_CUDA(cudaEventRecord(ev[6], stream));
        sync();
        rec.taylor_order = order;
        rec.delta_norm_expmv = lcn - rec.norm_post;
        ccur ^= 1;
        float ms = 0;
        PB_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[5]));
        times.expectation_ms += ms;
        PB_CUDA(cudaEventElapsedTime(&ms, ev[5], ev[6]));
        times.expmv_ms += ms;
        PB_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[6]));
        times.total_ms += ms;
        times.spmv_nnz += uint64_t(order) * old.nnz;
        if (old.has_code) times.spmv_nnz_coded += uint64_t(order) * old.nnz;
    } else {
        // engine.hpp:268-291
        Space& next = space[cur ^ 1];
        double n2_pre = 0;
        const uint64_t sel_seed = pb200_mix_seed(cfg.seed + s);
        // one GPU: remap / <H> / nnz stay on the device and come back with expmv's final read-back
        struct DeferGuard {
            bool& flag;
            ~DeferGuard() { flag = false; }
        } defer_guard{defer_reads};
        defer_reads = (!sharded);
        // incremental adapt (incremental.cuh): needs the previous H_eff with its expansion flags; the full path
        // remains for the first step after a load, m = 0, a memory cap (its transcript accounting) and overflows
        // (BFS distances are bytes with DIST_INF = 255: larger neighbour orders take the full path)
        bool incremental = !sharded && (!io || io->cached) && old.has_h && old.has_full && cfg.m >= 1 &&
                           cfg.m <= INC_MAX_ORDER && memory_cap_bytes() == 0 &&
                           std::getenv("PB200_NO_INCREMENTAL") == nullptr;
        // (shards: the table grows incrementally from the previous space when it can -- sharded.cu; the same on every rank)
        const bool inc_shard = sharded && old.has_h && old.has_full && cfg.m >= 1 && cfg.m <= INC_MAX_ORDER &&
                               md.max_deg + md.kind > 0 && memory_cap_bytes() == 0 &&
                               std::getenv("PB200_NO_INCREMENTAL") == nullptr;
        uint32_t kept = sharded ? select_sharded(old.words.as<uint32_t>(), c_old, old.n, cfg.q_nom, sel_seed, &n2_pre,
                                                 !inc_shard)
                                : select(old.words.as<uint32_t>(), c_old, old.n, cfg.q_nom, sel_seed, &n2_pre,
                                         !incremental);
        rec.norm_pre = std::sqrt(n2_pre);
        bool shard_discard_rides = false;
        bool shard_remapped = false;  // shards: the incremental table growth also remapped the coefficients (into term[0])
        PB_CUDA(cudaEventRecord(ev[1], stream));
        // (the incremental path remaps the coefficients straight into term[0], the first Taylor order's input)
        if (incremental && !grow_incremental(old, c_old, kept, cfg.m, next, term[0])) {
            incremental = false;
            ++inc_fallbacks;
            // the kept rows are still the rows at distance 0: turn them into the keep flags of the full path
            inc_keep_from_dist_kernel<<<grid_for(uint64_t(old.n) + 1), NT, 0, stream>>>(inc_dist.as<uint8_t>(), old.n,
                                                                                      flag_keep.as<uint32_t>());
            check_launch();
            compact_kept(old.words.as<uint32_t>(), old.n, kept);
        }
        if (incremental) {
            PB_CUDA(cudaEventRecord(ev[2], stream));
        } else if (sharded) {
            // grow() = expansion + assembly; split the timer inside via ev[2].  The table grows incrementally from the
            // previous space when it can (sharded.cu); a buffer bound hit on any rank sends every rank to the full path
            shard_remapped = inc_shard && grow_incremental_sharded(old, c_old, last_kept_global, cfg.m, next, term[0]);
            if (!shard_remapped) {
                if (inc_shard) {  // a buffer bound was hit on some rank: every rank takes the full expansion
                    ++inc_fallbacks;
                    kept = compact_kept_counted(old.words.as<uint32_t>(), old.n);
                }
                grow_sharded(seeds.as<uint32_t>(), kept, cfg.m, next);
            }
        } else {
            grow(seeds.as<uint32_t>(), kept, cfg.m, next);
        }
        PB_CUDA(cudaEventRecord(ev[3], stream));
        if (io && io->start_upload) {
            io->start_upload();
            io->start_upload = nullptr;
        }
        if (io) {
            // the new table is final: ship it to the host beside remap + <H> + expmv
            if (next.n > io->out_cap_rows) throw ArgError("step_io: output buffers too small for the new state");
            PB_CUDA(cudaEventRecord(ev_table, stream));
            PB_CUDA(cudaStreamWaitEvent(copy_stream, ev_table, 0));
            if (next.n)
                PB_CUDA(cudaMemcpyAsync(io->out_words, next.words.p, size_t(next.n) * md.W * 4, cudaMemcpyDeviceToHost,
                                        copy_stream));
        }
        require_memory((sharded ? next.n_global : uint64_t(next.n)) * 16 * 4, "state vectors");
        coeff[ccur ^ 1].ensure(size_t(next.n) * 16 + 16);
        double2* psi = coeff[ccur ^ 1].as<double2>();
        double e = 0, n2 = 0;
        bool shard_fused = false;
        if (defer_reads) {
            // the incremental path already produced psi and the discarded weight (Ctl::out[0])
            if (!incremental)
                remap_async(old.words.as<uint32_t>(), c_old, old.n, next.words.as<uint32_t>(), next.n, psi);
            PB_CUDA(cudaEventRecord(ev[4], stream));
            PB_CUDA(cudaEventRecord(ev[5], stream));  // <H> is produced by the first Taylor order
        } else if (sharded && shard_tiles(next)) {
            // shards on the tile kernels: the coefficients are remapped straight into the first Taylor order's input,
            // which also yields <H>, the norm and the finiteness check (no separate SpMV + halo exchange for <H>, no
            // copy of the state)
            shard_fused = true;
            if (shard_remapped) {
                // the incremental table growth already moved the coefficients into term[0] (index map, no key search)
                const size_t ext_bytes = (size_t(next.n) + next.halo_n) * 16 + 16;
                if (ext_bytes > term[0].cap) sync();  // (the copy of a growing buffer is not stream-ordered)
                term[0].ensure_keep(ext_bytes, size_t(next.n) * 16);
                shard_discard_rides = true;  // (its all-reduce rides on the first Taylor order's)
            } else {
                term[0].ensure((size_t(next.n) + next.halo_n) * 16 + 16);
                rec.discarded_weight = remap(old.words.as<uint32_t>(), c_old, old.n, next.words.as<uint32_t>(), next.n,
                                             term[0].as<double2>());
            }
            PB_CUDA(cudaEventRecord(ev[4], stream));
            PB_CUDA(cudaEventRecord(ev[5], stream));
        } else {
            if (shard_remapped) {  // (row-list Taylor kernels: the state is expected in psi)
                PB_CUDA(cudaMemcpyAsync(psi, term[0].p, size_t(next.n) * 16, cudaMemcpyDeviceToDevice, stream));
                rec.discarded_weight = allreduce_host(read_back<double>(dctl()->out));
            } else {
                rec.discarded_weight =
                    remap(old.words.as<uint32_t>(), c_old, old.n, next.words.as<uint32_t>(), next.n, psi);
            }
            PB_CUDA(cudaEventRecord(ev[4], stream));
            expectation(next, psi, &e, &n2, true);
            PB_CUDA(cudaEventRecord(ev[5], stream));
        }
        int order = 0;
        double ltn = 0, lcn = 0;
        if (sharded) {
            expmv_sharded(next, psi, cfg.dt, cfg.rtol, cfg.max_order, cfg.substeps, &order, &ltn, &lcn, shard_fused,
                          shard_fused ? &e : nullptr, shard_fused ? &n2 : nullptr,
                          shard_discard_rides ? &rec.discarded_weight : nullptr);
        } else {
            try {
                expmv(next, psi, cfg.dt, cfg.rtol, cfg.max_order, cfg.substeps, &order, &ltn, &lcn, true, incremental);
            } catch (const PacesError&) {
                // the reference checks its input before it iterates (propagator.hpp:55-57)
                if (last_ctl.out[3] != 0.0) throw PacesError("expmv: non-finite input coefficient");
                throw;
            }
            // deferred scalars, all produced before the read-back that filled last_ctl
            rec.discarded_weight = last_ctl.out[0];
            e = last_ctl.out[1];
            n2 = last_ctl.out[2];
            if (last_ctl.out[3] != 0.0) throw PacesError("expmv: non-finite input coefficient");
            next.nnz = last_ctl.nnz;
            // the reference's assembly buffer check: 2 entries of 16 bytes per transcript element (subspace.hpp:152)
            require_memory(uint64_t(next.nnz) * 2 * 16, "matrix assembly buffer");
        }
        rec.norm_post = std::sqrt(n2);
        rec.q_true = sharded ? next.n_global : next.n;
        rec.energy = e;
        PB_CUDA(cudaEventRecord(ev[6], stream));
        if (io && io->start_compare) {
            io->start_compare(ev[6]);
            io->start_compare = nullptr;
        }
        if (io && next.n)
            PB_CUDA(cudaMemcpyAsync(io->out_coeff, psi, size_t(next.n) * 16, cudaMemcpyDeviceToHost, stream));
        sync();
        if (io) PB_CUDA(cudaStreamSynchronize(copy_stream));
        if (io && io->cached) {
            // the uploads and their comparisons ran beside the step; nothing is committed before they agree
            PB_CUDA(cudaStreamSynchronize(io_stream));
            struct F {
                uint32_t v[2];
            };
            const F f = read_back<F>(io->mismatch);
            if (f.v[0] != 0 || f.v[1] != 0) throw CacheMiss{};
        }
        rec.taylor_order = order;
        rec.delta_norm_expmv = lcn - rec.norm_post;
        cur ^= 1;
        ccur ^= 1;
        float ms = 0;
        PB_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
        times.select_ms += ms;
        PB_CUDA(cudaEventElapsedTime(&ms, ev[1], ev[2]));
        times.grow_ms += ms;
        PB_CUDA(cudaEventElapsedTime(&ms, ev[2], ev[3]));
        times.assemble_ms += ms;
        PB_CUDA(cudaEventElapsedTime(&ms, ev[3], ev[4]));
        times.remap_ms += ms;
        PB_CUDA(cudaEventElapsedTime(&ms, ev[4], ev[5]));
        times.expectation_ms += ms;
        PB_CUDA(cudaEventElapsedTime(&ms, ev[5], ev[6]));
        times.expmv_ms += ms;
        PB_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[6]));
        times.total_ms += ms;
        times.spmv_nnz += uint64_t(order) * next.nnz;
        if (next.has_code) times.spmv_nnz_coded += uint64_t(order) * next.nnz;
        times.rows_sum += next.n;
        times.nnz_sum += next.nnz;
        times.rows_old_sum += old.n;
        times.kept_sum += kept;
    }
    t = t + cfg.dt;
    rec.t = t;
    steps_done = s;
    times.steps += 1;
    times.kernel_launches += launches - launches0;
    if (out) *out = rec;
}

}  // namespace pb
