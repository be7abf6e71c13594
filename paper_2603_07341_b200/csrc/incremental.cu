// incremental.cu -- orchestration of the incremental adapt phase (kernels and rationale: incremental.cuh).
#include "engine.cuh"

namespace pb {

#ifdef PB_ONLY_W
#define PB_DISPATCH_WI(Wv, ...)                                                                  \
    switch (Wv) {                                                                                \
        case PB_ONLY_W: { constexpr int W = PB_ONLY_W; __VA_ARGS__; } break;                     \
        default: throw PacesError("this development build only supports one key width (PB_ONLY_W)"); \
    }
#else
#define PB_DISPATCH_WI(Wv, ...)                                 \
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

bool Engine::grow_incremental(const Space& old, const double2* c_old, uint32_t kept, int m, Space& next,
                              DevBuf& c_new) {
    const int W = md.W;
    const uint32_t n = old.n;
    const int width = row_width;
    const int nmoves = md.max_deg + (md.kind == 1 ? 2 : 0);
    Ctl* c = dctl();
    inc_ctr.ensure(sizeof(IncCounters));
    IncCounters* ictr = inc_ctr.as<IncCounters>();
    const uint32_t side_cap = n;  // more new keys than old rows: not a steady state, use the full path

    inc_dist.ensure(size_t(n) + 1);
    inc_elist.ensure(size_t(n) * 4 + 4);
    uint8_t* dist = inc_dist.as<uint8_t>();
    inc_init_dist_kernel<<<grid_for(n), NT, 0, stream>>>(flag_keep.as<uint32_t>(), n, dist);
    check_launch();
    PB_CUDA(cudaMemsetAsync(ictr, 0, sizeof(IncCounters), stream));

    uint32_t side_n = 0;
    int scur = 0;
    for (auto& b : inc_side_keys) b.ensure(64);
    for (auto& b : inc_side_gap) b.ensure(64);
    for (auto& b : inc_side_dist) b.ensure(64);

    // candidate capacity: what the buffers already hold (the full path sized them for whole BFS levels), at least a
    // quarter of the table's moves; running out of it only sends this step to the full path
    {
        const uint64_t want = std::max<uint64_t>(uint64_t(n / 4 + 1024) * uint64_t(nmoves), 1u << 16);
        cand_keys.ensure(size_t(want) * W * 4);
        cand_gap.ensure(size_t(want) * 4);
    }
    const uint32_t cand_cap =
        uint32_t(std::min<uint64_t>({cand_keys.cap / (size_t(W) * 4), cand_gap.cap / 4, 0x7ffffff0ull}));
    gap.ensure((size_t(n) + 2) * 4);
    for (int k = 0; k < m; ++k) {
        PB_CUDA(cudaMemsetAsync(&ictr->n_expand, 0, 4, stream));
        inc_mark_level_kernel<<<grid_for(n), NT, 0, stream>>>(n, k, old.full.as<uint8_t>(), old.row_ptr.as<uint32_t>(),
                                                               old.col.as<int32_t>(), dist, inc_elist.as<uint32_t>(),
                                                               ictr);
        check_launch();
        if (nmoves == 0) continue;
        PB_CUDA(cudaMemsetAsync(gap.p, 0, (size_t(n) + 2) * 4, stream));
        PB_CUDA(cudaMemsetAsync(&c->grow, 0, sizeof(GrowCounters), stream));
        PB_DISPATCH_WI(W, inc_expand_kernel<W><<<grid_for(uint64_t(n) + side_n), NT, 0, stream>>>(
                              md, old.words.as<uint32_t>(), n, inc_elist.as<uint32_t>(), &ictr->n_expand,
                              inc_side_keys[scur].as<uint32_t>(), inc_side_dist[scur].as<uint8_t>(), side_n, k, dist,
                              cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), cand_cap, gap.as<uint32_t>(), &c->grow,
                              ictr));
        check_launch();
        inc_clamp_kernel<<<1, 1, 0, stream>>>(&c->grow.n_cand, cand_cap);
        check_launch();
        // unique new keys of this level, canonical order (the dedup machinery of the full path, on the device-side
        // candidate count); ONE read-back per level
        const uint32_t n_new = dedup_candidates(n, cand_cap);
        if (n_new == 0) continue;
        if (uint64_t(side_n) + n_new > side_cap) return false;
        inc_new_keys.ensure(size_t(n_new) * W * 4 + 4);
        inc_new_gap.ensure(size_t(n_new) * 4 + 4);
        PB_DISPATCH_WI(W, inc_emit_unique_kernel<W><<<grid_for(cand_cap), NT, 0, stream>>>(
                              cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), perm.as<uint32_t>(),
                              seg_rank.as<uint32_t>(), &c->grow.n_cand, row_len.as<uint32_t>(),
                              inc_new_keys.as<uint32_t>(), inc_new_gap.as<uint32_t>()));
        check_launch();
        const uint32_t merged = side_n + n_new;
        inc_side_keys[scur ^ 1].ensure(size_t(merged) * W * 4 + 4);
        inc_side_gap[scur ^ 1].ensure(size_t(merged) * 4 + 4);
        inc_side_dist[scur ^ 1].ensure(size_t(merged) + 4);
        PB_DISPATCH_WI(W, inc_side_merge_kernel<W><<<grid_for(merged), NT, 0, stream>>>(
                              inc_side_keys[scur].as<uint32_t>(), inc_side_gap[scur].as<uint32_t>(),
                              inc_side_dist[scur].as<uint8_t>(), side_n, inc_new_keys.as<uint32_t>(),
                              inc_new_gap.as<uint32_t>(), n_new, k + 1, inc_side_keys[scur ^ 1].as<uint32_t>(),
                              inc_side_gap[scur ^ 1].as<uint32_t>(), inc_side_dist[scur ^ 1].as<uint8_t>()));
        check_launch();
        scur ^= 1;
        side_n = merged;
    }

    // ---- index maps: pk = kept old rows before i, nb = side keys before row i
    pos_a.ensure((size_t(n) + 2) * 4);
    inc_keepflag_kernel<<<grid_for(uint64_t(n) + 1), NT, 0, stream>>>(dist, n, m, pos_a.as<uint32_t>());
    check_launch();
    exclusive_scan(pos_a.as<uint32_t>(), uint64_t(n) + 1);
    gap.ensure((size_t(n) + 2) * 4);
    PB_CUDA(cudaMemsetAsync(gap.p, 0, (size_t(n) + 2) * 4, stream));
    if (side_n) {
        inc_count_gaps_kernel<<<grid_for(side_n), NT, 0, stream>>>(inc_side_gap[scur].as<uint32_t>(), side_n,
                                                                    gap.as<uint32_t>());
        check_launch();
    }
    exclusive_scan(gap.as<uint32_t>(), uint64_t(n) + 2);
    // one read-back: overflow flag, statistics and the number of surviving old rows
    PB_CUDA(cudaMemcpyAsync(&ictr->n_keep, pos_a.as<uint32_t>() + n, 4, cudaMemcpyDeviceToDevice, stream));
    const IncCounters fin = read_back<IncCounters>(ictr);
    if (fin.overflow) return false;
    inc_expanded_total += fin.expanded_total;
    const uint32_t n_keep = fin.n_keep;
    const uint64_t n_new64 = uint64_t(n_keep) + side_n;
    if (n_new64 > 0x7fffffffull) throw PacesError("subspace growth: table exceeds 2^31 rows (CSR columns are int32)");
    const uint32_t n_new = uint32_t(n_new64);
    require_memory(uint64_t(n_new) * 16 * 4, "state vectors");

    // ---- new table, full flags, coefficients
    next.words.ensure(size_t(n_new) * W * 4 + 4);
    next.full.ensure(size_t(n_new) + 1);
    c_new.ensure(size_t(n_new) * 16 + 16);
    PB_CUDA(cudaMemsetAsync(c_new.p, 0, size_t(n_new) * 16, stream));
    inc_newidx.ensure(size_t(n) * 4 + 4);
    inc_side_newidx.ensure(size_t(side_n) * 4 + 4);
    inc_scatter_old_kernel<<<grid_for(n), NT, 0, stream>>>(c_old, n, m, dist, pos_a.as<uint32_t>(), gap.as<uint32_t>(),
                                                           inc_newidx.as<uint32_t>(), next.full.as<uint8_t>(),
                                                           c_new.as<double2>(), partials.as<double>(), &c->ticket,
                                                           c->out);
    check_launch();
    PB_DISPATCH_WI(W, inc_copy_rows_kernel<W><<<grid_for(uint64_t(n) * W), NT, 0, stream>>>(
                          old.words.as<uint32_t>(), n, inc_newidx.as<uint32_t>(), next.words.as<uint32_t>()));
    check_launch();
    if (side_n) {
        PB_DISPATCH_WI(W, inc_scatter_side_kernel<W><<<grid_for(side_n), NT, 0, stream>>>(
                              inc_side_keys[scur].as<uint32_t>(), inc_side_gap[scur].as<uint32_t>(),
                              inc_side_dist[scur].as<uint8_t>(), side_n, m, pos_a.as<uint32_t>(),
                              inc_side_newidx.as<uint32_t>(), next.words.as<uint32_t>(), next.full.as<uint8_t>()));
        check_launch();
    }

    // ---- CSR: rows of the side keys (+ symmetric extras), row lengths, fill
    inc_xcnt.ensure(size_t(n) * 4 + 4);
    PB_CUDA(cudaMemsetAsync(inc_xcnt.p, 0, size_t(n) * 4, stream));
    inc_s_col.ensure(size_t(side_n) * width * 4 + 4);
    inc_s_val.ensure(size_t(side_n) * width * 8 + 8);
    inc_s_len.ensure(size_t(side_n) * 4 + 4);
    if (side_n) {
        tmp_col.ensure(size_t(n) * width * 4);  // extras slots of the old rows
        tmp_val.ensure(size_t(n) * width * 8);
        PB_DISPATCH_WI(W, inc_side_rows_kernel<W><<<grid_for(side_n), NT, 0, stream>>>(
                              md, old.words.as<uint32_t>(), n, inc_newidx.as<uint32_t>(),
                              inc_side_keys[scur].as<uint32_t>(), inc_side_newidx.as<uint32_t>(), side_n, width,
                              inc_s_col.as<uint32_t>(), inc_s_val.as<double>(), inc_s_len.as<uint32_t>(),
                              tmp_col.as<uint32_t>(), tmp_val.as<double>(), inc_xcnt.as<uint32_t>()));
        check_launch();
    }
    next.row_ptr.ensure((size_t(n_new) + 1) * 4 + CSR_PAD);
    inc_simple.ensure(size_t(n) + 4);
    inc_row_len_kernel<<<grid_for(uint64_t(n) + side_n), NT, 0, stream>>>(
        n, inc_newidx.as<uint32_t>(), old.row_ptr.as<uint32_t>(), old.col.as<int32_t>(), inc_xcnt.as<uint32_t>(),
        inc_side_newidx.as<uint32_t>(), inc_s_len.as<uint32_t>(), side_n, next.row_ptr.as<uint32_t>(),
        inc_simple.as<uint8_t>());
    check_launch();
    PB_CUDA(cudaMemsetAsync(next.row_ptr.as<uint32_t>() + n_new, 0, 4, stream));
    exclusive_scan(next.row_ptr.as<uint32_t>(), uint64_t(n_new) + 1);
    PB_CUDA(cudaMemcpyAsync(&c->nnz, next.row_ptr.as<uint32_t>() + n_new, 4, cudaMemcpyDeviceToDevice, stream));
    next.col.ensure(size_t(n_new) * width * 4 + CSR_PAD);
    next.val.ensure(size_t(n_new) * width * 8 + CSR_PAD);
    inc_fill_kernel<<<grid_for(uint64_t(n) + side_n), NT, 0, stream>>>(
        n, inc_newidx.as<uint32_t>(), old.row_ptr.as<uint32_t>(), old.col.as<int32_t>(), old.val.as<double>(), width,
        tmp_col.as<uint32_t>(), tmp_val.as<double>(), inc_xcnt.as<uint32_t>(), inc_side_newidx.as<uint32_t>(),
        inc_s_col.as<uint32_t>(), inc_s_val.as<double>(), inc_s_len.as<uint32_t>(), side_n,
        next.row_ptr.as<uint32_t>(), inc_simple.as<uint8_t>(), next.col.as<int32_t>(), next.val.as<double>());
    check_launch();
    inc_fill_simple_kernel<<<grid_for(n), NT, 0, stream>>>(
        n, inc_newidx.as<uint32_t>(), old.row_ptr.as<uint32_t>(), old.col.as<int32_t>(), old.val.as<double>(),
        inc_simple.as<uint8_t>(), next.row_ptr.as<uint32_t>(), next.col.as<int32_t>(), next.val.as<double>());
    check_launch();
    next.n = n_new;
    next.nnz = 0;  // arrives with the step's final read-back (Ctl::nnz)
    next.q_nom = kept;
    next.order = m;
    next.max_row = width;
    next.has_h = true;
    next.has_full = true;
    ++inc_steps;
    inc_side_keys_total += side_n;
    return true;
}

}  // namespace pb
