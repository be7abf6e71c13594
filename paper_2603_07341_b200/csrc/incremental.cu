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
    PB_CUDA(cudaMemsetAsync(ictr, 0, sizeof(IncCounters), stream));

    // ---- capacities.  Nothing below is sized by a count the host would have to read back first: more new keys than
    // a quarter of the old rows (not a steady state) or more candidates than the buffer holds only raise `overflow`,
    // and the step is redone by the full path.
    const uint32_t side_cap = n / 4 + (1u << 16);
    const uint64_t n_bound = uint64_t(n) + side_cap;
    if (n_bound > 0x7fffffffull) return false;
    {
        const uint64_t want = std::max<uint64_t>(uint64_t(n / 8 + 1024) * uint64_t(std::max(nmoves, 1)), 1u << 16);
        cand_keys.ensure(size_t(want) * W * 4);
        cand_gap.ensure(size_t(want) * 4);
    }
    const uint32_t cand_cap =
        uint32_t(std::min<uint64_t>({cand_keys.cap / (size_t(W) * 4), cand_gap.cap / 4, 0x7ffffff0ull}));
    perm.ensure(size_t(cand_cap) * 4 + 4);
    seg_rank.ensure(size_t(cand_cap) * 4 + 4);
    for (int i = 0; i < 2; ++i) {
        inc_side_keys[i].ensure(size_t(side_cap) * W * 4 + 64);
        inc_side_gap[i].ensure(size_t(side_cap) * 4 + 64);
        inc_side_dist[i].ensure(size_t(side_cap) + 64);
    }
    inc_new_keys.ensure(size_t(cand_cap) * W * 4 + 64);
    inc_new_gap.ensure(size_t(cand_cap) * 4 + 64);
    inc_elist.ensure(size_t(n) * 4 + 4);
    // candidates are bucketed by (insertion gap >> sh): ~64 K buckets whatever the table size
    int sh = 0;
    while ((uint64_t(n) >> sh) > (1u << 16)) ++sh;
    const uint32_t nbuckets = uint32_t(uint64_t(n) >> sh) + 1;  // gaps run over [0, n]
    const size_t bstride = (size_t(nbuckets) + 2 + 3) & ~size_t(3);  // the scan reads 16-byte vectors: keep them aligned
    inc_buckets.ensure(3 * bstride * 4);
    uint32_t* b_start = inc_buckets.as<uint32_t>();   // counts -> segment starts
    uint32_t* b_fill = b_start + bstride;             // placement cursors
    uint32_t* b_kept = b_fill + bstride;              // survivors -> kept_before
    uint8_t* dist = inc_dist.as<uint8_t>();           // 0 on the kept rows, DIST_INF elsewhere (select())
    const int small_grid = sm_count * 4;

    int scur = 0;
    for (int k = 0; k < m; ++k) {
        inc_level_kernel<<<grid_for(n), NT, 0, stream>>>(n, k, old.full.as<uint8_t>(), old.row_ptr.as<uint32_t>(),
                                                          old.col.as<int32_t>(), dist, inc_elist.as<uint32_t>(), ictr);
        check_launch();
        if (nmoves == 0) continue;
        PB_CUDA(cudaMemsetAsync(b_start, 0, 3 * bstride * 4, stream));
        PB_DISPATCH_WI(W, inc_expand_kernel<W><<<small_grid, NT, 0, stream>>>(
                              md, old.words.as<uint32_t>(), n, inc_elist.as<uint32_t>(),
                              inc_side_keys[scur].as<uint32_t>(), inc_side_dist[scur].as<uint8_t>(), k, nmoves, dist,
                              cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), cand_cap, sh, b_start, ictr));
        check_launch();
        // unique new keys of this level in canonical order: counting sort by bucket, dedup + rank inside the buckets
        const uint32_t* nc_ptr = &ictr->n_cand[k];
        exclusive_scan(b_start, uint64_t(nbuckets) + 1);
        place_candidates_kernel<<<small_grid, NT, 0, stream>>>(cand_gap.as<uint32_t>(), nc_ptr, cand_cap, sh, b_start,
                                                               b_fill, perm.as<uint32_t>());
        check_launch();
        PB_DISPATCH_WI(W, segment_dedup_kernel<W><<<small_grid, NT, 0, stream>>>(
                              cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), perm.as<uint32_t>(), nc_ptr, cand_cap, sh,
                              b_start, seg_rank.as<uint32_t>(), b_kept, nullptr));
        check_launch();
        PB_DISPATCH_WI(W, segment_rank_kernel<W><<<small_grid, NT, 0, stream>>>(
                              cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), perm.as<uint32_t>(), nc_ptr, cand_cap, sh,
                              b_start, seg_rank.as<uint32_t>()));
        check_launch();
        exclusive_scan(b_kept, uint64_t(nbuckets) + 1);
        PB_DISPATCH_WI(W, inc_emit_unique_kernel<W><<<small_grid, NT, 0, stream>>>(
                              cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), perm.as<uint32_t>(),
                              seg_rank.as<uint32_t>(), k, cand_cap, sh, b_kept, nbuckets, inc_new_keys.as<uint32_t>(),
                              inc_new_gap.as<uint32_t>(), ictr));
        check_launch();
        PB_DISPATCH_WI(W, inc_side_merge_kernel<W><<<small_grid, NT, 0, stream>>>(
                              inc_side_keys[scur].as<uint32_t>(), inc_side_gap[scur].as<uint32_t>(),
                              inc_side_dist[scur].as<uint8_t>(), inc_new_keys.as<uint32_t>(), inc_new_gap.as<uint32_t>(), k,
                              side_cap, inc_side_keys[scur ^ 1].as<uint32_t>(), inc_side_gap[scur ^ 1].as<uint32_t>(),
                              inc_side_dist[scur ^ 1].as<uint8_t>(), ictr));
        check_launch();
        scur ^= 1;
    }
    const int levels = nmoves == 0 ? 0 : m;  // index of the final side count in IncCounters::side_n

    // ---- from the distances to the new space (see incremental.cuh): side-key neighbours, per-tile reductions, one
    // small scan, then one pass over the old rows for the index maps / table / coefficients / row pointer and one for
    // the entries
    next.words.ensure(size_t(n_bound) * W * 4 + 64);
    next.full.ensure(size_t(n_bound) + 64);
    c_new.ensure(size_t(n_bound) * 16 + 16);
    inc_newidx.ensure(size_t(n) * 4 + 4);
    inc_side_newidx.ensure(size_t(side_cap) * 4 + 4);
    inc_s_col.ensure(size_t(side_cap) * width * 4 + 4);
    inc_s_val.ensure(size_t(side_cap) * width * 8 + 8);
    inc_has_extra.ensure(size_t(n) + 64);  // `touched` flags: bit 0 = the row loses an entry, bit 1 = it gains one
    inc_simple.ensure(size_t(n) + 64);
    inc_row_len.ensure(size_t(n) + 64);
    const uint32_t ctiles = uint32_t((uint64_t(n) + 1 + INC_TILE - 1) / INC_TILE);
    inc_tile_jlo.ensure((size_t(ctiles) + 2) * 4 * 3);
    uint32_t* tile_jlo = inc_tile_jlo.as<uint32_t>();
    uint32_t* tile_keep = tile_jlo + (ctiles + 2);
    uint32_t* tile_nnz = tile_keep + (ctiles + 2);
    next.row_ptr.ensure((size_t(n_bound) + 1) * 4 + CSR_PAD);
    next.col.ensure(size_t(n_bound) * width * 4 + CSR_PAD);
    uint8_t* touched = inc_has_extra.as<uint8_t>();
    PB_CUDA(cudaMemsetAsync(touched, 0, size_t(n) + 1, stream));
    // value codes (taylor.cuh) travel with the entries when the previous space has them
    const bool carry_codes = use_codes && old.has_code && md.vt_n > 0;
    if (carry_codes) {
        inc_s_code.ensure(size_t(side_cap) * width * 2 + 4);
        next.code.ensure(size_t(n_bound) * width * 2 + CSR_PAD);
        if (!md.vt_diag) next.diag.ensure(size_t(n_bound) * 8 + CSR_PAD);
    }
    uint16_t* s_code = carry_codes ? inc_s_code.as<uint16_t>() : nullptr;
    // a coded space leaves the 8-byte values behind: the Taylor tile kernels read the codes (ensure_val() decodes)
    const bool with_val = !(carry_codes && drop_val);
    if (with_val) {
        ensure_val(old);
        next.val.ensure(size_t(n_bound) * width * 8 + CSR_PAD);
    }
    const uint32_t* skeys = inc_side_keys[scur].as<uint32_t>();
    const uint32_t* sgap = inc_side_gap[scur].as<uint32_t>();
    PB_DISPATCH_WI(W, inc_side_search_kernel<W><<<small_grid, NT, 0, stream>>>(
                          md, old.words.as<uint32_t>(), n, m, levels, dist, skeys, width, inc_s_col.as<uint32_t>(),
                          inc_s_val.as<double>(), s_code, touched, ictr));
    check_launch();
    // surviving old rows that gain entries: at most nmoves per side key; more than x_cap of them -> overflow
    const uint32_t x_cap = uint32_t(std::min<uint64_t>(uint64_t(n), uint64_t(side_cap) * 2));
    const int xs = std::max(nmoves, 1);
    inc_xlist.ensure(size_t(x_cap) * 4 + 4);
    inc_x_slot.ensure(size_t(n) * 4 + 4);
    inc_x_ref.ensure(size_t(x_cap) * xs * 4 + 4);
    inc_x_val.ensure(size_t(x_cap) * xs * 8 + 8);
    if (carry_codes) inc_x_code.ensure(size_t(x_cap) * xs * 2 + 4);
    uint16_t* x_code = carry_codes ? inc_x_code.as<uint16_t>() : nullptr;
    inc_tile_prep_kernel<<<ctiles, NT, 0, stream>>>(n, m, levels, dist, old.row_ptr.as<uint32_t>(), old.col.as<int32_t>(),
                                                    sgap, tile_keep, tile_jlo, ctiles, touched, inc_xlist.as<uint32_t>(),
                                                    inc_x_slot.as<uint32_t>(), x_cap, ictr);
    check_launch();
    PB_DISPATCH_WI(W, inc_extras_kernel<W><<<small_grid, NT, 0, stream>>>(
                          md, old.words.as<uint32_t>(), levels, inc_xlist.as<uint32_t>(), x_cap, skeys, xs,
                          inc_x_ref.as<uint32_t>(), inc_x_val.as<double>(), x_code, ictr));
    check_launch();
    inc_tile_nnz_kernel<<<ctiles, NT, 0, stream>>>(n, m, dist, touched, old.row_ptr.as<uint32_t>(), old.col.as<int32_t>(),
                                                   inc_x_slot.as<uint32_t>(), inc_x_ref.as<uint32_t>(), xs,
                                                   inc_s_col.as<uint32_t>(), width, tile_jlo, tile_nnz,
                                                   inc_row_len.as<uint8_t>(), inc_simple.as<uint8_t>());
    check_launch();
    inc_tile_scan_kernel<<<1, NT, 0, stream>>>(tile_keep, tile_nnz, ctiles, levels, ictr);
    check_launch();
    PB_DISPATCH_WI(W, inc_compact_kernel<W><<<ctiles, NT, 0, stream>>>(
                          n, m, levels, dist, inc_row_len.as<uint8_t>(), skeys, sgap, inc_side_dist[scur].as<uint8_t>(),
                          inc_s_col.as<uint32_t>(), width, tile_jlo, tile_keep, tile_nnz, inc_newidx.as<uint32_t>(),
                          inc_side_newidx.as<uint32_t>(), next.words.as<uint32_t>(), next.full.as<uint8_t>(),
                          c_new.as<double2>(), next.row_ptr.as<uint32_t>(), ctiles, ictr));
    check_launch();
    {
        // the bulk of the bytes: keys, flags and coefficients of the surviving old rows, one streaming pass
        const int mg = grid_for(n);
        if (size_t(mg) * 8 > partials.cap) throw CudaFail("internal error: reduction scratch too small for the grid");
        PB_DISPATCH_WI(W, inc_move_kernel<W><<<mg, NT, 0, stream>>>(
                              old.words.as<uint32_t>(), c_old, n, m, dist, inc_newidx.as<uint32_t>(),
                              next.words.as<uint32_t>(), next.full.as<uint8_t>(), c_new.as<double2>(),
                              partials.as<double>(), &c->ticket, c->out));
        check_launch();
    }
    inc_fill_kernel<<<grid_for(n), NT, 0, stream>>>(
        n, levels, inc_newidx.as<uint32_t>(), touched, old.row_ptr.as<uint32_t>(), old.col.as<int32_t>(),
        with_val ? old.val.as<double>() : nullptr, inc_x_slot.as<uint32_t>(), inc_x_ref.as<uint32_t>(),
        inc_x_val.as<double>(), xs,
        inc_side_newidx.as<uint32_t>(), inc_s_col.as<uint32_t>(), inc_s_val.as<double>(), width,
        next.row_ptr.as<uint32_t>(), inc_simple.as<uint8_t>(), next.col.as<int32_t>(),
        with_val ? next.val.as<double>() : nullptr, ictr, carry_codes ? old.code.as<uint16_t>() : nullptr,
        (carry_codes && !md.vt_diag) ? old.diag.as<double>() : nullptr, x_code, s_code, next.code.as<uint16_t>(),
        next.diag.as<double>());
    check_launch();

    // value codes of the new CSR (taylor.cuh): the row count is still on the device
    next.max_row = width;
    next.has_code = false;
    // (the previous space had none -- e.g. its values were not all tabulated --: one pass over the finished CSR)
    const bool coded = carry_codes || encode_values_async(next, n_bound, n_bound * uint64_t(width), &ictr->h.n_new,
                                                          &ictr->h.code_fail);

    // ---- the one read-back of the phase
    const IncHead fin = read_back<IncHead>(&ictr->h);
    if (fin.overflow) return false;
    if (!with_val && fin.code_fail) return false;  // a value outside the table and no values carried: full path
    next.has_code = coded && fin.code_fail == 0;
    next.val_valid = with_val;
    if (uint64_t(fin.n_new) > 0x7fffffffull) throw PacesError("subspace growth: table exceeds 2^31 rows (CSR columns are int32)");
    PB_CUDA(cudaMemcpyAsync(&c->nnz, &ictr->h.nnz_new, 4, cudaMemcpyDeviceToDevice, stream));
    inc_expanded_total += fin.expanded_total;
    next.n = fin.n_new;
    next.nnz = fin.nnz_new;
    next.q_nom = kept;
    next.order = m;
    next.max_row = width;
    next.has_h = true;
    next.has_full = true;
    ++inc_steps;
    inc_side_keys_total += fin.side_total;
    return true;
}

}  // namespace pb
