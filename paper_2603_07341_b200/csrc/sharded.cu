// sharded.cu -- multi-GPU orchestration: one context per rank, rows sharded by owner_of(key).
// Every method here is COLLECTIVE: all ranks call it in the same order.  Data-path exchanges:
//   expansion   : candidate keys owned elsewhere            (all-to-all-v of keys, once per BFS order)
//   assembly    : neighbour key -> owner-local row look-ups (all-to-all-v of keys, all-to-all-v of u32 replies)
//   Taylor order: complex128 halo values                    (all-to-all-v, once per order) + 2-double all-reduce
//   selection   : 2048-bin histogram all-reduce per radix pass; tie keys gathered and drawn identically everywhere
// Row sums keep the reference's order (entries sorted by neighbour key), so amplitudes do not depend on P.
#include "engine.cuh"

namespace pb {

#ifdef PB_ONLY_W  // development / profiling builds: one key width, small module, fast compile
#define PB_DISPATCH_WS(Wv, ...)                                  \
    switch (Wv) {                                               \
        case PB_ONLY_W: { constexpr int W = PB_ONLY_W; __VA_ARGS__; } break; \
        default: throw PacesError("this development build only supports one key width (PB_ONLY_W)"); \
    }
#else
#define PB_DISPATCH_WS(Wv, ...)                                 \
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
// routing helpers
// ------------------------------------------------------------------------------------------------
RouteBlock* Engine::route_block() {
    route_ctr.ensure(sizeof(RouteBlock));
    return route_ctr.as<RouteBlock>();
}

void Engine::route_async(const uint32_t* dest, const uint32_t* cnt_ptr, uint32_t cnt_bound, uint32_t* pos) {
    const uint32_t P = uint32_t(world);
    RouteBlock* rb = route_block();
    PB_CUDA(cudaMemsetAsync(rb->fill, 0, sizeof(rb->fill) + sizeof(rb->displ), stream));
    PB_CUDA(cudaMemsetAsync(rb->counts, 0, sizeof(rb->counts) + sizeof(rb->rcounts), stream));
    const int g = grid_for(cnt_bound);
    route_count_kernel<<<g, NT, 0, stream>>>(dest, cnt_ptr, cnt_bound, P, rb->counts);
    check_launch();
    route_scan_kernel<<<1, 32, 0, stream>>>(rb->counts, P, rb->displ);
    check_launch();
    route_place_kernel<<<g, NT, 0, stream>>>(dest, cnt_ptr, cnt_bound, rb->displ, rb->fill, pos);
    check_launch();
    // every peer learns how much it will receive: one u32 per pair, on the device
    std::vector<uint64_t> ones(P, 1);
    comm_check(ops.alltoallv_dev(ops.user, rb->counts, ones.data(), rb->rcounts, ones.data(), 4, stream),
               "alltoallv_dev(counts)");
}

ShardCounters Engine::route_finish() {
    const uint32_t P = uint32_t(world);
    const RouteInfo info = read_back<RouteInfo>(&route_block()->sc);
    h_send.assign(P, 0);
    h_recv.assign(P, 0);
    for (uint32_t p = 0; p < P; ++p) {
        h_send[p] = info.counts[p];
        h_recv[p] = info.rcounts[p];
    }
    return info.sc;
}

uint64_t Engine::exchange_known(const void* send, DevBuf& recv, uint64_t elem_bytes) {
    uint64_t total = 0;
    for (uint64_t v : h_recv) total += v;
    recv.ensure(total * elem_bytes + 16);
    comm_check(ops.alltoallv_dev(ops.user, send, h_send.data(), recv.p, h_recv.data(), elem_bytes, stream),
               "alltoallv_dev");
    return total;
}

void Engine::halo_exchange(const Space& sp, double2* x) {
    halo_stage.ensure(size_t(sp.send_total) * 16 + 16);
    if (sp.send_total) {
        halo_pack_kernel<<<grid_for(sp.send_total), NT, 0, stream>>>(x, sp.send_idx.as<uint32_t>(), sp.send_total,
                                                                     halo_stage.as<double2>());
        check_launch();
    }
    comm_check(ops.alltoallv_dev(ops.user, halo_stage.p, sp.halo_send.data(), x + sp.n, sp.halo_recv.data(), 16, stream),
               "alltoallv_dev(halo)");
}

void Engine::halo_start(const Space& sp, double2* x) {
    halo_stage.ensure(size_t(sp.send_total) * 16 + 16);
    if (sp.send_total) {
        halo_pack_kernel<<<grid_for(sp.send_total), NT, 0, stream>>>(x, sp.send_idx.as<uint32_t>(), sp.send_total,
                                                                     halo_stage.as<double2>());
        check_launch();
    }
    if (ops.alltoallv_dev2) {
        // independent channel: the exchange runs on its own stream beside the rows that need no halo
        PB_CUDA(cudaEventRecord(ev_pack, stream));
        PB_CUDA(cudaStreamWaitEvent(halo_stream, ev_pack, 0));
        comm_check(ops.alltoallv_dev2(ops.user, halo_stage.p, sp.halo_send.data(), x + sp.n, sp.halo_recv.data(), 16,
                                      halo_stream),
                   "alltoallv_dev2(halo)");
        PB_CUDA(cudaEventRecord(ev_halo, halo_stream));
    } else {
        comm_check(ops.alltoallv_dev(ops.user, halo_stage.p, sp.halo_send.data(), x + sp.n, sp.halo_recv.data(), 16, stream),
                   "alltoallv_dev(halo)");
    }
}

void Engine::halo_wait() {
    if (ops.alltoallv_dev2) PB_CUDA(cudaStreamWaitEvent(stream, ev_halo, 0));
}

/// Splits the rows of a sharded space into those without halo columns (they can run while the halo is in flight)
/// and those with.
void Engine::classify_rows(Space& sp) {
    const uint32_t n = sp.n;
    row_class.ensure((size_t(n) + 1) * 4 + 8);
    uint32_t* flag = row_class.as<uint32_t>();
    row_has_halo_kernel<<<grid_for(uint64_t(n) + 1), NT, 0, stream>>>(n, sp.row_ptr.as<uint32_t>(), sp.col.as<int32_t>(), flag);
    check_launch();
    scan_aligned.ensure((size_t(n) + 1) * 4 + 64);
    PB_CUDA(cudaMemcpyAsync(scan_aligned.p, flag, (size_t(n) + 1) * 4, cudaMemcpyDeviceToDevice, stream));
    exclusive_scan(scan_aligned.as<uint32_t>(), uint64_t(n) + 1);
    const uint32_t nb = read_back<uint32_t>(scan_aligned.as<uint32_t>() + n);
    sp.n_boundary = nb;
    sp.n_interior = n - nb;
    sp.row_lists = true;
    sp.rows_int.ensure(size_t(sp.n_interior) * 4 + 4);
    sp.rows_bnd.ensure(size_t(nb) * 4 + 4);
    if (n) {
        split_rows_kernel<<<grid_for(n), NT, 0, stream>>>(n, flag, scan_aligned.as<uint32_t>(), sp.rows_int.as<uint32_t>(),
                                                          sp.rows_bnd.as<uint32_t>());
        check_launch();
    }
}

// ------------------------------------------------------------------------------------------------
// grow_subspace on shards
// ------------------------------------------------------------------------------------------------
void Engine::grow_sharded(const uint32_t* d_seeds, uint32_t ns, int order, Space& out) {
    require_model();
    if (order < 0) throw PacesError("grow_subspace: neighbor order must be >= 0");
    const uint64_t ns_global = allreduce_host_u64(ns);
    if (ns_global == 0) throw PacesError("grow_subspace: empty seed set");
    const int W = md.W;
    const uint32_t P = uint32_t(world);
    const int nmoves = md.max_deg + (md.kind == 1 ? 2 : 0);
    out.words.ensure(size_t(ns) * W * 4 + 4);
    if (ns) PB_CUDA(cudaMemcpyAsync(out.words.p, d_seeds, size_t(ns) * W * 4, cudaMemcpyDeviceToDevice, stream));
    uint32_t n = ns, nf = ns;
    bool identity_frontier = true;
    int fcur = 0;
    Ctl* c = dctl();
    ShardCounters* dsc = &route_block()->sc;

    int levels_done = 0;
    for (int k = 0; k < order; ++k, ++levels_done) {
        if (allreduce_host_u64(nf) == 0) break;  // every frontier is empty: the ball is complete
        const uint64_t cap64 = uint64_t(nf) * uint64_t(nmoves) + 1;
        if (cap64 > 0x7ffffff0ull) throw PacesError("subspace growth: candidate count exceeds 32-bit indexing");
        const uint32_t cap = uint32_t(cap64);
        cand_keys.ensure(size_t(cap) * W * 4);
        cand_gap.ensure(size_t(cap) * 4);
        out_keys.ensure(size_t(cap) * W * 4);
        out_dest.ensure(size_t(cap) * 4);
        route_pos.ensure(size_t(cap) * 4);
        sendbuf.ensure(size_t(cap) * W * 4 + 16);
        gap.ensure((size_t(n) + 2) * 4);
        PB_CUDA(cudaMemsetAsync(gap.p, 0, (size_t(n) + 2) * 4, stream));
        PB_CUDA(cudaMemsetAsync(&c->grow, 0, sizeof(GrowCounters), stream));
        PB_CUDA(cudaMemsetAsync(dsc, 0, sizeof(ShardCounters), stream));
        const uint32_t* fr = identity_frontier ? nullptr : frontier[fcur].as<uint32_t>();
        const uint32_t xchunk = chunk_for(nf);
        if (nf) {
            PB_DISPATCH_WS(W, expand_level_sharded_kernel<W><<<grid_chunked(nf, xchunk), NT, 0, stream>>>(
                                  md, uint32_t(rank), P, out.words.as<uint32_t>(), n, fr, nf, xchunk,
                                  cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), cap, gap.as<uint32_t>(), &c->grow,
                                  out_keys.as<uint32_t>(), out_dest.as<uint32_t>(), cap, dsc));
            check_launch();
        }
        // ship the keys owned by other ranks: bucketing, payload scatter and the exchange of the per-peer counts are
        // enqueued against the device-side count; ONE read-back then tells the host what to send and what arrives
        route_async(out_dest.as<uint32_t>(), &dsc->n_out, cap, route_pos.as<uint32_t>());
        PB_DISPATCH_WS(W, route_scatter_keys_kernel<W><<<grid_for(cap), NT, 0, stream>>>(
                              out_keys.as<uint32_t>(), route_pos.as<uint32_t>(), &dsc->n_out, cap, sendbuf.as<uint32_t>()));
        check_launch();
        const ShardCounters hsc = route_finish();
        if (hsc.overflow) throw CudaFail("internal error: candidate buffer overflow during expansion");
        const uint64_t nr = exchange_known(sendbuf.p, recvbuf, uint64_t(W) * 4);
        if (nr) {
            // the local candidates (at most cap - 1 of them, their count is still on the device) keep their places
            const uint64_t need = uint64_t(cap) + nr;
            if (need > 0x7ffffff0ull) throw PacesError("subspace growth: candidate count exceeds 32-bit indexing");
            if (size_t(need) * W * 4 > cand_keys.cap || size_t(need) * 4 > cand_gap.cap) {
                sync();
                cand_keys.ensure_keep(size_t(need) * W * 4, size_t(cap) * W * 4);
                cand_gap.ensure_keep(size_t(need) * 4, size_t(cap) * 4);
            }
            PB_DISPATCH_WS(W, classify_received_kernel<W><<<grid_for(nr), NT, 0, stream>>>(
                                  out.words.as<uint32_t>(), n, recvbuf.as<uint32_t>(), uint32_t(nr),
                                  cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), uint32_t(need), gap.as<uint32_t>(),
                                  &c->grow));
            check_launch();
        }
        const GrowCounters gc = read_back<GrowCounters>(&c->grow);
        if (gc.overflow) throw CudaFail("internal error: candidate buffer overflow during expansion");
        const uint32_t nc = gc.n_cand;
        uint32_t n_new = 0;
        if (nc) n_new = merge_level(out, n, nc, fcur);
        identity_frontier = false;
        if (!nc) {
            // nothing new on this rank: the next frontier is empty, the table is unchanged
            frontier[fcur].ensure(4);
        }
        n += n_new;
        nf = n_new;
    }
    out.n = n;
    out.q_nom = ns_global;
    out.order = order;
    // which rows had their neighbourhood generated (remote neighbours included: they went to their owners): all but the
    // last frontier, when every order ran (the incremental growth of the next step needs it)
    out.full.ensure(size_t(n) + 1);
    PB_CUDA(cudaMemsetAsync(out.full.p, order == 0 ? 0 : 1, n, stream));
    if (order > 0 && levels_done == order && nf > 0 && !identity_frontier) {
        inc_clear_full_kernel<<<grid_for(nf), NT, 0, stream>>>(frontier[fcur].as<uint32_t>(), nf, out.full.as<uint8_t>());
        check_launch();
    }
    out.has_full = true;
    PB_CUDA(cudaEventRecord(ev[2], stream));
    assemble_sharded(out);
}

// ------------------------------------------------------------------------------------------------
// grow_subspace on shards, incremental: the new TABLE from the previous space (sharded.cuh, "Incremental TABLE growth
// on a shard"); H_eff of the new table is then assembled the usual way.  Collective; returns false on every rank when
// any rank hit a buffer bound (the caller then runs grow_sharded from the kept keys).
// ------------------------------------------------------------------------------------------------
bool Engine::grow_incremental_sharded(const Space& old, const double2* c_old, uint64_t kept_global, int m, Space& next,
                                      DevBuf& c_new) {
    const int W = md.W;
    const uint32_t P = uint32_t(world);
    const uint32_t n = old.n;
    const int nmoves = md.max_deg + (md.kind == 1 ? 2 : 0);
    Ctl* c = dctl();
    inc_ctr.ensure(sizeof(IncCounters));
    IncCounters* ictr = inc_ctr.as<IncCounters>();
    PB_CUDA(cudaMemsetAsync(ictr, 0, sizeof(IncCounters), stream));
    ShardCounters* dsc = &route_block()->sc;

    // capacities (as incremental.cu): nothing is sized by a count the host would have to read first; a bound that is
    // hit only raises `overflow`
    const uint32_t side_cap = n / 4 + (1u << 16);
    const uint64_t n_bound = uint64_t(n) + side_cap;
    bool local_fail = n_bound > 0x7fffffffull;
    {
        const uint64_t want = std::max<uint64_t>(uint64_t(n / 8 + 1024) * uint64_t(std::max(nmoves, 1)), 1u << 16);
        cand_keys.ensure(size_t(want) * W * 4);
        cand_gap.ensure(size_t(want) * 4);
    }
    const uint32_t cand_cap =
        uint32_t(std::min<uint64_t>({cand_keys.cap / (size_t(W) * 4), cand_gap.cap / 4, 0x7ffffff0ull}));
    const uint32_t out_cap = cand_cap;
    out_keys.ensure(size_t(out_cap) * W * 4);
    out_dest.ensure(size_t(out_cap) * 4);
    route_pos.ensure(size_t(out_cap) * 4);
    sendbuf.ensure(size_t(out_cap) * W * 4 + 16);
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
    int sh = 0;
    while ((uint64_t(n) >> sh) > (1u << 16)) ++sh;
    const uint32_t nbuckets = uint32_t(uint64_t(n) >> sh) + 1;  // gaps run over [0, n]
    const size_t bstride = (size_t(nbuckets) + 2 + 3) & ~size_t(3);
    inc_buckets.ensure(3 * bstride * 4);
    uint32_t* b_start = inc_buckets.as<uint32_t>();
    uint32_t* b_fill = b_start + bstride;
    uint32_t* b_kept = b_fill + bstride;
    const int small_grid = sm_count * 4;

    // distances: 0 on the kept rows (select_sharded's flags), the halo slots behind the local rows
    const uint32_t n_ext = n + old.halo_n;
    inc_dist.ensure(size_t(n_ext) + 16);
    uint8_t* dist = inc_dist.as<uint8_t>();
    inc_dist_from_keep_kernel<<<grid_for(n_ext), NT, 0, stream>>>(flag_keep.as<uint32_t>(), n, n_ext, dist);
    check_launch();
    halo_stage.ensure(size_t(old.send_total) + 16);

    int scur = 0;
    for (int k = 0; k < m; ++k) {
        // the owners' distances of my halo rows (one byte per halo entry; the SpMV's pack lists carry them)
        if (old.send_total) {
            halo_pack_u8_kernel<<<grid_for(old.send_total), NT, 0, stream>>>(dist, old.send_idx.as<uint32_t>(), old.send_total,
                                                                             halo_stage.as<uint8_t>());
            check_launch();
        }
        comm_check(ops.alltoallv_dev(ops.user, halo_stage.p, old.halo_send.data(), dist + n, old.halo_recv.data(), 1, stream),
                   "alltoallv_dev(distances)");
        inc_level_kernel<<<grid_for(n), NT, 0, stream>>>(n, k, old.full.as<uint8_t>(), old.row_ptr.as<uint32_t>(),
                                                          old.col.as<int32_t>(), dist, inc_elist.as<uint32_t>(), ictr);
        check_launch();
        PB_CUDA(cudaMemsetAsync(b_start, 0, 3 * bstride * 4, stream));
        PB_CUDA(cudaMemsetAsync(dsc, 0, sizeof(ShardCounters), stream));
        PB_DISPATCH_WS(W, inc_expand_sharded_kernel<W><<<small_grid, NT, 0, stream>>>(
                              md, uint32_t(rank), P, old.words.as<uint32_t>(), n, inc_elist.as<uint32_t>(),
                              inc_side_keys[scur].as<uint32_t>(), inc_side_dist[scur].as<uint8_t>(), k, nmoves, dist,
                              cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), cand_cap, sh, b_start, ictr,
                              out_keys.as<uint32_t>(), out_dest.as<uint32_t>(), out_cap, dsc));
        check_launch();
        // neighbours owned elsewhere -> their owners (device-side count, one read-back)
        route_async(out_dest.as<uint32_t>(), &dsc->n_out, out_cap, route_pos.as<uint32_t>());
        PB_DISPATCH_WS(W, route_scatter_keys_kernel<W><<<grid_for(out_cap), NT, 0, stream>>>(
                              out_keys.as<uint32_t>(), route_pos.as<uint32_t>(), &dsc->n_out, out_cap, sendbuf.as<uint32_t>()));
        check_launch();
        const ShardCounters hsc = route_finish();
        if (hsc.overflow) local_fail = true;  // (the exchange still runs: every rank keeps the same sequence of collectives)
        const uint64_t nr = exchange_known(sendbuf.p, recvbuf, uint64_t(W) * 4);
        if (nr) {
            PB_DISPATCH_WS(W, inc_classify_received_kernel<W><<<grid_for(nr), NT, 0, stream>>>(
                                  old.words.as<uint32_t>(), n, inc_side_keys[scur].as<uint32_t>(), k, recvbuf.as<uint32_t>(),
                                  uint32_t(nr), dist, cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), cand_cap, sh, b_start,
                                  ictr));
            check_launch();
        }
        // unique new keys of this level in canonical order, merged into the side list (incremental.cu's chain)
        const uint32_t* nc_ptr = &ictr->n_cand[k];
        exclusive_scan(b_start, uint64_t(nbuckets) + 1);
        place_candidates_kernel<<<small_grid, NT, 0, stream>>>(cand_gap.as<uint32_t>(), nc_ptr, cand_cap, sh, b_start,
                                                               b_fill, perm.as<uint32_t>());
        check_launch();
        PB_DISPATCH_WS(W, segment_dedup_kernel<W><<<small_grid, NT, 0, stream>>>(
                              cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), perm.as<uint32_t>(), nc_ptr, cand_cap, sh,
                              b_start, seg_rank.as<uint32_t>(), b_kept, nullptr));
        check_launch();
        PB_DISPATCH_WS(W, segment_rank_kernel<W><<<small_grid, NT, 0, stream>>>(
                              cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), perm.as<uint32_t>(), nc_ptr, cand_cap, sh,
                              b_start, seg_rank.as<uint32_t>()));
        check_launch();
        exclusive_scan(b_kept, uint64_t(nbuckets) + 1);
        PB_DISPATCH_WS(W, inc_emit_unique_kernel<W><<<small_grid, NT, 0, stream>>>(
                              cand_keys.as<uint32_t>(), cand_gap.as<uint32_t>(), perm.as<uint32_t>(),
                              seg_rank.as<uint32_t>(), k, cand_cap, sh, b_kept, nbuckets, inc_new_keys.as<uint32_t>(),
                              inc_new_gap.as<uint32_t>(), ictr));
        check_launch();
        PB_DISPATCH_WS(W, inc_side_merge_kernel<W><<<small_grid, NT, 0, stream>>>(
                              inc_side_keys[scur].as<uint32_t>(), inc_side_gap[scur].as<uint32_t>(),
                              inc_side_dist[scur].as<uint8_t>(), inc_new_keys.as<uint32_t>(), inc_new_gap.as<uint32_t>(), k,
                              side_cap, inc_side_keys[scur ^ 1].as<uint32_t>(), inc_side_gap[scur ^ 1].as<uint32_t>(),
                              inc_side_dist[scur ^ 1].as<uint8_t>(), ictr));
        check_launch();
        scur ^= 1;
    }

    // ---- the new table: survivors (distance <= m) and side keys at their merged positions
    inc_newidx.ensure((size_t(n) + 2) * 4);  // add[]
    pos_a.ensure((size_t(n) + 2) * 4);       // v[] -> its exclusive scan
    uint32_t* add = inc_newidx.as<uint32_t>();
    uint32_t* vs = pos_a.as<uint32_t>();
    PB_CUDA(cudaMemsetAsync(add, 0, (size_t(n) + 2) * 4, stream));
    inc_shard_mark_kernel<<<small_grid, NT, 0, stream>>>(inc_side_gap[scur].as<uint32_t>(), m, ictr, add);
    check_launch();
    inc_shard_count_kernel<<<grid_for(uint64_t(n) + 1), NT, 0, stream>>>(n, m, dist, add, vs);
    check_launch();
    exclusive_scan(vs, uint64_t(n) + 2);
    inc_shard_head_kernel<<<1, 32, 0, stream>>>(n, vs, m, ictr);
    check_launch();
    {
        // test hook: rank 0 pretends to have hit a bound on every k-th step (the other ranks must follow it)
        static const char* fe = std::getenv("PB200_SHARD_INC_FAIL_EVERY");
        if (fe != nullptr && rank == 0 && std::atoi(fe) > 0 && steps_done % uint64_t(std::atoi(fe)) == 0) local_fail = true;
    }
    // any rank's overflow sends every rank to the full path: the flags are summed on the device, the one read-back of
    // the phase brings the verdict with the sizes
    if (local_fail) PB_CUDA(cudaMemsetAsync(&ictr->h.overflow, 1, 4, stream));
    comm_check(ops.allreduce_u32_dev(ops.user, &ictr->h.overflow, 1, stream), "allreduce_u32_dev(overflow)");
    const IncHead fin = read_back<IncHead>(&ictr->h);
    if (fin.overflow != 0) return false;
    if (uint64_t(fin.n_new) > 0x7fffffffull) throw PacesError("subspace growth: table exceeds 2^31 rows (CSR columns are int32)");
    next.words.ensure(size_t(fin.n_new) * W * 4 + 64);
    next.full.ensure(size_t(fin.n_new) + 64);
    inc_inv.ensure(size_t(fin.n_new) * 4 + 4);  // origin of every new row
    PB_DISPATCH_WS(W, inc_shard_table_kernel<W><<<grid_for(std::max<uint64_t>(n, fin.side_total)), NT, 0, stream>>>(
                          n, m, m, dist, old.words.as<uint32_t>(), inc_side_keys[scur].as<uint32_t>(),
                          inc_side_gap[scur].as<uint32_t>(), inc_side_dist[scur].as<uint8_t>(), add, vs, ictr,
                          next.words.as<uint32_t>(), next.full.as<uint8_t>(), inc_inv.as<uint32_t>()));
    check_launch();
    // the assembly hint: surviving rows next to a local side key are searched, the others read the previous H_eff
    AsmHint hint{};
    const bool hinted = old.has_move && std::getenv("PB200_NO_ASSEMBLY_HINT") == nullptr;
    if (hinted) {
        inc_has_extra.ensure(size_t(n) + 64);
        uint8_t* touched = inc_has_extra.as<uint8_t>();
        PB_CUDA(cudaMemsetAsync(touched, 0, size_t(n) + 1, stream));
        if (fin.side_total && nmoves) {
            PB_DISPATCH_WS(W, inc_shard_touch_kernel<W><<<small_grid, NT, 0, stream>>>(
                                  md, uint32_t(rank), P, old.words.as<uint32_t>(), n, m, m, dist,
                                  inc_side_keys[scur].as<uint32_t>(), nmoves, touched, ictr));
            check_launch();
        }
        hint.origin = inc_inv.as<uint32_t>();
        hint.touched = touched;
        hint.newidx = add;  // (converted in place once the remap below has used the counts)
        hint.row_ptr = old.row_ptr.as<uint32_t>();
        hint.col = old.col.as<int32_t>();
        hint.move = old.move.as<uint8_t>();
        hint.n_old = n;
    }
    // the coefficients move with their rows (remap_state); the discarded weight lands in Ctl::out[0].  Room for a halo
    // of the previous size behind the rows: the first Taylor order reads the vector from here
    c_new.ensure((size_t(fin.n_new) + old.halo_n + old.halo_n / 4 + 1024) * 16 + 16);
    {
        const int rg = grid_for(uint64_t(n) + fin.side_total);
        if (size_t(rg) * 8 > partials.cap) throw CudaFail("internal error: reduction scratch too small for the grid");
        inc_shard_remap_kernel<<<rg, NT, 0, stream>>>(n, m, m, dist, inc_side_gap[scur].as<uint32_t>(), add, vs, ictr, c_old,
                                                      c_new.as<double2>(), partials.as<double>(), &c->ticket, c->out);
        check_launch();
    }
    if (hinted && n) {
        inc_shard_newidx_kernel<<<grid_for(n), NT, 0, stream>>>(n, m, dist, vs, add);
        check_launch();
    }
    next.n = fin.n_new;
    next.q_nom = kept_global;
    next.order = m;
    next.has_full = true;
    ++inc_steps;
    inc_side_keys_total += fin.side_total;
    inc_expanded_total += fin.expanded_total;
    PB_CUDA(cudaEventRecord(ev[2], stream));
    assemble_sharded(next, hinted ? &hint : nullptr);
    return true;
}

// ------------------------------------------------------------------------------------------------
// row-wise assembly on shards + halo plan
// ------------------------------------------------------------------------------------------------
void Engine::assemble_sharded(Space& sp, const AsmHint* hint) {
    const int W = md.W;
    const uint32_t P = uint32_t(world);
    const uint32_t n = sp.n;
    const int width = row_width;
    Ctl* c = dctl();
    tmp_col.ensure(size_t(n) * width * 4 + 4);
    tmp_val.ensure(size_t(n) * width * 8 + 8);
    tmp_cnt.ensure(size_t(n) * 4 + 4);
    tmp_move.ensure(size_t(n) * width + 4);
    sp.row_ptr.ensure((size_t(n) + 1) * 4 + CSR_PAD);
    const uint64_t req_cap64 = uint64_t(n) * uint64_t(width) + 1;
    if (req_cap64 > 0x7ffffff0ull) throw PacesError("assembly: request count exceeds 31-bit indexing");
    const uint32_t req_cap = uint32_t(req_cap64);
    req_keys.ensure(size_t(req_cap) * W * 4);
    req_dest.ensure(size_t(req_cap) * 4);
    req_pos.ensure(size_t(req_cap) * 4);
    sendbuf.ensure(size_t(req_cap) * W * 4 + 16);
    ShardCounters* dsc = &route_block()->sc;
    PB_CUDA(cudaMemsetAsync(dsc, 0, sizeof(ShardCounters), stream));
    const uint32_t achunk = chunk_for(n);
    if (n && hint != nullptr) {
        // the table grew incrementally: rows that survived untouched take their local columns from the previous H_eff
        PB_DISPATCH_WS(W, assemble_rows_hinted_sharded_kernel<W><<<grid_for(n), NT, 0, stream>>>(
                              md, uint32_t(rank), P, sp.words.as<uint32_t>(), n, width, *hint, tmp_col.as<uint32_t>(),
                              tmp_val.as<double>(), tmp_move.as<uint8_t>(), tmp_cnt.as<uint32_t>(), req_keys.as<uint32_t>(),
                              req_dest.as<uint32_t>(), req_cap, dsc));
        check_launch();
    } else if (n) {
        PB_DISPATCH_WS(W, assemble_rows_sharded_kernel<W><<<grid_chunked(n, achunk), NT, 0, stream>>>(
                              md, uint32_t(rank), P, sp.words.as<uint32_t>(), n, achunk, width, tmp_col.as<uint32_t>(),
                              tmp_val.as<double>(), tmp_move.as<uint8_t>(), tmp_cnt.as<uint32_t>(), req_keys.as<uint32_t>(),
                              req_dest.as<uint32_t>(), req_cap, dsc));
        check_launch();
    }
    // requests -> owners (device-side count; one read-back for the counters and both count vectors)
    route_async(req_dest.as<uint32_t>(), &dsc->n_req, req_cap, req_pos.as<uint32_t>());
    PB_DISPATCH_WS(W, route_scatter_keys_kernel<W><<<grid_for(req_cap), NT, 0, stream>>>(
                          req_keys.as<uint32_t>(), req_pos.as<uint32_t>(), &dsc->n_req, req_cap, sendbuf.as<uint32_t>()));
    check_launch();
    const ShardCounters hsc = route_finish();
    if (hsc.overflow) throw CudaFail("internal error: request buffer overflow during assembly");
    const uint32_t nreq = hsc.n_req;
    const std::vector<uint64_t> req_send = h_send;  // requests I send per peer
    const std::vector<uint64_t> req_recv = h_recv;  // requests I answer per peer
    const uint64_t nr = exchange_known(sendbuf.p, recvbuf, uint64_t(W) * 4);

    // owner side: answers + the list of local rows to pack for every later SpMV
    answer.ensure(size_t(nr) * 4 + 4);
    found.ensure((size_t(nr) + 1) * 4);
    PB_DISPATCH_WS(W, answer_requests_kernel<W><<<grid_for(nr), NT, 0, stream>>>(
                          sp.words.as<uint32_t>(), n, recvbuf.as<uint32_t>(), uint32_t(nr), answer.as<uint32_t>(),
                          found.as<uint32_t>()));
    check_launch();
    exclusive_scan(found.as<uint32_t>(), nr + 1);
    // per-requester found counts = differences of the scan at the bucket boundaries: picked on the device, they come
    // back with the halo counts and nnz in ONE read-back further down (the send list is sized by its bound meanwhile)
    asm_info.ensure(sizeof(ShardAsmInfo));
    ShardAsmInfo* dinfo = asm_info.as<ShardAsmInfo>();
    auto offsets_of = [&](const std::vector<uint64_t>& per_peer) {
        PeerOffsets o{};
        uint64_t off = 0;
        for (uint32_t p = 0; p <= P; ++p) {
            o.v[p] = uint32_t(off);
            if (p < P) off += per_peer[p];
        }
        return o;
    };
    pick_boundaries_kernel<<<1, 96, 0, stream>>>(found.as<uint32_t>(), offsets_of(req_recv), P, nullptr, dinfo->found_at);
    check_launch();
    sp.send_idx.ensure(size_t(nr) * 4 + 4);
    build_send_list_kernel<<<grid_for(nr), NT, 0, stream>>>(answer.as<uint32_t>(), found.as<uint32_t>(), uint32_t(nr),
                                                            sp.send_idx.as<uint32_t>());
    check_launch();

    // replies -> requesters (same buckets, reversed roles)
    h_send = req_recv;
    h_recv = req_send;  // one reply per request: the counts are known on both sides
    const uint64_t nrep = exchange_known(answer.p, reply, 4);
    if (nrep != nreq) throw CudaFail("internal error: look-up replies do not match the requests");
    halo_flag.ensure((size_t(nreq) + 1) * 4);
    reply_flags_kernel<<<grid_for(nreq), NT, 0, stream>>>(reply.as<uint32_t>(), nreq, halo_flag.as<uint32_t>());
    check_launch();
    exclusive_scan(halo_flag.as<uint32_t>(), uint64_t(nreq) + 1);
    resolve_requests_kernel<<<grid_for(n), NT, 0, stream>>>(n, width, tmp_col.as<uint32_t>(), tmp_val.as<double>(),
                                                            tmp_move.as<uint8_t>(), tmp_cnt.as<uint32_t>(),
                                                            req_pos.as<uint32_t>(),
                                                            reply.as<uint32_t>(), halo_flag.as<uint32_t>(),
                                                            sp.row_ptr.as<uint32_t>());
    check_launch();
    PB_CUDA(cudaMemsetAsync(sp.row_ptr.as<uint32_t>() + n, 0, 4, stream));
    exclusive_scan(sp.row_ptr.as<uint32_t>(), uint64_t(n) + 1);
    pick_boundaries_kernel<<<1, 96, 0, stream>>>(halo_flag.as<uint32_t>(), offsets_of(req_send), P,
                                                 sp.row_ptr.as<uint32_t>() + n, dinfo->halo_at);
    check_launch();
    const ShardAsmInfo info = read_back<ShardAsmInfo>(dinfo);
    sp.halo_send.assign(P, 0);
    sp.halo_recv.assign(P, 0);
    for (uint32_t p = 0; p < P; ++p) {
        sp.halo_send[p] = info.found_at[p + 1] - info.found_at[p];
        sp.halo_recv[p] = info.halo_at[p + 1] - info.halo_at[p];
    }
    sp.send_total = info.found_at[P];
    sp.halo_n = info.halo_at[P];
    if (uint64_t(n) + sp.halo_n > 0x7fffffffull) throw PacesError("assembly: local rows + halo exceed int32 columns");
    const uint32_t nnz = info.halo_at[65];
    sp.col.ensure(size_t(nnz) * 4 + CSR_PAD);
    sp.val.ensure(size_t(nnz) * 8 + CSR_PAD);
    sp.move.ensure(size_t(nnz) + CSR_PAD);  // the generator's move id of every entry (the next step's assembly hint)
    // value codes for the Taylor tile kernels, produced by the compaction itself (no pass of their own)
    const bool tiles = taylor_tiles_usable(width);
    const bool want_codes = tiles && use_codes && md.vt_n > 0;
    uint32_t* fail = &c->code_fail;
    if (want_codes) {
        sp.code.ensure(size_t(nnz) * 2 + CSR_PAD);
        if (!md.vt_diag) sp.diag.ensure(size_t(n) * 8 + CSR_PAD);
        PB_CUDA(cudaMemsetAsync(fail, 0, 4, stream));
    }
    assemble_compact_sharded_kernel<<<grid_for(n), NT, 0, stream>>>(
        n, width, tmp_col.as<uint32_t>(), tmp_val.as<double>(), tmp_move.as<uint8_t>(), sp.row_ptr.as<uint32_t>(),
        sp.col.as<int32_t>(), sp.val.as<double>(), sp.move.as<uint8_t>(), md.vtab, md.vt_n, md.vt_diag,
        want_codes ? sp.code.as<uint16_t>() : nullptr, sp.diag.as<double>(), fail);
    check_launch();
    sp.nnz = nnz;
    sp.max_row = width;
    sp.has_h = true;
    sp.val_valid = true;
    // global sizes and the code-failure verdict: one device all-reduce of three doubles, one read-back
    shard_sizes_kernel<<<1, 32, 0, stream>>>(n, nnz, want_codes ? fail : nullptr, c->out + 4);
    check_launch();
    comm_check(ops.allreduce_f64_dev(ops.user, c->out + 4, 3, stream), "allreduce_f64_dev(sizes)");
    struct Sizes {
        double v[3];
    };
    const Sizes gs = read_back<Sizes>(c->out + 4);
    sp.has_code = want_codes && gs.v[2] == 0.0;
    sp.has_move = true;
    // the tile kernels tell rows without / with halo columns apart themselves; the row-list kernels need the lists
    sp.n_interior = sp.n_boundary = 0;
    sp.row_lists = false;
    if (!tiles) classify_rows(sp);
    sp.n_global = uint64_t(gs.v[0]);
    sp.nnz_global = uint64_t(gs.v[1]);
    require_memory(sp.nnz_global * 2 * 16, "matrix assembly buffer");
    (void)c;
}

// ------------------------------------------------------------------------------------------------
// truncate_select on shards: global k-th largest weight, ties drawn identically on every rank
// ------------------------------------------------------------------------------------------------
uint32_t Engine::select_sharded(const uint32_t* d_words, const double2* d_c, uint32_t n, uint64_t q_nom, uint64_t seed,
                                double* norm2_out, bool compact) {
    require_model();
    if (q_nom < 1) throw PacesError("truncate_select: q_nom must be >= 1");
    const int W = md.W;
    const uint32_t P = uint32_t(world);
    Ctl* c = dctl();
    weights.ensure(size_t(n) * 8 + 8);
    flag_keep.ensure((size_t(n) + 1) * 4);
    PB_CUDA(cudaMemsetAsync(hist.p, 0, SEL_BINS * sizeof(uint32_t), stream));
    const int g = grid_for(n);
    SelectCtl init{};
    init.k = q_nom;
    std::memcpy(pinned, &init, sizeof(init));
    PB_CUDA(cudaMemcpyAsync(&c->select, pinned, sizeof(SelectCtl), cudaMemcpyHostToDevice, stream));
    // Two histogram passes (the first fused with the weights), each all-reduced; the group that still shares the
    // cutoff's first 22 bits is almost always a handful of values, so every rank stages its members, ONE more all-reduce
    // gathers them (disjoint zero-initialised slots) and one CTA per rank finishes the remaining 42 bits on identical
    // data.  The sum of the weights and the support count ride on the device collectives: ONE read-back.
    double* gsum = c->tsum;  // (free between the Taylor phases)
    sel_list.ensure(size_t(SEL_LIST_CAP) * 8);
    sel_stage.ensure(size_t(P) * SHARD_STAGE_WORDS * 4);
    PB_CUDA(cudaMemsetAsync(sel_stage.p, 0, size_t(P) * SHARD_STAGE_WORDS * 4, stream));
    weights_hist_kernel<<<g, NT, 0, stream>>>(d_c, n, weights.as<double>(), partials.as<double>(), &c->select,
                                              hist.as<uint32_t>(), gsum);
    check_launch();
    comm_check(ops.allreduce_u32_dev(ops.user, hist.as<uint32_t>(), SEL_BINS, stream), "allreduce_u32_dev");
    comm_check(ops.allreduce_f64_dev(ops.user, gsum, 2, stream), "allreduce_f64_dev");
    select_pick_global_kernel<<<1, NT, 0, stream>>>(hist.as<uint32_t>(), 11, &c->select, gsum);
    check_launch();
    const int sg = std::min(g, sm_count * 2);
    select_pass_kernel<<<sg, NT, 0, stream>>>(weights.as<double>(), n, 42, 11, &c->select, hist.as<uint32_t>(), 0);
    check_launch();
    comm_check(ops.allreduce_u32_dev(ops.user, hist.as<uint32_t>(), SEL_BINS, stream), "allreduce_u32_dev");
    select_pick_global_kernel<<<1, NT, 0, stream>>>(hist.as<uint32_t>(), 11, &c->select);
    check_launch();
    select_gather_kernel<<<g, NT, 0, stream>>>(weights.as<double>(), n, 42, &c->select,
                                               sel_list.as<unsigned long long>(), SHARD_LIST_CAP);
    check_launch();
    select_stage_kernel<<<4, NT, 0, stream>>>(sel_list.as<unsigned long long>(), &c->select, uint32_t(rank),
                                              sel_stage.as<uint32_t>());
    check_launch();
    comm_check(ops.allreduce_u32_dev(ops.user, sel_stage.as<uint32_t>(), uint64_t(P) * SHARD_STAGE_WORDS, stream),
               "allreduce_u32_dev(select members)");
    select_union_kernel<<<1, NT, 0, stream>>>(sel_stage.as<uint32_t>(), P, sel_list.as<unsigned long long>(), &c->select);
    check_launch();
    // (PB200_SHARD_NO_TAIL=1: tests force the full-pass fallback that massive exact ties would take)
    static const bool no_tail = std::getenv("PB200_SHARD_NO_TAIL") != nullptr;
    if (!no_tail) {
        select_tail_kernel<<<1, NT, 0, stream>>>(sel_list.as<unsigned long long>(), &c->select, SHARD_LIST_CAP);
        check_launch();
    }
    SelectCtl sc = read_back<SelectCtl>(&c->select);  // identical on every rank (all-reduced inputs)
    const double norm2 = sc.norm2;
    const uint64_t support = sc.support;
    if (norm2_out) *norm2_out = norm2;
    if (support == 0) throw PacesError("truncate_select: state has no support");
    last_kept_global = std::min<uint64_t>(support, q_nom);

    uint32_t* keep = flag_keep.as<uint32_t>();
    if (support <= q_nom) {
        select_flags_kernel<<<g, NT, 0, stream>>>(weights.as<double>(), n, 0, &c->select, 1, keep, nullptr, nullptr);
        check_launch();
    } else {
        if (!sc.tail_done) {
            // the group sharing the first 22 bits is larger than the staged lists (massive exact ties): full passes
            static const int shifts[4] = {31, 20, 9, 0};
            static const int widths[4] = {11, 11, 11, 9};
            for (int p = 0; p < 4; ++p) {
                select_pass_kernel<<<sg, NT, 0, stream>>>(weights.as<double>(), n, shifts[p], widths[p], &c->select,
                                                          hist.as<uint32_t>(), 0);
                check_launch();
                comm_check(ops.allreduce_u32_dev(ops.user, hist.as<uint32_t>(), SEL_BINS, stream), "allreduce_u32_dev");
                select_pick_global_kernel<<<1, NT, 0, stream>>>(hist.as<uint32_t>(), widths[p], &c->select);
                check_launch();
            }
            sc = read_back<SelectCtl>(&c->select);
        }
        const uint64_t need = q_nom - sc.count_gt;
        if (need >= sc.count_eq) {
            select_flags_kernel<<<g, NT, 0, stream>>>(weights.as<double>(), n, 1, &c->select, 1, keep, nullptr, nullptr);
            check_launch();
        } else {
            // gather the tie KEYS of all ranks, order them canonically, draw exactly as engine.hpp:137-142
            if (pending_words) {
                PB_CUDA(cudaStreamWaitEvent(stream, ev_words, 0));
                pending_words = false;
                if (!rows_sorted_on_device(d_words, n)) throw PacesError("truncate_select: state table must be sorted");
            }
            flag_tie.ensure((size_t(n) + 1) * 4);
            pos_a.ensure((size_t(n) + 1) * 4);
            select_flags_kernel<<<g, NT, 0, stream>>>(weights.as<double>(), n, 1, &c->select, 0, keep,
                                                      flag_tie.as<uint32_t>(), nullptr);
            check_launch();
            PB_CUDA(cudaMemcpyAsync(pos_a.p, flag_tie.p, (size_t(n) + 1) * 4, cudaMemcpyDeviceToDevice, stream));
            exclusive_scan(pos_a.as<uint32_t>(), uint64_t(n) + 1);
            const uint32_t nt_local = read_back<uint32_t>(pos_a.as<uint32_t>() + n);
            sel_keys.ensure(size_t(std::max<uint64_t>(nt_local, sc.count_eq)) * W * 4 + 16);
            PB_DISPATCH_WS(W, compact_rows_kernel<W><<<g, NT, 0, stream>>>(d_words, flag_tie.as<uint32_t>(),
                                                                          pos_a.as<uint32_t>(), n,
                                                                          sel_keys.as<uint32_t>()));
            check_launch();
            std::vector<uint32_t> mine(size_t(nt_local) * W);
            if (nt_local)
                PB_CUDA(cudaMemcpyAsync(mine.data(), sel_keys.p, mine.size() * 4, cudaMemcpyDeviceToHost, stream));
            sync();
            // fixed-size all-gather: counts first, then keys padded to the largest contribution
            std::vector<uint64_t> cnts(P, 0);
            uint64_t my = nt_local;
            comm_check(ops.allgather_host(ops.user, &my, 8, cnts.data()), "allgather_host");
            uint64_t mx = 0;
            for (uint64_t v : cnts) mx = std::max(mx, v);
            std::vector<uint32_t> padded(size_t(mx) * W, 0), all(size_t(mx) * W * P, 0);
            std::copy(mine.begin(), mine.end(), padded.begin());
            if (mx) comm_check(ops.allgather_host(ops.user, padded.data(), mx * W * 4, all.data()), "allgather_host");
            std::vector<std::vector<uint32_t>> ties;
            for (uint32_t p = 0; p < P; ++p)
                for (uint64_t j = 0; j < cnts[p]; ++j) {
                    const uint32_t* k = all.data() + (size_t(p) * mx + j) * W;
                    ties.emplace_back(k, k + W);
                }
            std::sort(ties.begin(), ties.end());  // vector<uint32_t> compares word-lexicographically = canonical order
            std::mt19937_64 rng(seed);
            for (size_t i = ties.size(); i > 1 && need < ties.size(); --i) {
                const size_t j = size_t(rng() % i);
                std::swap(ties[i - 1], ties[j]);
            }
            std::vector<uint32_t> chosen;
            for (uint64_t i = 0; i < need; ++i) chosen.insert(chosen.end(), ties[i].begin(), ties[i].end());
            sel_keys.ensure(chosen.size() * 4 + 16);
            PB_CUDA(cudaMemcpyAsync(sel_keys.p, chosen.data(), chosen.size() * 4, cudaMemcpyHostToDevice, stream));
            PB_DISPATCH_WS(W, mark_selected_kernel<W><<<grid_for(need), NT, 0, stream>>>(
                                  md, uint32_t(rank), P, d_words, n, sel_keys.as<uint32_t>(), uint32_t(need), keep));
            check_launch();
            sync();
        }
    }
    // the kept keys themselves are only needed by the full expansion; the incremental growth works on the flags
    if (!compact) {
        n_seeds = 0;
        return 0;
    }
    return compact_kept_counted(d_words, n);
}

/// The rows flagged in flag_keep -> this->seeds (order preserving); returns their number (one read-back).
uint32_t Engine::compact_kept_counted(const uint32_t* d_words, uint32_t n) {
    const int W = md.W;
    const int g = grid_for(n);
    uint32_t* keep = flag_keep.as<uint32_t>();
    pos_a.ensure((size_t(n) + 2) * 4);
    PB_CUDA(cudaMemcpyAsync(pos_a.p, keep, (size_t(n) + 1) * 4, cudaMemcpyDeviceToDevice, stream));
    exclusive_scan(pos_a.as<uint32_t>(), uint64_t(n) + 1);
    if (pending_words) {
        PB_CUDA(cudaStreamWaitEvent(stream, ev_words, 0));
        pending_words = false;
        if (!rows_sorted_on_device(d_words, n)) throw PacesError("truncate_select: state table must be sorted");
    }
    const uint32_t kept = read_back<uint32_t>(pos_a.as<uint32_t>() + n);
    seeds.ensure(size_t(kept) * W * 4 + 4);
    PB_DISPATCH_WS(W, compact_rows_kernel<W><<<g, NT, 0, stream>>>(d_words, keep, pos_a.as<uint32_t>(), n,
                                                                  seeds.as<uint32_t>()));
    check_launch();
    n_seeds = kept;
    return kept;
}

// ------------------------------------------------------------------------------------------------
// expmv on shards.  Per order: pack + halo exchange (own channel / stream when the transport has one), the rows
// without halo columns meanwhile, then the rows with halo columns, ONE all-reduce of the partial norms, the stop rule
// on every rank.  Orders are paired as on one GPU (taylor.cu): an order whose predecessor missed the stop rule leaves
// c alone and its |term|^2 rides on the next order's all-reduce.  Nothing here returns to the host between orders.
// ------------------------------------------------------------------------------------------------
void Engine::expmv_sharded(const Space& sp, double2* c_vec, double dt, double rtol, int max_order, int substeps,
                           int* order_used, double* last_term_norm, double* last_c_norm, bool fuse_first, double* exp_out,
                           double* norm2_out, double* discarded_out) {
    if (!(dt > 0)) throw PacesError("propagator: dt must be > 0");
    if (!(rtol > 0) || !(rtol < 1)) throw PacesError("propagator: rtol must be in (0, 1)");
    if (max_order < 1) throw PacesError("propagator: max_order must be >= 1");
    if (substeps < 1) throw PacesError("propagator: substeps must be >= 1");
    const uint32_t n = sp.n;
    Ctl* c = dctl();
    const size_t ext = (size_t(n) + sp.halo_n) * 16 + 16;
    term[0].ensure(ext);
    term[1].ensure(ext);
    const double dt_sub = dt / substeps;
    // tile kernels (the single-GPU path's, with a row filter) when the rows are short enough; row lists otherwise
    const bool tiles = shard_tiles(sp);
    if (fuse_first && !tiles) throw CudaFail("internal error: fused first order needs the tile kernels");
    const bool any_halo = sp.halo_n != 0;
    TaylorCodes codes_tmp{};
    const TaylorCodes* codes = codes_of(sp, codes_tmp);
    if (!tiles && !sp.row_lists) throw CudaFail("internal error: sharded space without row lists");
    const int gi = grid_for(sp.n_interior), gb = grid_for(sp.n_boundary);
    const uint32_t* rp = sp.row_ptr.as<uint32_t>();
    const int32_t* cl = sp.col.as<int32_t>();
    const double* vl = sp.val.as<double>();
    double* pt = partials.as<double>();
    TaylorCtl tc{};
    double exp_sums[4] = {0, 0, 0, -1};
    PB_CUDA(cudaMemsetAsync(&c->taylor, 0, sizeof(TaylorCtl), stream));
    PB_CUDA(cudaMemsetAsync(c->tsum, 0, sizeof(c->tsum), stream));  // a part that never launches deposits nothing
    // the remap's discarded weight (Ctl::out[0], this rank's part) rides on the fused first order's all-reduce
    const bool ride = fuse_first && discarded_out != nullptr;
    if (ride) PB_CUDA(cudaMemcpyAsync(c->tsum + 14, c->out, sizeof(double), cudaMemcpyDeviceToDevice, stream));
    for (int s = 0; s < substeps; ++s) {
        // (fused first order: the caller left the state in term[0]; the launch writes c_vec, it does not read it)
        if (!(fuse_first && s == 0))
            PB_CUDA(cudaMemcpyAsync(term[0].p, c_vec, size_t(n) * 16, cudaMemcpyDeviceToDevice, stream));
        if (s > 0) {
            tc.done = 0;
            tc.streak = 0;
            tc.ticket = 0;
            std::memcpy(pinned, &tc, sizeof(tc));
            PB_CUDA(cudaMemcpyAsync(&c->taylor, pinned, sizeof(TaylorCtl), cudaMemcpyHostToDevice, stream));
        }
        int order = 1;
        bool converged = false;
        bool singles = !taylor_defer;
        const int k0 = (last_order > 2 && (last_order & 1) == 0) ? 3 : 2;
        int batch = last_order > 2 ? last_order : 8;
        while (order <= max_order) {
            const int end = std::min(max_order, order + batch - 1);
            for (; order <= end; ++order) {
                const double b = -dt_sub / double(order);
                double2* tin = term[(order - 1) & 1].as<double2>();
                double2* tout = term[order & 1].as<double2>();
                int mode = TAYLOR_ROWS_SINGLE;
                const bool first = fuse_first && s == 0 && order == 1;
                if (first)
                    mode = TAYLOR_ROWS_FIRST;
                else if (!singles && order >= k0 && ((order - k0) & 1))
                    mode = TAYLOR_ROWS_CATCHUP;
                else if (!singles && order >= k0 && order < max_order)
                    mode = TAYLOR_ROWS_DEFER;
                halo_start(sp, tin);
                if (tiles) {
                    // part 1 (rows without halo columns) beside the exchange, part 2 once the halo has landed; a rank
                    // without halo columns runs all its rows in one launch
                    taylor_launch_tile_shard(mode, any_halo ? 1 : 0, sm_count, stream, n, rp, cl, vl, codes, tin, tout, c_vec,
                                             b, order, sp.max_row, pt, &c->taylor, c->tsum, c->tsum + 8, first ? 1 : 0);
                    check_launch();
                    halo_wait();
                    if (any_halo) {
                        taylor_launch_tile_shard(mode, 2, sm_count, stream, n, rp, cl, vl, codes, tin, tout, c_vec, b, order,
                                                 sp.max_row, pt, &c->taylor, c->tsum + 4, c->tsum + 11, first ? 1 : 0);
                        check_launch();
                    }
                } else {
                    taylor_launch_rows(mode, gi, stream, sp.n_interior, sp.rows_int.as<uint32_t>(), rp, cl, vl, tin, tout,
                                       c_vec, b, order, pt, &c->taylor, c->tsum);
                    check_launch();
                    halo_wait();
                    taylor_launch_rows(mode, gb, stream, sp.n_boundary, sp.rows_bnd.as<uint32_t>(), rp, cl, vl, tin, tout,
                                       c_vec, b, order, pt, &c->taylor, c->tsum + 4);
                    check_launch();
                }
                if (mode == TAYLOR_ROWS_DEFER) continue;  // its |term|^2 rides on the next order's all-reduce
                // (the first order's <x|H|x>, |x|^2 and non-finite count ride on its all-reduce)
                comm_check(ops.allreduce_f64_dev(ops.user, c->tsum, first ? (ride ? 15 : 14) : 8, stream), "allreduce_f64_dev");
                if (mode == TAYLOR_ROWS_CATCHUP)
                    taylor_stop_pair_kernel<<<1, 32, 0, stream>>>(&c->taylor, c->tsum, order, rtol);
                else
                    taylor_stop_kernel<<<1, 32, 0, stream>>>(&c->taylor, c->tsum, order, rtol);
                check_launch();
            }
            last_ctl = read_back<Ctl>(c);  // the stop flag and, after the first batch, the fused first order's sums
            if (fuse_first && s == 0 && exp_sums[3] < 0) {
                exp_sums[0] = last_ctl.tsum[8] + last_ctl.tsum[11];
                exp_sums[1] = last_ctl.tsum[9] + last_ctl.tsum[12];
                exp_sums[2] = last_ctl.tsum[10] + last_ctl.tsum[13];
                exp_sums[3] = 0;
                if (ride) *discarded_out = last_ctl.tsum[14];
                // the reference checks its input before it iterates (propagator.hpp:55-57)
                if (exp_sums[2] != 0.0) throw PacesError("expmv: non-finite input coefficient");
            }
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
    if (exp_out) *exp_out = exp_sums[0];
    if (norm2_out) *norm2_out = exp_sums[1];
}

}  // namespace pb
