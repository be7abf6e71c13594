// incremental.cuh -- kernels of the incremental adapt phase (single GPU, resident trajectory).
//
// T_new = { k : dist(k, S) <= m } (grow_subspace, subspace.hpp:195-249), where S -- the kept keys -- is a subset of
// the PREVIOUS table, whose H_eff already lists every edge among its keys (assemble_effective_hamiltonian keeps all
// in-table elements, subspace.hpp:225-241).  So the ball is grown in OLD INDEX SPACE with a distance array instead
// of key searches:
//   * a row whose neighbourhood was complete in the previous space (`full`: it was expanded there) spreads its
//     distance along its CSR row;
//   * the other rows within distance m-1 (previous final-frontier rows that a seed has moved next to) and the few
//     keys they bring in from outside the old table ("side" keys) are expanded the classic way: generate neighbour
//     keys, search the old table / the side list, collect what is absent.
// The new table is the old one compacted + the side keys merged in; CSR_new is CSR_old filtered by distance and
// renumbered through a prefix sum, plus the rows of the side keys and their symmetric entries; the coefficient
// remap (remap_state, subspace.hpp:281-305) is a gather through the same index map.  Every value is either copied
// from CSR_old or produced by the same neighbour generator as the full assembly, so the result is bit-identical to
// the full path (and to the reference).
#pragma once
#include "kernels.cuh"

namespace pb {

constexpr uint8_t DIST_INF = 255;
constexpr int INC_MAX_ORDER = 250;  // distances are bytes: m + 1 must stay below DIST_INF
constexpr uint32_t IDX_NONE = 0xffffffffu;

struct IncCounters {
    uint32_t n_expand;        // old rows at the current distance whose neighbourhood must be generated
    uint32_t overflow;        // a side / candidate buffer was too small: the step falls back to the full path
    uint32_t expanded_total;  // sum of n_expand over the levels of this step (statistics)
    uint32_t n_keep;          // old rows that survive (copied from the prefix sum for the final read-back)
};

/// dist[i] = 0 for kept rows, INF otherwise.
static __global__ void __launch_bounds__(NT) inc_init_dist_kernel(const uint32_t* __restrict__ keep, uint32_t n,
                                                           uint8_t* __restrict__ dist) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) dist[i] = keep[i] ? 0 : DIST_INF;
}

/// One BFS level in old index space: rows at distance k either spread k+1 along their CSR row (complete
/// neighbourhood) or are queued for key-based expansion.  Concurrent byte stores of the same value are benign.
static __global__ void __launch_bounds__(NT) inc_mark_level_kernel(uint32_t n, int k, const uint8_t* __restrict__ full,
                                                            const uint32_t* __restrict__ row_ptr,
                                                            const int32_t* __restrict__ col, uint8_t* dist,
                                                            uint32_t* __restrict__ elist, IncCounters* ctr) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        if (dist[i] != uint8_t(k)) continue;
        if (full[i]) {
            const uint32_t kb = __ldg(row_ptr + i), ke = __ldg(row_ptr + i + 1);
            for (uint32_t e = kb; e < ke; ++e) {
                const uint32_t j = uint32_t(__ldg(col + e));
                if (dist[j] > uint8_t(k + 1)) dist[j] = uint8_t(k + 1);
            }
        } else {
            elist[append_slot(&ctr->n_expand)] = i;
            atomicAdd(&ctr->expanded_total, 1u);
        }
    }
}

/// Binary search of a key in the (small, sorted) side list.
template <int W>
__device__ __forceinline__ bool side_find(const uint32_t* __restrict__ side_keys, uint32_t side_n, const Key<W>& k,
                                          uint32_t& pos) {
    return find_row_in<W>(side_keys, 0, side_n, k, pos);
}

/// Key-based expansion of one BFS level: sources are the queued old rows (elist) followed by the side keys at
/// distance k.  A neighbour found in the old table gets distance k+1; one found in the side list is already known;
/// anything else becomes a candidate with its insertion gap in the OLD table (gap_count feeds the dedup machinery).
template <int W>
static __global__ void __launch_bounds__(NT) inc_expand_kernel(ModelDev m, const uint32_t* __restrict__ table, uint32_t n,
                                                        const uint32_t* __restrict__ elist,
                                                        const uint32_t* __restrict__ n_elist_ptr,
                                                        const uint32_t* __restrict__ side_keys,
                                                        const uint8_t* __restrict__ side_dist, uint32_t side_n, int k,
                                                        uint8_t* dist, uint32_t* __restrict__ cand_keys,
                                                        uint32_t* __restrict__ cand_gap, uint32_t cand_cap,
                                                        uint32_t* __restrict__ gap_count, GrowCounters* gctr,
                                                        IncCounters* ictr) {
    const uint32_t n_elist = *n_elist_ptr;  // stays on the device: no host round trip between mark and expand
    const uint32_t total = n_elist + side_n;
    for (uint32_t t = blockIdx.x * NT + threadIdx.x; t < total; t += gridDim.x * NT) {
        Key<W> key;
        if (t < n_elist) {
            key = load_key<W>(table + size_t(__ldg(elist + t)) * W);
        } else {
            const uint32_t j = t - n_elist;
            if (side_dist[j] != uint8_t(k)) continue;
            key = load_key<W>(side_keys + size_t(j) * W);
        }
        for_each_neighbor<W>(m, key, false, [&](int, const Key<W>& kk, double, bool) {
            uint32_t pos, spos;
            if (find_row<W>(table, n, kk, pos)) {
                if (dist[pos] > uint8_t(k + 1)) dist[pos] = uint8_t(k + 1);
            } else if (!side_find<W>(side_keys, side_n, kk, spos)) {
                const uint32_t slot = append_slot(&gctr->n_cand);
                if (slot < cand_cap) {
                    store_key<W>(cand_keys + size_t(slot) * W, kk);
                    cand_gap[slot] = pos;
                    atomicAdd(gap_count + pos, 1u);
                } else {
                    ictr->overflow = 1;
                }
            }
        });
    }
}

/// After an overflowing expansion the candidate counter exceeds the buffer: clamp it so the dedup kernels stay in
/// bounds (the step is discarded anyway -- IncCounters::overflow is set).
static __global__ void inc_clamp_kernel(uint32_t* n_cand, uint32_t cap) {
    if (*n_cand > cap) *n_cand = cap;
}

/// Unique candidates of one level in canonical order: survivor of gap g with rank r -> index kept_before[g] + r.
template <int W>
static __global__ void __launch_bounds__(NT) inc_emit_unique_kernel(const uint32_t* __restrict__ cand_keys,
                                                             const uint32_t* __restrict__ cand_gap,
                                                             const uint32_t* __restrict__ perm,
                                                             const uint32_t* __restrict__ seg_rank,
                                                             const uint32_t* __restrict__ nc_ptr,
                                                             const uint32_t* __restrict__ kept_before,
                                                             uint32_t* __restrict__ out_keys,
                                                             uint32_t* __restrict__ out_gap) {
    const uint32_t nc = *nc_ptr;
    for (uint32_t s = blockIdx.x * NT + threadIdx.x; s < nc; s += gridDim.x * NT) {
        const uint32_t r = seg_rank[s];
        if (r == SEG_DUP) continue;
        const uint32_t c = perm[s];
        const uint32_t g = cand_gap[c];
        const uint32_t ord = kept_before[g] + r;
        store_key<W>(out_keys + size_t(ord) * W, load_key<W>(cand_keys + size_t(c) * W));
        out_gap[ord] = g;
    }
}

/// Merge of two sorted, disjoint key lists A (side so far) and B (this level's new keys, distance `kb`):
/// out index of A[j] = j + #B < A[j], of B[t] = t + #A < B[t].
template <int W>
static __global__ void __launch_bounds__(NT) inc_side_merge_kernel(const uint32_t* __restrict__ a_keys,
                                                            const uint32_t* __restrict__ a_gap,
                                                            const uint8_t* __restrict__ a_dist, uint32_t na,
                                                            const uint32_t* __restrict__ b_keys,
                                                            const uint32_t* __restrict__ b_gap, uint32_t nb, int kb,
                                                            uint32_t* __restrict__ o_keys, uint32_t* __restrict__ o_gap,
                                                            uint8_t* __restrict__ o_dist) {
    for (uint32_t t = blockIdx.x * NT + threadIdx.x; t < na + nb; t += gridDim.x * NT) {
        uint32_t pos;
        if (t < na) {
            const Key<W> k = load_key<W>(a_keys + size_t(t) * W);
            find_row_in<W>(b_keys, 0, nb, k, pos);
            const uint32_t o = t + pos;
            store_key<W>(o_keys + size_t(o) * W, k);
            o_gap[o] = a_gap[t];
            o_dist[o] = a_dist[t];
        } else {
            const uint32_t j = t - na;
            const Key<W> k = load_key<W>(b_keys + size_t(j) * W);
            find_row_in<W>(a_keys, 0, na, k, pos);
            const uint32_t o = j + pos;
            store_key<W>(o_keys + size_t(o) * W, k);
            o_gap[o] = b_gap[j];
            o_dist[o] = uint8_t(kb);
        }
    }
}

/// keepflag[i] = dist[i] <= m (n+1 entries, trailing 0, scanned in place afterwards).
static __global__ void __launch_bounds__(NT) inc_keepflag_kernel(const uint8_t* __restrict__ dist, uint32_t n, int m,
                                                          uint32_t* __restrict__ keepflag) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i <= n; i += gridDim.x * NT)
        keepflag[i] = (i < n && dist[i] <= uint8_t(m)) ? 1u : 0u;
}

/// cntgap[gap]++ for every side key (array zeroed before; scanned afterwards).
static __global__ void __launch_bounds__(NT) inc_count_gaps_kernel(const uint32_t* __restrict__ side_gap, uint32_t side_n,
                                                            uint32_t* __restrict__ cntgap) {
    for (uint32_t j = blockIdx.x * NT + threadIdx.x; j < side_n; j += gridDim.x * NT) atomicAdd(cntgap + side_gap[j], 1u);
}

/// New index of every old row (IDX_NONE when dropped), `full` flags of the new space, and the coefficient remap
/// fused in: kept rows carry their coefficient, dropped rows add |c|^2 to the discarded weight.
/// pk = exclusive scan of keepflag, nb = exclusive scan of cntgap (side keys with gap <= i precede row i).
static __global__ void __launch_bounds__(NT) inc_scatter_old_kernel(const double2* __restrict__ c_old, uint32_t n, int m,
                                                             const uint8_t* __restrict__ dist,
                                                             const uint32_t* __restrict__ pk,
                                                             const uint32_t* __restrict__ nb,
                                                             uint32_t* __restrict__ newidx,
                                                             uint8_t* __restrict__ out_full,
                                                             double2* __restrict__ c_new, double* __restrict__ partials,
                                                             unsigned* ticket, double* __restrict__ out) {
    __shared__ double smem[NT / 32];
    double acc[1] = {0.0};
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        const double2 x = c_old[i];
        if (dist[i] <= uint8_t(m)) {
            const uint32_t o = pk[i] + nb[i + 1];
            newidx[i] = o;
            out_full[o] = dist[i] < uint8_t(m) ? 1 : 0;
            c_new[o] = x;
        } else {
            newidx[i] = IDX_NONE;
            acc[0] = __dadd_rn(acc[0], __dadd_rn(__dmul_rn(x.x, x.x), __dmul_rn(x.y, x.y)));
        }
    }
    double tot[1];
    if (grid_sum<1>(acc, partials, ticket, tot, smem) && threadIdx.x == 0) out[0] = tot[0];
}

/// The surviving old rows into the new table, one thread per WORD: surviving rows come in long runs, so both the
/// reads and the writes are coalesced whatever the key width (a thread per row moves 4W bytes at a 4W-byte stride).
template <int W>
static __global__ void __launch_bounds__(NT) inc_copy_rows_kernel(const uint32_t* __restrict__ table, uint32_t n,
                                                           const uint32_t* __restrict__ newidx,
                                                           uint32_t* __restrict__ out_table) {
    const uint64_t total = uint64_t(n) * W;
    for (uint64_t w = uint64_t(blockIdx.x) * NT + threadIdx.x; w < total; w += uint64_t(gridDim.x) * NT) {
        const uint32_t i = uint32_t(w / W);
        const uint32_t o = __ldg(newidx + i);
        if (o != IDX_NONE) out_table[uint64_t(o) * W + (w - uint64_t(i) * W)] = __ldg(table + w);
    }
}

/// Side keys into the new table (c_new was zeroed: they start with zero amplitude).
template <int W>
static __global__ void __launch_bounds__(NT) inc_scatter_side_kernel(const uint32_t* __restrict__ side_keys,
                                                              const uint32_t* __restrict__ side_gap,
                                                              const uint8_t* __restrict__ side_dist, uint32_t side_n,
                                                              int m, const uint32_t* __restrict__ pk,
                                                              uint32_t* __restrict__ side_newidx,
                                                              uint32_t* __restrict__ out_table,
                                                              uint8_t* __restrict__ out_full) {
    for (uint32_t j = blockIdx.x * NT + threadIdx.x; j < side_n; j += gridDim.x * NT) {
        const uint32_t o = pk[side_gap[j]] + j;
        side_newidx[j] = o;
        store_key<W>(out_table + size_t(o) * W, load_key<W>(side_keys + size_t(j) * W));
        out_full[o] = side_dist[j] < uint8_t(m) ? 1 : 0;
    }
}

/// Rows of the side keys: neighbours in canonical order, looked up in the old table (kept rows only) and in the
/// side list.  An old-row neighbour also receives the symmetric entry (extras slots of that row: x_col/x_val with
/// stride `width`, counted in x_cnt).
template <int W>
static __global__ void __launch_bounds__(NT) inc_side_rows_kernel(ModelDev m, const uint32_t* __restrict__ table, uint32_t n,
                                                           const uint32_t* __restrict__ newidx,
                                                           const uint32_t* __restrict__ side_keys,
                                                           const uint32_t* __restrict__ side_newidx, uint32_t side_n,
                                                           int width, uint32_t* __restrict__ s_col,
                                                           double* __restrict__ s_val, uint32_t* __restrict__ s_len,
                                                           uint32_t* __restrict__ x_col, double* __restrict__ x_val,
                                                           uint32_t* __restrict__ x_cnt) {
    for (uint32_t j = blockIdx.x * NT + threadIdx.x; j < side_n; j += gridDim.x * NT) {
        const Key<W> key = load_key<W>(side_keys + size_t(j) * W);
        const uint32_t me = side_newidx[j];
        uint32_t len = 0;
        for_each_neighbor<W>(m, key, true, [&](int, const Key<W>& kk, double amp, bool is_diag) {
            uint32_t pos, c = IDX_NONE;
            if (is_diag) {
                c = me;
            } else if (find_row<W>(table, n, kk, pos)) {
                c = newidx[pos];  // IDX_NONE when that old row was dropped
                if (c != IDX_NONE) {
                    const uint32_t t = atomicAdd(x_cnt + pos, 1u);
                    x_col[size_t(pos) * width + t] = me;
                    x_val[size_t(pos) * width + t] = amp;
                }
            } else if (side_find<W>(side_keys, side_n, kk, pos)) {
                c = side_newidx[pos];
            }
            if (c != IDX_NONE) {
                s_col[size_t(j) * width + len] = c;
                s_val[size_t(j) * width + len] = amp;
                ++len;
            }
        });
        s_len[j] = len;
    }
}

/// Row lengths of the new CSR (written at the NEW row index; every new row is written exactly once).
static __global__ void __launch_bounds__(NT) inc_row_len_kernel(uint32_t n, const uint32_t* __restrict__ newidx,
                                                         const uint32_t* __restrict__ row_ptr,
                                                         const int32_t* __restrict__ col,
                                                         const uint32_t* __restrict__ x_cnt,
                                                         const uint32_t* __restrict__ side_newidx,
                                                         const uint32_t* __restrict__ s_len, uint32_t side_n,
                                                         uint32_t* __restrict__ len_new, uint8_t* __restrict__ simple) {
    for (uint32_t t = blockIdx.x * NT + threadIdx.x; t < n + side_n; t += gridDim.x * NT) {
        if (t < n) {
            const uint32_t o = newidx[t];
            if (o == IDX_NONE) {
                simple[t] = 0;
                continue;
            }
            const uint32_t nx = x_cnt[t];
            uint32_t len = nx;
            const uint32_t kb = __ldg(row_ptr + t), ke = __ldg(row_ptr + t + 1);
            for (uint32_t e = kb; e < ke; ++e) len += (newidx[uint32_t(__ldg(col + e))] != IDX_NONE) ? 1u : 0u;
            len_new[o] = len;
            // simple: the row keeps every entry and gains none -> its entries are a straight copy with renumbering
            simple[t] = (nx == 0 && len == ke - kb) ? 1 : 0;
        } else {
            len_new[side_newidx[t - n]] = s_len[t - n];
        }
    }
}

/// Entries of the new CSR.  Old rows: the old entries whose column survives, renumbered (a monotone map, so they
/// stay ascending), merged with the row's extras (a handful, insertion-sorted by column).  Side rows: copied.
static __global__ void __launch_bounds__(NT) inc_fill_kernel(uint32_t n, const uint32_t* __restrict__ newidx,
                                                      const uint32_t* __restrict__ row_ptr,
                                                      const int32_t* __restrict__ col, const double* __restrict__ val,
                                                      int width, const uint32_t* __restrict__ x_col,
                                                      const double* __restrict__ x_val,
                                                      const uint32_t* __restrict__ x_cnt,
                                                      const uint32_t* __restrict__ side_newidx,
                                                      const uint32_t* __restrict__ s_col,
                                                      const double* __restrict__ s_val,
                                                      const uint32_t* __restrict__ s_len, uint32_t side_n,
                                                      const uint32_t* __restrict__ row_ptr_new,
                                                      const uint8_t* __restrict__ simple,
                                                      int32_t* __restrict__ col_new, double* __restrict__ val_new) {
    for (uint32_t t = blockIdx.x * NT + threadIdx.x; t < n + side_n; t += gridDim.x * NT) {
        if (t < n && simple[t]) continue;  // copied by inc_fill_simple_kernel
        if (t >= n) {
            const uint32_t j = t - n;
            uint32_t w = row_ptr_new[side_newidx[j]];
            for (uint32_t e = 0; e < s_len[j]; ++e, ++w) {
                col_new[w] = int32_t(s_col[size_t(j) * width + e]);
                val_new[w] = s_val[size_t(j) * width + e];
            }
            continue;
        }
        const uint32_t o = newidx[t];
        if (o == IDX_NONE) continue;
        uint32_t w = row_ptr_new[o];
        const uint32_t kb = __ldg(row_ptr + t), ke = __ldg(row_ptr + t + 1);
        const uint32_t nx = x_cnt[t];
        if (nx == 0) {
            for (uint32_t e = kb; e < ke; ++e) {
                const uint32_t c = newidx[uint32_t(__ldg(col + e))];
                if (c != IDX_NONE) {
                    col_new[w] = int32_t(c);
                    val_new[w] = __ldg(val + e);
                    ++w;
                }
            }
            continue;
        }
        // extras of this row sorted by column (nx <= width <= MAX_ROW)
        uint32_t xc[MAX_ROW];
        double xv[MAX_ROW];
        for (uint32_t a = 0; a < nx; ++a) {
            const uint32_t c = x_col[size_t(t) * width + a];
            const double v = x_val[size_t(t) * width + a];
            uint32_t b = a;
            while (b > 0 && xc[b - 1] > c) {
                xc[b] = xc[b - 1];
                xv[b] = xv[b - 1];
                --b;
            }
            xc[b] = c;
            xv[b] = v;
        }
        uint32_t xi = 0;
        for (uint32_t e = kb; e < ke; ++e) {
            const uint32_t c = newidx[uint32_t(__ldg(col + e))];
            if (c == IDX_NONE) continue;
            while (xi < nx && xc[xi] < c) {
                col_new[w] = int32_t(xc[xi]);
                val_new[w] = xv[xi];
                ++w, ++xi;
            }
            col_new[w] = int32_t(c);
            val_new[w] = __ldg(val + e);
            ++w;
        }
        for (; xi < nx; ++xi, ++w) {
            col_new[w] = int32_t(xc[xi]);
            val_new[w] = xv[xi];
        }
    }
}

/// The common case of inc_fill -- rows that keep all their entries and gain none -- as a coalesced copy: a warp
/// takes 32 consecutive OLD rows, whose entries are one contiguous run of CSR_old; every lane moves entries of that
/// run (the source row of an entry is found by a 5-step search over the 32 row offsets, as in
/// assemble_compact_kernel), renumbering the column through the index map.
static __global__ void __launch_bounds__(NT) inc_fill_simple_kernel(uint32_t n, const uint32_t* __restrict__ newidx,
                                                             const uint32_t* __restrict__ row_ptr,
                                                             const int32_t* __restrict__ col,
                                                             const double* __restrict__ val,
                                                             const uint8_t* __restrict__ simple,
                                                             const uint32_t* __restrict__ row_ptr_new,
                                                             int32_t* __restrict__ col_new,
                                                             double* __restrict__ val_new) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = uint64_t(gridDim.x) * (NT / 32);
    for (uint64_t base = (uint64_t(blockIdx.x) * (NT / 32) + (threadIdx.x >> 5)) * 32; base < n; base += nwarps * 32) {
        const uint64_t i = base + lane;
        const bool in = i < n;
        const uint32_t rp = __ldg(row_ptr + (in ? i : n));
        const bool smp = in && simple[i];
        const uint32_t dst0 = smp ? row_ptr_new[newidx[i]] : 0u;  // new offset of the row's first entry
        const unsigned smask = __ballot_sync(0xffffffffu, smp);
        const uint32_t rp0 = __shfl_sync(0xffffffffu, rp, 0);
        const uint32_t end = __ldg(row_ptr + (base + 32 < n ? base + 32 : n));
        const uint32_t total = end - rp0;
        if (smask == 0) continue;
        for (uint32_t k0 = 0; k0 < total; k0 += 32) {
            const uint32_t k = k0 + lane;
            const uint32_t e = rp0 + (k < total ? k : total - 1);
            uint32_t r = 0;  // last row whose offset is <= e
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, rp, (r + step) & 31);
                if (v <= e) r += step;
            }
            const uint32_t off = e - __shfl_sync(0xffffffffu, rp, r);
            const uint32_t d0 = __shfl_sync(0xffffffffu, dst0, r);
            if (k < total && ((smask >> r) & 1u)) {
                col_new[d0 + off] = int32_t(newidx[uint32_t(__ldg(col + e))]);
                val_new[d0 + off] = __ldg(val + e);
            }
        }
    }
}

/// full[i] = 1 everywhere, then 0 for the rows listed (the final frontier of a full grow_subspace).
static __global__ void __launch_bounds__(NT) inc_clear_full_kernel(const uint32_t* __restrict__ rows, uint32_t cnt,
                                                            uint8_t* __restrict__ full) {
    for (uint32_t t = blockIdx.x * NT + threadIdx.x; t < cnt; t += gridDim.x * NT) full[rows[t]] = 0;
}

}  // namespace pb
