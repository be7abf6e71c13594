// incremental.cuh -- kernels of the incremental adapt phase (single GPU, resident trajectory).
//
// T_new = { k : dist(k, S) <= m } (grow_subspace, subspace.hpp:195-249), where S -- the kept keys -- is a subset of
// the PREVIOUS table, whose H_eff already lists every edge among its keys (assemble_effective_hamiltonian keeps all
// in-table elements, subspace.hpp:225-241).  So the ball is grown in OLD INDEX SPACE with a distance array instead
// of key searches:
//   * distances spread along the rows of the previous H_eff (it is structurally symmetric, so a row PULLS: it is at
//     distance k+1 if one of its columns is at distance k);
//   * rows within distance m-1 whose neighbourhood was not complete in the previous space (its final frontier) and
//     the few keys they bring in from outside the old table ("side" keys) are expanded the classic way: generate
//     neighbour keys, search the old table / the side list, collect what is absent.
// The new table is the old one compacted + the side keys merged in; CSR_new is CSR_old filtered by distance and
// renumbered, plus the rows of the side keys and their symmetric entries; the coefficient remap (remap_state,
// subspace.hpp:281-305) is a gather through the same index map.  Every value is either copied from CSR_old or
// produced by the same neighbour generator as the full assembly, so the result is bit-identical to the full path
// (and to the reference).
//
// Every size that is only known on the device STAYS there (IncCounters): the kernels of a step are enqueued back to
// back against capacity-sized buffers and the host reads one small block at the end.
#pragma once
#include "kernels.cuh"

namespace pb {

constexpr uint8_t DIST_INF = 255;
constexpr int INC_MAX_ORDER = 250;  // distances are bytes: m + 1 must stay below DIST_INF
constexpr uint32_t IDX_NONE = 0xffffffffu;
constexpr uint32_t INV_SIDE = 0x80000000u;  // inv[o] = INV_SIDE | j: new row o is side key j (old rows: < 2^31)
constexpr int INC_LEVELS = 256;
constexpr int INC_IPT = 8;
constexpr int INC_TILE = NT * INC_IPT;  // rows per CTA of the fused scan kernels

/// Head of the counter block: what the host reads back at the end of the phase.
struct IncHead {
    uint32_t overflow;    // a side / candidate buffer was too small: the step falls back to the full path
    uint32_t n_keep;      // old rows that survive
    uint32_t n_new;       // rows of the new table = n_keep + side_total
    uint32_t nnz_new;
    uint32_t side_total;  // side keys after the last level
    uint32_t expanded_total;  // old rows expanded by key over all levels (statistics)
    uint32_t n_x;         // surviving old rows that gain entries (neighbours among the side keys)
    uint32_t done_c;
    uint32_t code_fail;   // a matrix element outside the model's value table: the new space carries no value codes
    uint32_t pad[1];
};
struct IncCounters {
    IncHead h;
    uint32_t n_expand[INC_LEVELS];    // old rows at distance k whose neighbourhood must be generated
    uint32_t n_cand[INC_LEVELS];      // candidates of level k (with duplicates; may exceed the buffer on overflow)
    uint32_t n_uniq[INC_LEVELS];      // unique new keys of level k
    uint32_t side_n[INC_LEVELS + 1];  // side keys before level k (side_n[0] = 0)
};

/// keep[i] = 1 for rows at distance 0 (n + 1 entries, trailing 0): the full path's flags, for a fallback.
static __global__ void __launch_bounds__(NT) inc_keep_from_dist_kernel(const uint8_t* __restrict__ dist, uint32_t n,
                                                                       uint32_t* __restrict__ keep) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i <= n; i += gridDim.x * NT) keep[i] = (i < n && dist[i] == 0) ? 1u : 0u;
}

/// One BFS level in old index space.  A row at distance k whose neighbourhood is not complete is queued for key-based
/// expansion; a row farther than k+1 moves to k+1 if one of its CSR columns is at distance k.  (Concurrent writers
/// only turn values > k+1 into k+1 and readers only test for == k, so the races are benign.)
static __global__ void __launch_bounds__(NT) inc_level_kernel(uint32_t n, int k, const uint8_t* __restrict__ full,
                                                              const uint32_t* __restrict__ row_ptr,
                                                              const int32_t* __restrict__ col, uint8_t* dist,
                                                              uint32_t* __restrict__ elist, IncCounters* ctr) {
    const uint8_t dk = uint8_t(k);
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        const uint8_t d = dist[i];
        if (d == dk) {
            if (!full[i]) elist[append_slot(&ctr->n_expand[k])] = i;
            continue;
        }
        if (d <= uint8_t(k + 1)) continue;
        const uint32_t kb = __ldg(row_ptr + i), len = __ldg(row_ptr + i + 1) - kb;
        // all columns first, then all distances: two exposed latencies per row instead of two per entry
        int32_t cj[MAX_ROW];
#pragma unroll
        for (int u = 0; u < MAX_ROW; ++u)
            if (uint32_t(u) < len) cj[u] = __ldg(col + kb + u);
        bool hit = false;
#pragma unroll
        for (int u = 0; u < MAX_ROW; ++u)
            if (uint32_t(u) < len) hit |= (dist[uint32_t(cj[u])] == dk);
        for (uint32_t e = kb + MAX_ROW; e < kb + len; ++e) hit |= (dist[uint32_t(__ldg(col + e))] == dk);  // never for model-built H_eff
        if (hit) dist[i] = uint8_t(k + 1);
    }
}

/// Binary search of a key in the (small, sorted) side list.
template <int W>
__device__ __forceinline__ bool side_find(const uint32_t* __restrict__ side_keys, uint32_t side_n, const Key<W>& k,
                                          uint32_t& pos) {
    return find_row_in4<W>(side_keys, 0, side_n, k, pos);
}

/// Key-based expansion of one BFS level, one thread per (source, neighbour slot): sources are the queued old rows
/// followed by the side keys at distance k.  A neighbour found in the old table gets distance k+1; one found in the
/// side list is already known; anything else becomes a candidate with its insertion gap in the OLD table, counted in
/// the coarse bucket gap >> sh (the dedup kernels' segments).
template <int W>
static __global__ void __launch_bounds__(NT) inc_expand_kernel(ModelDev m, const uint32_t* __restrict__ table, uint32_t n,
                                                               const uint32_t* __restrict__ elist,
                                                               const uint32_t* __restrict__ side_keys,
                                                               const uint8_t* __restrict__ side_dist, int k, int nslots,
                                                               uint8_t* dist, uint32_t* __restrict__ cand_keys,
                                                               uint32_t* __restrict__ cand_gap, uint32_t cand_cap,
                                                               int sh, uint32_t* __restrict__ bucket_count,
                                                               IncCounters* ctr) {
    const uint32_t n_elist = ctr->n_expand[k], side_n = ctr->side_n[k];
    const uint64_t total = (uint64_t(n_elist) + side_n) * uint64_t(nslots);
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&ctr->h.expanded_total, n_elist);
    for (uint64_t t = uint64_t(blockIdx.x) * NT + threadIdx.x; t < total; t += uint64_t(gridDim.x) * NT) {
        const uint32_t src = uint32_t(t / uint32_t(nslots));
        const int slot = int(t - uint64_t(src) * uint32_t(nslots));
        Key<W> key;
        if (src < n_elist) {
            key = load_key<W>(table + size_t(__ldg(elist + src)) * W);
        } else {
            const uint32_t j = src - n_elist;
            if (side_dist[j] != uint8_t(k)) continue;
            key = load_key<W>(side_keys + size_t(j) * W);
        }
        int idx = 0;
        for_each_neighbor<W>(m, key, false, [&](int, const Key<W>& kk, double, bool) {
            if (idx++ != slot) return;
            uint32_t pos, spos;
            if (find_row_in4<W>(table, 0, n, kk, pos)) {
                if (dist[pos] > uint8_t(k + 1)) dist[pos] = uint8_t(k + 1);
            } else if (!side_find<W>(side_keys, side_n, kk, spos)) {
                const uint32_t c = append_slot(&ctr->n_cand[k]);
                if (c < cand_cap) {
                    store_key<W>(cand_keys + size_t(c) * W, kk);
                    cand_gap[c] = pos;
                    atomicAdd(bucket_count + (pos >> sh), 1u);
                } else {
                    ctr->h.overflow = 1;
                }
            }
        });
    }
}

/// Unique candidates of one level in canonical order: survivor of bucket b with rank r -> index kept_before[b] + r.
template <int W>
static __global__ void __launch_bounds__(NT) inc_emit_unique_kernel(const uint32_t* __restrict__ cand_keys,
                                                                    const uint32_t* __restrict__ cand_gap,
                                                                    const uint32_t* __restrict__ perm,
                                                                    const uint32_t* __restrict__ seg_rank, int k,
                                                                    uint32_t cand_cap, int sh,
                                                                    const uint32_t* __restrict__ kept_before,
                                                                    uint32_t nbuckets, uint32_t* __restrict__ out_keys,
                                                                    uint32_t* __restrict__ out_gap, IncCounters* ctr) {
    const uint32_t nc = min(ctr->n_cand[k], cand_cap);
    if (blockIdx.x == 0 && threadIdx.x == 0) ctr->n_uniq[k] = kept_before[nbuckets];
    for (uint32_t s = blockIdx.x * NT + threadIdx.x; s < nc; s += gridDim.x * NT) {
        const uint32_t r = seg_rank[s];
        if (r == SEG_DUP) continue;
        const uint32_t c = perm[s];
        const uint32_t g = cand_gap[c];
        const uint32_t ord = kept_before[g >> sh] + r;
        store_key<W>(out_keys + size_t(ord) * W, load_key<W>(cand_keys + size_t(c) * W));
        out_gap[ord] = g;
    }
}

/// Merge of two sorted, disjoint key lists A (side so far) and B (this level's new keys, distance k+1):
/// out index of A[j] = j + #B < A[j], of B[t] = t + #A < B[t].
template <int W>
static __global__ void __launch_bounds__(NT) inc_side_merge_kernel(const uint32_t* __restrict__ a_keys,
                                                                   const uint32_t* __restrict__ a_gap,
                                                                   const uint8_t* __restrict__ a_dist,
                                                                   const uint32_t* __restrict__ b_keys,
                                                                   const uint32_t* __restrict__ b_gap, int k,
                                                                   uint32_t side_cap, uint32_t* __restrict__ o_keys,
                                                                   uint32_t* __restrict__ o_gap,
                                                                   uint8_t* __restrict__ o_dist, IncCounters* ctr) {
    const uint32_t na = ctr->side_n[k], nb = ctr->n_uniq[k];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const uint64_t merged = uint64_t(na) + nb;
        if (merged > side_cap) ctr->h.overflow = 1;
        ctr->side_n[k + 1] = uint32_t(merged > side_cap ? side_cap : merged);
    }
    for (uint32_t t = blockIdx.x * NT + threadIdx.x; t < na + nb; t += gridDim.x * NT) {
        uint32_t pos;
        if (t < na) {
            const Key<W> key = load_key<W>(a_keys + size_t(t) * W);
            find_row_in<W>(b_keys, 0, nb, key, pos);
            const uint32_t o = t + pos;
            if (o >= side_cap) continue;  // overflow: the step is discarded, only stay in bounds
            store_key<W>(o_keys + size_t(o) * W, key);
            o_gap[o] = a_gap[t];
            o_dist[o] = a_dist[t];
        } else {
            const uint32_t j = t - na;
            const Key<W> key = load_key<W>(b_keys + size_t(j) * W);
            find_row_in<W>(a_keys, 0, na, key, pos);
            const uint32_t o = j + pos;
            if (o >= side_cap) continue;
            store_key<W>(o_keys + size_t(o) * W, key);
            o_gap[o] = b_gap[j];
            o_dist[o] = uint8_t(k + 1);
        }
    }
}

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* __restrict__ a, uint32_t n, uint32_t v) {
    uint32_t lo = 0, len = n;
    while (len > 0) {
        const uint32_t half = len >> 1;
        const bool lt = __ldg(a + lo + half) < v;
        lo = lt ? lo + half + 1 : lo;
        len = lt ? len - half - 1 : half;
    }
    return lo;
}

// ------------------------------------------------------------------------------------------------
// From the distances to the new space.  No kernel below waits for another CTA: everything a tile of old rows needs to
// know about the tiles before it (kept rows, matrix entries) is reduced per tile first and scanned by one small CTA,
// so a tile with a cluster of irregular rows (frontier regions) delays nobody.
// ------------------------------------------------------------------------------------------------

/// A reference stored for slot s of side key j: IDX_NONE (no such neighbour), an OLD row index, or INV_SIDE | side index.
__device__ __forceinline__ bool side_ref_valid(uint32_t ref, const uint8_t* __restrict__ dist, int m) {
    return ref != IDX_NONE && ((ref & INV_SIDE) || dist[ref] <= uint8_t(m));
}

/// Neighbours of the side keys, one thread per (side key, neighbour slot), in canonical order (diagonal included):
/// s_ref/s_val[j * width + s].  An old row that survives and gains the symmetric entry is marked touched |= 2 (it
/// regenerates its own neighbours when its row is written).
template <int W>
static __global__ void __launch_bounds__(NT) inc_side_search_kernel(ModelDev m, const uint32_t* __restrict__ table,
                                                                    uint32_t n, int order, int levels,
                                                                    const uint8_t* __restrict__ dist,
                                                                    const uint32_t* __restrict__ side_keys, int width,
                                                                    uint32_t* __restrict__ s_ref,
                                                                    double* __restrict__ s_val,
                                                                    uint16_t* __restrict__ s_code,
                                                                    uint8_t* __restrict__ touched,
                                                                    IncCounters* __restrict__ ctr) {
    const uint32_t side_n = ctr->side_n[levels];
    const uint64_t total = uint64_t(side_n) * uint32_t(width);
    for (uint64_t t = uint64_t(blockIdx.x) * NT + threadIdx.x; t < total; t += uint64_t(gridDim.x) * NT) {
        const uint32_t j = uint32_t(t / uint32_t(width));
        const int slot = int(t - uint64_t(j) * uint32_t(width));
        const Key<W> key = load_key<W>(side_keys + size_t(j) * W);
        uint32_t ref = IDX_NONE;
        double a = 0.0;
        int idx = 0;
        for_each_neighbor<W>(m, key, true, [&](int, const Key<W>& kk, double amp, bool is_diag) {
            if (idx++ != slot) return;
            uint32_t pos;
            a = amp;
            if (is_diag) {
                ref = INV_SIDE | j;
            } else if (find_row_in4<W>(table, 0, n, kk, pos)) {
                ref = pos;
                if (dist[pos] <= uint8_t(order)) touched[pos] |= 2;  // every writer of this byte stores the same value here
            } else if (side_find<W>(side_keys, side_n, kk, pos)) {
                ref = INV_SIDE | pos;
            }
        });
        s_ref[t] = ref;
        s_val[t] = a;
        if (s_code != nullptr && ref != IDX_NONE) {  // value code of the entry (taylor.cuh, TaylorCodes)
            uint32_t cd = 0xffffu;                    // diagonal element kept per row
            if (ref != (INV_SIDE | j) || m.vt_diag) {
                cd = vt_find(m.vtab, m.vt_n, a);
                if (cd == 0xfffeu) ctr->h.code_fail = 1u;
            }
            s_code[t] = uint16_t(cd);
        }
    }
}

/// Per tile of INC_TILE old rows (the scan covers n + 1 slots: slot n is a virtual dropped row that owns the side keys
/// beyond the last old row): kept rows, first side key of the tile; a dropped row marks the rows of its CSR columns as
/// touched |= 1 (they lose an entry; H_eff is structurally symmetric); a surviving row that gains entries (touched & 2)
/// is queued in xlist (its slot in x_slot) for inc_extras_kernel.
static __global__ void __launch_bounds__(NT) inc_tile_prep_kernel(uint32_t n, int m, int levels,
                                                                  const uint8_t* __restrict__ dist,
                                                                  const uint32_t* __restrict__ row_ptr,
                                                                  const int32_t* __restrict__ col,
                                                                  const uint32_t* __restrict__ side_gap,
                                                                  uint32_t* __restrict__ tile_keep,
                                                                  uint32_t* __restrict__ tile_jlo, uint32_t ntiles,
                                                                  uint8_t* __restrict__ touched,
                                                                  uint32_t* __restrict__ xlist,
                                                                  uint32_t* __restrict__ x_slot, uint32_t x_cap,
                                                                  IncCounters* ctr) {
    __shared__ uint32_t scan_s[NT / 32];
    const uint32_t tile = blockIdx.x;
    const uint64_t t0 = uint64_t(tile) * INC_TILE;
    if (threadIdx.x == 0) {
        const uint32_t side_n = ctr->side_n[levels];
        tile_jlo[tile] = lower_bound_u32(side_gap, side_n, uint32_t(t0));
        if (tile == ntiles - 1) tile_jlo[ntiles] = side_n;
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int q = 0; q < INC_IPT; ++q) {
        const uint64_t i = t0 + uint32_t(q) * NT + threadIdx.x;
        if (i >= n) continue;
        if (dist[i] <= uint8_t(m)) {
            ++cnt;
            if (touched[i] & 2) {
                const uint32_t slot = append_slot(&ctr->h.n_x);
                if (slot < x_cap) {
                    xlist[slot] = uint32_t(i);
                    x_slot[i] = slot;
                } else {
                    ctr->h.overflow = 1;
                }
            }
        } else {
            const uint32_t kb = __ldg(row_ptr + i), ke = __ldg(row_ptr + i + 1);
            for (uint32_t e = kb; e < ke; ++e) touched[uint32_t(__ldg(col + e))] |= 1;
        }
    }
    uint32_t total;
    block_exclusive_scan_u32(cnt, scan_s, total);
    if (threadIdx.x == 0) tile_keep[tile] = total;
}

/// Neighbours among the side keys of the queued old rows, one thread per (queued row, off-diagonal neighbour slot), in
/// canonical order: x_ref[slot * nslots + s] = side index or IDX_NONE, x_val the matrix element.
template <int W>
static __global__ void __launch_bounds__(NT) inc_extras_kernel(ModelDev m, const uint32_t* __restrict__ table, int levels,
                                                               const uint32_t* __restrict__ xlist, uint32_t x_cap,
                                                               const uint32_t* __restrict__ side_keys, int nslots,
                                                               uint32_t* __restrict__ x_ref, double* __restrict__ x_val,
                                                               uint16_t* __restrict__ x_code,
                                                               IncCounters* __restrict__ ctr) {
    const uint32_t side_n = ctr->side_n[levels];
    const uint64_t total = uint64_t(min(ctr->h.n_x, x_cap)) * uint32_t(nslots);
    for (uint64_t t = uint64_t(blockIdx.x) * NT + threadIdx.x; t < total; t += uint64_t(gridDim.x) * NT) {
        const uint32_t xi = uint32_t(t / uint32_t(nslots));
        const int slot = int(t - uint64_t(xi) * uint32_t(nslots));
        const Key<W> key = load_key<W>(table + size_t(__ldg(xlist + xi)) * W);
        uint32_t ref = IDX_NONE;
        double a = 0.0;
        int idx = 0;
        for_each_neighbor<W>(m, key, false, [&](int, const Key<W>& kk, double amp, bool) {
            if (idx++ != slot) return;
            uint32_t pos;
            if (side_find<W>(side_keys, side_n, kk, pos)) {
                ref = pos;
                a = amp;
            }
        });
        x_ref[t] = ref;
        x_val[t] = a;
        if (x_code != nullptr && ref != IDX_NONE) {
            const uint32_t cd = vt_find(m.vtab, m.vt_n, a);
            if (cd == 0xfffeu) ctr->h.code_fail = 1u;
            x_code[t] = uint16_t(cd);
        }
    }
}

/// Entries of the new row of a surviving OLD row: untouched -> its old length; touched -> its old entries whose column
/// survives + its neighbours among the side keys.  simple = keeps every entry and gains none.
__device__ __forceinline__ uint32_t new_row_len(uint32_t i, int m, const uint8_t* __restrict__ dist, uint8_t tch,
                                                const uint32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                                const uint32_t* __restrict__ x_slot, const uint32_t* __restrict__ x_ref,
                                                int nslots, bool& simple) {
    const uint32_t kb = __ldg(row_ptr + i), ke = __ldg(row_ptr + i + 1);
    simple = (tch == 0);
    if (tch == 0) return ke - kb;
    uint32_t len = 0;
    for (uint32_t e = kb; e < ke; ++e) len += (dist[uint32_t(__ldg(col + e))] <= uint8_t(m)) ? 1u : 0u;
    if (tch & 2) {
        const uint32_t* xr = x_ref + size_t(x_slot[i]) * nslots;
        for (int s = 0; s < nslots; ++s) len += (xr[s] != IDX_NONE) ? 1u : 0u;
    }
    return len;
}

__device__ __forceinline__ uint32_t side_row_len(const uint32_t* __restrict__ s_ref, uint32_t j, int width,
                                                 const uint8_t* __restrict__ dist, int m) {
    uint32_t len = 0;
    for (int s = 0; s < width; ++s) len += side_ref_valid(s_ref[size_t(j) * width + s], dist, m) ? 1u : 0u;
    return len;
}

/// Per tile of old rows: entries of the new rows the tile produces (its surviving rows + its side keys); per old row,
/// the length of its new row and whether that row is a straight copy (simple) -- inc_compact_kernel and
/// inc_fill_kernel read them instead of walking the touched rows again.
static __global__ void __launch_bounds__(NT) inc_tile_nnz_kernel(uint32_t n, int m, const uint8_t* __restrict__ dist,
                                                                 const uint8_t* __restrict__ touched,
                                                                 const uint32_t* __restrict__ row_ptr,
                                                                 const int32_t* __restrict__ col,
                                                                 const uint32_t* __restrict__ x_slot,
                                                                 const uint32_t* __restrict__ x_ref, int nslots,
                                                                 const uint32_t* __restrict__ s_ref, int width,
                                                                 const uint32_t* __restrict__ tile_jlo,
                                                                 uint32_t* __restrict__ tile_nnz,
                                                                 uint8_t* __restrict__ row_len_new,
                                                                 uint8_t* __restrict__ simple) {
    __shared__ uint32_t scan_s[NT / 32];
    const uint32_t tile = blockIdx.x;
    const uint64_t t0 = uint64_t(tile) * INC_TILE;
    uint32_t cnt = 0;
#pragma unroll
    for (int q = 0; q < INC_IPT; ++q) {
        const uint64_t i = t0 + uint32_t(q) * NT + threadIdx.x;
        if (i >= n) continue;
        uint32_t len = 0;
        bool smp = false;
        if (dist[i] <= uint8_t(m)) len = new_row_len(uint32_t(i), m, dist, touched[i], row_ptr, col, x_slot, x_ref, nslots, smp);
        row_len_new[i] = uint8_t(len);  // (0 for a dropped row; a row holds at most MAX_ROW entries)
        simple[i] = smp ? 1 : 0;
        cnt += len;
    }
    const uint32_t jlo = tile_jlo[tile], jhi = tile_jlo[tile + 1];
    for (uint32_t j = jlo + threadIdx.x; j < jhi; j += NT) cnt += side_row_len(s_ref, j, width, dist, m);
    uint32_t total;
    block_exclusive_scan_u32(cnt, scan_s, total);
    if (threadIdx.x == 0) tile_nnz[tile] = total;
}

/// One CTA: exclusive prefixes of the per-tile kept rows and entries (in place), and the sizes of the new space.
static __global__ void __launch_bounds__(NT) inc_tile_scan_kernel(uint32_t* __restrict__ tile_keep,
                                                                  uint32_t* __restrict__ tile_nnz, uint32_t ntiles,
                                                                  int levels, IncCounters* ctr) {
    __shared__ uint32_t scan_s[NT / 32];
    const uint32_t per = (ntiles + NT - 1) / NT;
    const uint32_t b = threadIdx.x * per, e = min(ntiles, b + per);
    uint32_t sk = 0, sz = 0;
    for (uint32_t t = b; t < e; ++t) {
        sk += tile_keep[t];
        sz += tile_nnz[t];
    }
    uint32_t tk, tz;
    uint32_t rk = block_exclusive_scan_u32(sk, scan_s, tk);
    uint32_t rz = block_exclusive_scan_u32(sz, scan_s, tz);
    for (uint32_t t = b; t < e; ++t) {
        const uint32_t k = tile_keep[t], z = tile_nnz[t];
        tile_keep[t] = rk;
        tile_nnz[t] = rz;
        rk += k;
        rz += z;
    }
    if (threadIdx.x == 0) {
        const uint32_t side_n = ctr->side_n[levels];
        ctr->h.n_keep = tk;
        ctr->h.n_new = tk + side_n;
        ctr->h.nnz_new = tz;
        ctr->h.side_total = side_n;
    }
}

/// Index of local row r inside the tile's shared arrays: one pad word per 32 rows, so that both the coalesced pass
/// (thread t -> rows t, t + NT, ...) and the scan pass (thread t -> rows 8t .. 8t + 7) are free of bank conflicts.
__device__ __forceinline__ uint32_t tile_slot(uint32_t r) { return r + (r >> 5); }
constexpr int INC_TILE_PAD = INC_TILE + INC_TILE / 32;

/// The index maps and everything that hangs on them, one CTA per tile of old rows: new index of every surviving old
/// row = (kept rows before it) + (side keys whose insertion gap is <= it), new index of side key j = (kept rows before
/// its gap) + j.  Writes newidx (old -> new, IDX_NONE when dropped), the row pointer of the new CSR, per old row
/// whether its new row is a straight copy (simple), and everything about the (few) side rows: key, `full` flag, zero
/// coefficient (remap_state: new rows start at zero).  The old rows' keys, flags and coefficients follow in
/// inc_move_kernel.
template <int W>
static __global__ void __launch_bounds__(NT) inc_compact_kernel(
    uint32_t n, int m, int levels, const uint8_t* __restrict__ dist, const uint8_t* __restrict__ row_len_new,
    const uint32_t* __restrict__ side_keys, const uint32_t* __restrict__ side_gap,
    const uint8_t* __restrict__ side_dist, const uint32_t* __restrict__ s_ref, int width,
    const uint32_t* __restrict__ tile_jlo, const uint32_t* __restrict__ tile_keep_pre,
    const uint32_t* __restrict__ tile_nnz_pre, uint32_t* __restrict__ newidx, uint32_t* __restrict__ side_newidx,
    uint32_t* __restrict__ out_table, uint8_t* __restrict__ out_full, double2* __restrict__ c_new,
    uint32_t* __restrict__ row_ptr_new, uint32_t ntiles, IncCounters* ctr) {
    __shared__ uint32_t o_s[INC_TILE_PAD];    // local rank among the new rows of the tile (IDX_NONE: dropped)
    __shared__ uint32_t pk_s[INC_TILE_PAD];   // kept rows of the tile before local row r
    __shared__ uint32_t cnt_s[INC_TILE_PAD];  // side keys whose gap is local row r
    __shared__ uint32_t len_s[INC_TILE_PAD];  // entries of local row r (0 when dropped); then: entries before it in the tile
    __shared__ uint32_t sl_s[INC_TILE_PAD];   // entries of the side rows whose gap is local row r
    __shared__ uint8_t keep_s[INC_TILE];      // the row survives
    __shared__ uint32_t scan_s[NT / 32];
    const uint32_t tile = blockIdx.x;
    const uint64_t t0 = uint64_t(tile) * INC_TILE;  // first old row of the tile
    const uint32_t jlo = __ldg(tile_jlo + tile), jhi = __ldg(tile_jlo + tile + 1);
    const uint32_t P = __ldg(tile_keep_pre + tile), Q = __ldg(tile_nnz_pre + tile);
    // row lengths and survival flags (coalesced), and the side keys of the tile
    for (uint32_t r = threadIdx.x; r < INC_TILE; r += NT) {
        const uint64_t i = t0 + r;
        const bool kept = i < n && dist[i] <= uint8_t(m);
        len_s[tile_slot(r)] = kept ? uint32_t(row_len_new[i]) : 0u;
        keep_s[r] = kept ? 1 : 0;
        cnt_s[tile_slot(r)] = 0;
        sl_s[tile_slot(r)] = 0;
    }
    __syncthreads();
    for (uint32_t j = jlo + threadIdx.x; j < jhi; j += NT) {
        const uint32_t r = __ldg(side_gap + j) - uint32_t(t0);
        atomicAdd(&cnt_s[tile_slot(r)], 1u);
        atomicAdd(&sl_s[tile_slot(r)], side_row_len(s_ref, j, width, dist, m));
    }
    __syncthreads();
    // thread t owns local rows [t*IPT, (t+1)*IPT): three exclusive scans (kept rows, side keys, entries)
    const uint32_t r0 = threadIdx.x * INC_IPT;
    uint32_t keep[INC_IPT];
    uint32_t ksum = 0, csum = 0, zsum = 0;
#pragma unroll
    for (int q = 0; q < INC_IPT; ++q) {
        keep[q] = keep_s[r0 + q];
        ksum += keep[q];
        csum += cnt_s[tile_slot(r0 + q)];
        zsum += len_s[tile_slot(r0 + q)] + sl_s[tile_slot(r0 + q)];
    }
    uint32_t tot;
    const uint32_t kpre = block_exclusive_scan_u32(ksum, scan_s, tot);
    const uint32_t cpre = block_exclusive_scan_u32(csum, scan_s, tot);
    const uint32_t zpre = block_exclusive_scan_u32(zsum, scan_s, tot);
    {
        uint32_t kr = kpre, cr = cpre, zr = zpre;
#pragma unroll
        for (int q = 0; q < INC_IPT; ++q) {
            const uint32_t sl = tile_slot(r0 + q);
            const uint32_t lr = len_s[sl], sr = sl_s[sl];
            cr += cnt_s[sl];  // side keys with gap <= this row precede it
            pk_s[sl] = kr;
            o_s[sl] = keep[q] ? kr + cr : IDX_NONE;
            len_s[sl] = zr;   // entries of the tile before the side rows of gap r (those come first, then row r)
            zr += lr + sr;
            kr += keep[q];
        }
    }
    __syncthreads();
    const uint32_t base = P + jlo;  // new index of the first new row of this tile
    // ---- old rows: index map and row pointer (their keys, flags and coefficients move in inc_move_kernel)
    for (uint32_t r = threadIdx.x; r < INC_TILE; r += NT) {
        const uint64_t i = t0 + r;
        if (i >= n) break;
        const uint32_t sl = tile_slot(r);
        const uint32_t lo = o_s[sl];
        if (lo != IDX_NONE) {
            const uint32_t o = base + lo;
            newidx[i] = o;
            row_ptr_new[o] = Q + len_s[sl] + sl_s[sl];
        } else {
            newidx[i] = IDX_NONE;
        }
    }
    // ---- side keys whose gap lies in this tile (those that share a gap are consecutive: a short backward walk)
    for (uint32_t j = jlo + threadIdx.x; j < jhi; j += NT) {
        const uint32_t g = __ldg(side_gap + j);
        const uint32_t sl = tile_slot(g - uint32_t(t0));
        const uint32_t o = P + pk_s[sl] + j;
        uint32_t before = 0;
        for (uint32_t jj = j; jj > jlo && __ldg(side_gap + jj - 1) == g; --jj) before += side_row_len(s_ref, jj - 1, width, dist, m);
        side_newidx[j] = o;
        store_key<W>(out_table + size_t(o) * W, load_key<W>(side_keys + size_t(j) * W));
        out_full[o] = side_dist[j] < uint8_t(m) ? 1 : 0;
        c_new[o] = make_double2(0.0, 0.0);
        row_ptr_new[o] = Q + len_s[sl] + before;
    }
    if (threadIdx.x == 0 && tile == ntiles - 1) row_ptr_new[ctr->h.n_new] = ctr->h.nnz_new;
}

/// The bulk of the data movement, as one streaming pass over the old rows (a warp per 32 consecutive rows, several
/// batches in flight): surviving rows carry their key, `full` flag (dist < m) and coefficient to their new index
/// (remap_state, subspace.hpp:281-305: kept rows carry theirs), dropped rows add |c|^2 to the discarded weight
/// (per-CTA partials combined in CTA order by the last CTA).  Key words move word by word across the warp -- coalesced
/// reads and, over runs of surviving rows, coalesced writes.
template <int W>
static __global__ void __launch_bounds__(NT) inc_move_kernel(const uint32_t* __restrict__ table,
                                                             const double2* __restrict__ c_old, uint32_t n, int m,
                                                             const uint8_t* __restrict__ dist,
                                                             const uint32_t* __restrict__ newidx,
                                                             uint32_t* __restrict__ out_table,
                                                             uint8_t* __restrict__ out_full, double2* __restrict__ c_new,
                                                             double* __restrict__ partials, unsigned* ticket,
                                                             double* __restrict__ disc_out) {
    __shared__ double red_s[NT / 32];
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = uint64_t(gridDim.x) * (NT / 32);
    double acc[1] = {0.0};
    for (uint64_t base = (uint64_t(blockIdx.x) * (NT / 32) + (threadIdx.x >> 5)) * 32; base < n; base += nwarps * 32) {
        const uint64_t i = base + lane;
        const bool in = i < n;
        uint32_t o = IDX_NONE;
        double2 x = make_double2(0.0, 0.0);
        uint8_t d = 0;
        if (in) {
            o = __ldg(newidx + i);
            x = __ldg(c_old + i);
            d = __ldg(dist + i);
        }
        // key words of the 32 rows: word w belongs to row w / W, whose new index sits in that lane
        uint32_t kw[W];
#pragma unroll
        for (int q = 0; q < W; ++q) {
            const uint64_t w = base * W + uint32_t(q) * 32 + lane;
            kw[q] = (w < uint64_t(n) * W) ? __ldg(table + w) : 0u;
        }
#pragma unroll
        for (int q = 0; q < W; ++q) {
            const uint32_t wl = uint32_t(q) * 32 + lane;  // word index inside the batch
            const uint32_t r = wl / W;
            const uint32_t orow = __shfl_sync(0xffffffffu, o, int(r));
            if (orow != IDX_NONE) out_table[uint64_t(orow) * W + (wl - r * W)] = kw[q];
        }
        if (in) {
            if (o != IDX_NONE) {
                c_new[o] = x;
                out_full[o] = d < uint8_t(m) ? 1 : 0;
            } else {
                acc[0] = __dadd_rn(acc[0], __dadd_rn(__dmul_rn(x.x, x.x), __dmul_rn(x.y, x.y)));
            }
        }
    }
    double tot[1];
    if (grid_sum<1>(acc, partials, ticket, tot, red_s) && threadIdx.x == 0) disc_out[0] = tot[0];
}

/// Entries of the new CSR.  Old rows, a warp per 32 consecutive rows: their old entries are one contiguous run of
/// CSR_old; for the simple rows every lane moves entries of that run (source row by a 5-step search over the 32 row
/// offsets, as in assemble_compact_kernel; four chunks of 32 in flight) to the row's new offset, renumbering the column
/// through the index map -- coalesced loads and nearly coalesced stores.  The other surviving rows are written by their
/// own lane: old entries filtered by newidx, merged with the row's neighbours among the side keys (regenerated in
/// canonical = ascending new-index order).  Side rows (grid-stride over the side keys) write their valid slots.
static __global__ void __launch_bounds__(NT) inc_fill_kernel(
    uint32_t n, int levels, const uint32_t* __restrict__ newidx, const uint8_t* __restrict__ touched,
    const uint32_t* __restrict__ row_ptr, const int32_t* __restrict__ col, const double* __restrict__ val,
    const uint32_t* __restrict__ x_slot, const uint32_t* __restrict__ x_ref, const double* __restrict__ x_val, int nslots,
    const uint32_t* __restrict__ side_newidx,
    const uint32_t* __restrict__ s_ref, const double* __restrict__ s_val, int width,
    const uint32_t* __restrict__ row_ptr_new, const uint8_t* __restrict__ simple, int32_t* __restrict__ col_new,
    double* __restrict__ val_new, const IncCounters* __restrict__ ctr,
    // value codes (taylor.cuh, TaylorCodes) travel with the entries: code_old == nullptr -> none
    const uint16_t* __restrict__ code_old, const double* __restrict__ diag_old, const uint16_t* __restrict__ x_code,
    const uint16_t* __restrict__ s_code, uint16_t* __restrict__ code_new, double* __restrict__ diag_new) {
    __shared__ uint32_t dst_s[(NT / 32) * 32 * MAX_ROW];
    const uint32_t side_n = ctr->side_n[levels];
    const bool coded = code_old != nullptr;
    const bool with_val = val_new != nullptr;  // a coded space may leave the 8-byte values behind (Space::val_valid)
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = uint64_t(gridDim.x) * (NT / 32);
    uint64_t base = (uint64_t(blockIdx.x) * (NT / 32) + (threadIdx.x >> 5)) * 32;
    // the next 32 rows' offsets and new indices are requested while this batch is copied
    uint32_t rp_n = 0, o_n = IDX_NONE;
    if (base < n) {
        rp_n = __ldg(row_ptr + min(base + lane, uint64_t(n)));
        o_n = base + lane < n ? newidx[base + lane] : IDX_NONE;
    }
    for (; base < n; base += nwarps * 32) {
        const uint64_t i = base + lane;
        const bool in = i < n;
        const uint32_t rp = rp_n;
        const uint32_t o = o_n;
        {
            const uint64_t nb = base + nwarps * 32;
            if (nb < n) {
                rp_n = __ldg(row_ptr + min(nb + lane, uint64_t(n)));
                o_n = nb + lane < n ? newidx[nb + lane] : IDX_NONE;
            }
        }
        const bool kept = o != IDX_NONE;
        const uint32_t rp0 = __shfl_sync(0xffffffffu, rp, 0);
        const uint32_t end = __ldg(row_ptr + (base + 32 < n ? base + 32 : n));
        const uint32_t total = end - rp0;
        // straight copies move cooperatively (below); a batch with rows longer than a model-built H_eff has (never in
        // practice) leaves all its rows to the per-row path
        const bool smp = kept && simple[i] && total <= 32u * MAX_ROW;
        if (coded && diag_old != nullptr && kept) diag_new[o] = __ldg(diag_old + i);
        const uint32_t d0 = kept ? row_ptr_new[o] : 0u;  // new offset of the row's first entry
        const unsigned smask = __ballot_sync(0xffffffffu, smp);
        if (smask != 0) {
            // Destination of every entry of the batch: a row lane writes d0 + j for its (<= MAX_ROW) entries into the
            // warp's slice of shared memory (IDX_NONE for rows that are not straight copies), entry lanes read it back
            // coalesced -- one LDS per entry instead of a search over the 32 row offsets.
            uint32_t* dst_w = dst_s + (threadIdx.x >> 5) * (32 * MAX_ROW);
            {
                const uint32_t nxt = __shfl_down_sync(0xffffffffu, rp, 1);
                const uint32_t len = (lane == 31 ? end : nxt) - rp;
                const uint32_t st = rp - rp0;
                for (uint32_t j = 0; j < len; ++j) dst_w[st + j] = smp ? d0 + j : IDX_NONE;
            }
            __syncwarp();
            for (uint32_t k0 = 0; k0 < total; k0 += 128) {
                uint32_t dst[4];
                bool ok[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t k = k0 + uint32_t(u) * 32 + lane;
                    dst[u] = k < total ? dst_w[k] : IDX_NONE;
                    ok[u] = dst[u] != IDX_NONE;
                }
                int32_t cv[4];
                double vv[4];
                uint16_t cc[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (ok[u]) {
                        const uint32_t e = rp0 + k0 + uint32_t(u) * 32 + lane;
                        cv[u] = __ldg(col + e);
                        if (with_val) vv[u] = __ldg(val + e);
                        if (coded) cc[u] = __ldg(code_old + e);
                    }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (ok[u]) cv[u] = int32_t(newidx[uint32_t(cv[u])]);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (ok[u]) {
                        col_new[dst[u]] = cv[u];
                        if (with_val) val_new[dst[u]] = vv[u];
                        if (coded) code_new[dst[u]] = cc[u];
                    }
            }
            __syncwarp();  // the slice is rewritten by the next batch
        }
        if (!kept || smp) continue;
        // extras of this row: its neighbours among the side keys, ascending
        uint32_t xc[MAX_ROW];
        double xv[MAX_ROW];
        uint16_t xk[MAX_ROW];
        uint32_t nx = 0;
        if (touched[i] & 2) {
            const size_t xb = size_t(x_slot[i]) * nslots;
            for (int s2 = 0; s2 < nslots; ++s2) {
                const uint32_t ref = x_ref[xb + s2];
                if (ref != IDX_NONE) {
                    xc[nx] = side_newidx[ref];
                    xv[nx] = x_val[xb + s2];
                    if (coded) xk[nx] = x_code[xb + s2];
                    ++nx;
                }
            }
        }
        uint32_t w = d0;
        const uint32_t kb = rp, ke = __ldg(row_ptr + i + 1);
        uint32_t xi = 0;
        for (uint32_t e = kb; e < ke; ++e) {
            const uint32_t c = newidx[uint32_t(__ldg(col + e))];
            if (c == IDX_NONE) continue;
            while (xi < nx && xc[xi] < c) {
                col_new[w] = int32_t(xc[xi]);
                if (with_val) val_new[w] = xv[xi];
                if (coded) code_new[w] = xk[xi];
                ++w, ++xi;
            }
            col_new[w] = int32_t(c);
            if (with_val) val_new[w] = __ldg(val + e);
            if (coded) code_new[w] = __ldg(code_old + e);
            ++w;
        }
        for (; xi < nx; ++xi, ++w) {
            col_new[w] = int32_t(xc[xi]);
            if (with_val) val_new[w] = xv[xi];
            if (coded) code_new[w] = xk[xi];
        }
    }
    for (uint32_t j = blockIdx.x * NT + threadIdx.x; j < side_n; j += gridDim.x * NT) {
        const uint32_t row = side_newidx[j];
        uint32_t w = row_ptr_new[row];
        for (int s = 0; s < width; ++s) {
            const uint32_t ref = s_ref[size_t(j) * width + s];
            if (ref == IDX_NONE) continue;
            const uint32_t c = (ref & INV_SIDE) ? side_newidx[ref & ~INV_SIDE] : newidx[ref];
            if (c == IDX_NONE) continue;
            col_new[w] = int32_t(c);
            if (with_val) val_new[w] = s_val[size_t(j) * width + s];
            if (coded) {
                const uint16_t cd = s_code[size_t(j) * width + s];
                code_new[w] = cd;
                if (cd == uint16_t(0xffffu)) diag_new[row] = s_val[size_t(j) * width + s];
            }
            ++w;
        }
    }
}

/// full[i] = 1 everywhere, then 0 for the rows listed (the final frontier of a full grow_subspace).
static __global__ void __launch_bounds__(NT) inc_clear_full_kernel(const uint32_t* __restrict__ rows, uint32_t cnt,
                                                            uint8_t* __restrict__ full) {
    for (uint32_t t = blockIdx.x * NT + threadIdx.x; t < cnt; t += gridDim.x * NT) full[rows[t]] = 0;
}

}  // namespace pb
