// window.cuh -- warp-cooperative sliding-window look-ups in the canonical (sorted) table.
//
// Every look-up of the adapt phase has the same shape: a warp holds 32 CONSECUTIVE sorted rows, applies ONE
// order-preserving move to all of them (hop to a fixed partner / lower / raise the exciton's phonon register /
// identity for remap) and asks where the resulting keys sit in a sorted table.  The move adds a fixed multi-word
// constant to keys that share the exciton site, so the 32 queries are ascending and their answers lie in a
// window of the table only a little longer than 32 rows -- and the next 32 rows of the same warp continue where
// this window ended.  So the warp keeps ONE cursor per move (a merge join), copies table[cursor, cursor + 64) into
// its shared-memory window with coalesced asynchronous copies (LDGSTS), and each lane finishes with a 7-step binary
// search in shared memory that compares only the last few words -- 64 consecutive sorted rows share the rest.  No per-lane chains of dependent global loads, no divergence inside the search, and global traffic is
// one pass over the target range per move.
//
// Replaces the find_row calls (basis_codec.hpp:334-348) inside apply_to_rows/diff_rows (subspace.hpp:102-134,
// basis_codec.hpp:273-295), assemble_effective_hamiltonian (subspace.hpp:155-158), the final-frontier filter
// (subspace.hpp:225-241) and remap_state (subspace.hpp:281-305).
#pragma once
#include "kernels.cuh"

namespace pb {

constexpr int WIN_ROWS = 64;  // table rows per window
constexpr unsigned FULL = 0xffffffffu;

/// A window holds 64 consecutive table rows, unpadded (row r at win[r*W]).
template <int W>
struct WinRow {
    static constexpr int WORDS = WIN_ROWS * W;  // per-warp window size in words
};

/// Asynchronous 4-byte global -> shared copy (LDGSTS): the issuing lane does not wait for the data.
__device__ __forceinline__ void cp_async_u32(uint32_t* smem_dst, const uint32_t* gmem_src) {
    const unsigned d = unsigned(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

/// Lower bound + equality of q among the cnt rows of a window whose rows all share their first W-S words
/// (64 consecutive sorted rows of a large table differ only in their last few words): q is compared with that
/// common prefix once, and the binary search then looks at the last S words only.
template <int W, int S>
__device__ __forceinline__ void win_search(const uint32_t* win, uint32_t cnt, const Key<W>& q, uint32_t& lo_out,
                                           bool& eq_out) {
    int c = 0;  // q's prefix vs the window's common prefix: -1 / 0 / +1
#pragma unroll
    for (int i = W - S - 1; i >= 0; --i) {
        const uint32_t v = win[i];
        if (q.w[i] != v) c = (q.w[i] < v) ? -1 : 1;
    }
    if (c != 0) {  // q sorts before / after every row of the window
        lo_out = c < 0 ? 0u : cnt;
        eq_out = false;
        return;
    }
    uint32_t lo = 0, len = cnt;
    while (len > 0) {
        const uint32_t half = len >> 1;
        const uint32_t mid = lo + half;
        const uint32_t* r = win + mid * W + (W - S);
        bool lt = false;
#pragma unroll
        for (int j = S - 1; j >= 0; --j) {
            const uint32_t v = r[j], qq = q.w[W - S + j];
            lt = (v < qq) || (v == qq && lt);
        }
        lo = lt ? mid + 1 : lo;
        len = lt ? len - half - 1 : half;
    }
    bool eq = lo < cnt;
    if (eq) {
        const uint32_t* r = win + lo * W + (W - S);
#pragma unroll
        for (int j = 0; j < S; ++j) eq = eq && (r[j] == q.w[W - S + j]);
    }
    lo_out = lo;
    eq_out = eq;
}

/// Lower bound of k in table[0, n) by one warp: every round probes 32 rows, so a search from scratch takes
/// ceil(log33 n) rounds of independent loads; with a hint (answer within [hint-32, hint+992)) it takes two.
template <int W>
__device__ __forceinline__ uint32_t warp_lower_bound(const uint32_t* __restrict__ table, uint32_t n, const Key<W>& k,
                                                     uint32_t hint) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t lo = 0, hi = n;  // answer in [lo, hi]
    if (hint != CUR_NONE && hint <= n) {
        const uint32_t h0 = hint >= 32 ? hint - 32 : 0;
        const uint64_t p = uint64_t(h0) + 32ull * lane;
        const bool less = (p < n) && row_less_key<W>(table + size_t(p) * W, k);
        const uint32_t cnt = __popc(__ballot_sync(FULL, less));
        if (cnt == 0) {
            hi = h0;  // table[h0] >= k (or h0 == n)
        } else {
            lo = h0 + 32 * (cnt - 1) + 1;
            if (cnt < 32) {
                const uint64_t e = uint64_t(h0) + 32ull * cnt;
                hi = e < n ? uint32_t(e) : n;
            }
        }
    }
    while (hi > lo) {
        const uint32_t len = hi - lo;
        if (len <= 32) {
            const bool less = (lane < len) && row_less_key<W>(table + size_t(lo + lane) * W, k);
            lo += __popc(__ballot_sync(FULL, less));
            break;
        }
        const uint32_t stride = (len + 32) / 33;
        const uint64_t p = uint64_t(lo) + uint64_t(lane + 1) * stride - 1;
        const bool less = (p < hi) && row_less_key<W>(table + size_t(p) * W, k);
        const uint32_t cnt = __popc(__ballot_sync(FULL, less));
        const uint64_t nlo = uint64_t(lo) + uint64_t(cnt) * stride;
        const uint64_t nhi = uint64_t(lo) + uint64_t(cnt + 1) * stride - 1;
        lo = nlo < hi ? uint32_t(nlo) : hi;
        hi = (cnt < 32 && nhi < hi) ? uint32_t(nhi) : hi;
    }
    return lo;
}

template <int W>
__device__ __forceinline__ Key<W> warp_bcast_key(const Key<W>& k, int src) {
    Key<W> r;
#pragma unroll
    for (int i = 0; i < W; ++i) r.w[i] = __shfl_sync(FULL, k.w[i], src);
    return r;
}

/// Warp-wide look-up: every lane passes one query (valid or not); the VALID queries are ascending in the lane
/// index and none is smaller than any query this cursor has served before.  On return pos = lower bound of q in
/// table[0, n) and found = the row there equals q (defined where valid).  `cursor` is warp-uniform: a table
/// position not beyond the answer of any later query (CUR_NONE: unknown yet).  `win` is this warp's window.
/// Must be called by all 32 lanes.
template <int W>
__device__ __forceinline__ void warp_window_find(const uint32_t* __restrict__ table, uint32_t n, uint32_t* win,
                                                 uint32_t& cursor, const Key<W>& q, bool valid, uint32_t& pos,
                                                 bool& found) {
    const uint32_t lane = threadIdx.x & 31;
    const unsigned need = __ballot_sync(FULL, valid);
    pos = n;
    found = false;
    if (need == 0) return;
    uint32_t c = cursor;
    if (c == CUR_NONE) c = warp_lower_bound<W>(table, n, warp_bcast_key<W>(q, __ffs(need) - 1), CUR_NONE);
    bool open = valid;
    int slides = 0;
    for (;;) {
        const uint32_t cnt = min(uint32_t(WIN_ROWS), n - c);
        const uint32_t* src = table + size_t(c) * W;
        for (uint32_t w = lane; w < cnt * W; w += 32) cp_async_u32(win + w, src + w);
        cp_async_wait_all();
        __syncwarp();
        // words that differ between the first and the last row of the window: only the suffix from the first
        // such word on can differ between ANY two rows of it (the rows are sorted)
        uint32_t differs = 0;
        if (cnt > 1) {
            const bool ne = (lane < uint32_t(W)) && (win[lane] != win[(cnt - 1) * W + lane]);
            differs = __ballot_sync(FULL, ne);
        }
        const int suffix = differs ? W - (__ffs(differs) - 1) : 1;  // words the search has to look at (>= 1)
        if (open) {
            uint32_t lo;
            bool eq;
            if (suffix <= 1)
                win_search<W, 1>(win, cnt, q, lo, eq);
            else if (W >= 2 && suffix <= 2)
                win_search<W, (W >= 2 ? 2 : 1)>(win, cnt, q, lo, eq);
            else if (W >= 3 && suffix <= 3)
                win_search<W, (W >= 3 ? 3 : 1)>(win, cnt, q, lo, eq);
            else if (W >= 4 && suffix <= 4)
                win_search<W, (W >= 4 ? 4 : 1)>(win, cnt, q, lo, eq);
            else
                win_search<W, W>(win, cnt, q, lo, eq);
            if (lo < cnt || c + cnt >= n) {
                pos = c + lo;
                found = eq;
                open = false;
            }
        }
        const unsigned still = __ballot_sync(FULL, open);
        __syncwarp();
        if (still == 0) break;
        // every remaining query is larger than the whole window
        c += cnt;
        if (++slides >= 2) {  // sparse stretch: jump straight to the smallest remaining query
            c = warp_lower_bound<W>(table, n, warp_bcast_key<W>(q, __ffs(still) - 1), c);
            slides = 0;
        }
    }
    cursor = __shfl_sync(FULL, pos, 31 - __clz(need));  // later queries are larger than this batch's largest
}

/// Runs f(move, key', amp, valid) over the off-diagonal moves of a warp whose 32 rows share exciton site e, in
/// CANONICAL (ascending key) order -- hops to partners t < e | lower | [diag(k) between] | raise | hops to t > e --
/// with every lane converged (rows without the move pass valid = false).  diag() is called once, between lower
/// and raise.  Amplitudes follow lattice_models.hpp:236-248.
template <int W, class F, class D>
__device__ __forceinline__ void for_each_move_warp(const ModelDev& m, const Key<W>& k, bool live, uint32_t e, F&& f,
                                                   D&& diag) {
    const int* nbs = m.nb_site + size_t(e) * MAX_NB;
    const double* nba = m.nb_amp + size_t(e) * MAX_NB;
    int d = 0;
    for (; d < MAX_NB; ++d) {
        const int t = __ldg(nbs + d);
        if (t < 0 || uint32_t(t) > e) break;
        Key<W> kk = k;
        kk.w[0] += (uint32_t(t) - e) << (32 - m.b0);  // rewrite the exciton register (hops need b0 >= 1)
        f(d, kk, __ldg(nba + d), live);
    }
    uint32_t occ = 0;
    double ge = 0.0;
    if (m.nph > 0 && m.bp > 0) {
        occ = phonon_occ<W>(m, k, int(e));
        ge = __ldg(m.g + e);
    }
    if (ge != 0.0) {  // warp-uniform: e is
        Key<W> kk = k;
        const bool ok = live && occ >= 1;
        if (ok) set_bits<W>(kk, m.b0 + int(e) * m.bp, m.bp, occ - 1);
        f(MOVE_LOWER, kk, __dmul_rn(ge, __dsqrt_rn(double(occ))), ok);
    }
    diag();
    if (ge != 0.0) {
        Key<W> kk = k;
        const bool ok = live && occ + 1 < m.d_pho;
        if (ok) set_bits<W>(kk, m.b0 + int(e) * m.bp, m.bp, occ + 1);
        f(MOVE_RAISE, kk, __dmul_rn(ge, __dsqrt_rn(double(occ + 1))), ok);
    }
    for (; d < MAX_NB; ++d) {
        const int t = __ldg(nbs + d);
        if (t < 0) break;
        Key<W> kk = k;
        kk.w[0] += (uint32_t(t) - e) << (32 - m.b0);
        f(d, kk, __ldg(nba + d), live);
    }
}

// ================================================================================================
// K1  expansion: candidates of one BFS order
// ================================================================================================
/// For every frontier row: generate the off-diagonal neighbours (apply_terms, lattice_models.hpp:212-267;
/// apply_to_rows, subspace.hpp:102-134), look each one up in the sorted table and append those that are absent,
/// together with their insertion gap.  gap_count[g] counts the candidates that fall between table rows g-1 and g.
/// A warp walks 32*chunk consecutive frontier rows, 32 at a time.  frontier == nullptr means "all rows".
template <int W>
static __global__ void __launch_bounds__(NT) expand_window_kernel(ModelDev m, const uint32_t* __restrict__ table, uint32_t n,
                                                           const uint32_t* __restrict__ frontier, uint32_t nf,
                                                           uint32_t chunk, uint32_t* __restrict__ cand_keys,
                                                           uint32_t* __restrict__ cand_gap, uint32_t cand_cap,
                                                           uint32_t* __restrict__ gap_count, GrowCounters* ctr,
                                                           int count_emitted) {
    __shared__ uint32_t win_all[(NT / 32) * WinRow<W>::WORDS];
    __shared__ uint32_t cur_all[NT / 32][N_MOVES];
    uint32_t* win = win_all + (threadIdx.x >> 5) * WinRow<W>::WORDS;
    uint32_t* cur = cur_all[threadIdx.x >> 5];
    const uint32_t lane = threadIdx.x & 31;
    unsigned long long emitted = 0;
    const uint64_t wstart = (uint64_t(blockIdx.x) * (NT / 32) + (threadIdx.x >> 5)) * 32ull * chunk;
    const uint64_t wend = (wstart + 32ull * chunk < uint64_t(nf)) ? wstart + 32ull * chunk : uint64_t(nf);
    uint32_t cur_site = 0xffffffffu;

    auto emit_absent = [&](const Key<W>& kk, uint32_t pos) {
        const uint32_t slot = append_slot(&ctr->n_cand);
        if (slot < cand_cap) {
            store_key<W>(cand_keys + size_t(slot) * W, kk);
            cand_gap[slot] = pos;
            atomicAdd(gap_count + pos, 1u);
        } else {
            ctr->overflow = 1;
        }
    };

    for (uint64_t b = wstart; b < wend; b += 32) {
        const uint64_t f = b + lane;
        const bool live = f < nf;
        const uint32_t row = live ? (frontier ? __ldg(frontier + f) : uint32_t(f)) : 0u;
        const Key<W> k = load_key<W>(table + size_t(row) * W);
        const uint32_t e = exciton_site<W>(m, k);
        const uint32_t e0 = __shfl_sync(FULL, e, 0);
        if (count_emitted && live && diagonal_element<W>(m, k, e) != 0.0) ++emitted;
        if (!__all_sync(FULL, !live || e == e0)) {
            // the 32 rows straddle two exciton sites: independent binary searches, cursors start over
            if (live) {
                for_each_neighbor<W>(m, k, false, [&](int, const Key<W>& kk, double, bool) {
                    ++emitted;
                    uint32_t pos;
                    if (!find_row<W>(table, n, kk, pos)) emit_absent(kk, pos);
                });
            }
            cur_site = 0xffffffffu;
            __syncwarp();
            continue;
        }
        if (e0 != cur_site) {
            if (lane < N_MOVES) cur[lane] = CUR_NONE;
            cur_site = e0;
            __syncwarp();
        }
        for_each_move_warp<W>(
            m, k, live, e0,
            [&](int move, const Key<W>& kk, double, bool valid) {
                uint32_t c = cur[move], pos;
                bool found;
                __syncwarp();  // all lanes hold the cursor before lane 0 rewrites it (no other barrier if no lane is valid)
                warp_window_find<W>(table, n, win, c, kk, valid, pos, found);
                if (lane == 0) cur[move] = c;
                if (valid) {
                    ++emitted;
                    if (!found) emit_absent(kk, pos);
                }
                __syncwarp();
            },
            [] {});
    }
    if (count_emitted) {
        for (int o = 16; o > 0; o >>= 1) emitted += __shfl_xor_sync(FULL, emitted, o);
        if (lane == 0 && emitted) atomicAdd(&ctr->emitted, emitted);
    }
}

// ================================================================================================
// K3  row-wise assembly of H_eff, pass 1
// ================================================================================================
/// Row i of H_eff = {(index(k'), a) : (k', a) in apply_terms(key_i), k' in table} (replaces
/// assemble_effective_hamiltonian, subspace.hpp:142-187, and the final-frontier filter, :225-241).  Neighbours
/// are generated in ascending key order, so the found columns are already ascending.  Results are parked in
/// fixed-width scratch (stride `width`) and compacted by assemble_compact_kernel.
template <int W>
static __global__ void __launch_bounds__(NT) assemble_window_kernel(ModelDev m, const uint32_t* __restrict__ table, uint32_t n,
                                                             uint32_t chunk, int width, uint32_t* __restrict__ tmp_col,
                                                             double* __restrict__ tmp_val,
                                                             uint32_t* __restrict__ row_len) {
    __shared__ uint32_t win_all[(NT / 32) * WinRow<W>::WORDS];
    __shared__ uint32_t cur_all[NT / 32][N_MOVES];
    uint32_t* win = win_all + (threadIdx.x >> 5) * WinRow<W>::WORDS;
    uint32_t* cur = cur_all[threadIdx.x >> 5];
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t wstart = (uint64_t(blockIdx.x) * (NT / 32) + (threadIdx.x >> 5)) * 32ull * chunk;
    const uint64_t wend = (wstart + 32ull * chunk < uint64_t(n)) ? wstart + 32ull * chunk : uint64_t(n);
    uint32_t cur_site = 0xffffffffu;
    for (uint64_t b = wstart; b < wend; b += 32) {
        const uint64_t ii = b + lane;
        const bool live = ii < n;
        const uint32_t i = live ? uint32_t(ii) : 0u;
        const Key<W> k = load_key<W>(table + size_t(i) * W);
        const uint32_t e = exciton_site<W>(m, k);
        const uint32_t e0 = __shfl_sync(FULL, e, 0);
        uint32_t* tc = tmp_col + size_t(i) * width;
        double* tv = tmp_val + size_t(i) * width;
        int len = 0;
        if (!__all_sync(FULL, !live || e == e0)) {
            if (live) {
                for_each_neighbor<W>(m, k, true, [&](int, const Key<W>& kk, double amp, bool is_diag) {
                    uint32_t pos = i;
                    if (is_diag || find_row<W>(table, n, kk, pos)) {
                        tc[len] = pos;
                        tv[len] = amp;
                        ++len;
                    }
                });
                row_len[i] = uint32_t(len);
            }
            cur_site = 0xffffffffu;
            __syncwarp();
            continue;
        }
        if (e0 != cur_site) {
            if (lane < N_MOVES) cur[lane] = CUR_NONE;
            cur_site = e0;
            __syncwarp();
        }
        for_each_move_warp<W>(
            m, k, live, e0,
            [&](int move, const Key<W>& kk, double amp, bool valid) {
                uint32_t c = cur[move], pos;
                bool found;
                __syncwarp();  // all lanes hold the cursor before lane 0 rewrites it (no other barrier if no lane is valid)
                warp_window_find<W>(table, n, win, c, kk, valid, pos, found);
                if (lane == 0) cur[move] = c;
                if (valid && found) {
                    tc[len] = pos;
                    tv[len] = amp;
                    ++len;
                }
                __syncwarp();
            },
            [&] {
                if (live) {
                    const double dg = diagonal_element<W>(m, k, e0);
                    if (dg != 0.0) {
                        tc[len] = i;
                        tv[len] = dg;
                        ++len;
                    }
                }
            });
        if (live) row_len[i] = uint32_t(len);
    }
}

// ================================================================================================
// K7  remap (remap_state, subspace.hpp:281-305): merge join of the old table with the new one; copy the
//     coefficient when the key is present, otherwise add |c|^2 to the discarded weight.  dst must be zeroed.
// ================================================================================================
template <int W>
static __global__ void __launch_bounds__(NT) remap_window_kernel(const uint32_t* __restrict__ src_table,
                                                          const double2* __restrict__ src_c, uint32_t ns,
                                                          const uint32_t* __restrict__ dst_table, uint32_t nd,
                                                          uint32_t chunk, double2* __restrict__ dst_c,
                                                          double* __restrict__ partials, unsigned* ticket,
                                                          double* __restrict__ out) {
    __shared__ uint32_t win_all[(NT / 32) * WinRow<W>::WORDS];
    __shared__ double smem[NT / 32];
    uint32_t* win = win_all + (threadIdx.x >> 5) * WinRow<W>::WORDS;
    const uint32_t lane = threadIdx.x & 31;
    double acc[1] = {0.0};
    // the grid is bounded (grid_sum's partials are sized for <= 8 CTAs per SM): a warp takes every
    // (total warps)-th run of 32*chunk consecutive rows and restarts its cursor for each run
    const uint64_t span = 32ull * chunk;
    const uint64_t nwarps = uint64_t(gridDim.x) * (NT / 32);
    for (uint64_t wstart = (uint64_t(blockIdx.x) * (NT / 32) + (threadIdx.x >> 5)) * span; wstart < ns;
         wstart += nwarps * span) {
        const uint64_t wend = (wstart + span < uint64_t(ns)) ? wstart + span : uint64_t(ns);
        uint32_t cursor = CUR_NONE;
        for (uint64_t b = wstart; b < wend; b += 32) {
            const uint64_t ii = b + lane;
            const bool live = ii < ns;
            const Key<W> k = load_key<W>(src_table + size_t(live ? ii : 0) * W);
            const double2 x = live ? src_c[ii] : make_double2(0.0, 0.0);
            uint32_t pos;
            bool found;
            warp_window_find<W>(dst_table, nd, win, cursor, k, live, pos, found);
            if (live) {
                if (found)
                    dst_c[pos] = x;
                else
                    acc[0] = __dadd_rn(acc[0], __dadd_rn(__dmul_rn(x.x, x.x), __dmul_rn(x.y, x.y)));
            }
        }
    }
    double tot[1];
    if (grid_sum<1>(acc, partials, ticket, tot, smem) && threadIdx.x == 0) out[0] = tot[0];
}

}  // namespace pb
