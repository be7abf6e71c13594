// sharded.cuh -- kernels that exist only on the multi-GPU path: the table is sharded over P ranks by
// owner_of(key) (hash of the phonon part of the key); every rank keeps ITS rows in canonical order and runs
// the single-GPU kernels on them.  What is added here is the routing of keys that belong to another rank
// (expansion candidates, assembly look-up requests), the halo pack for the SpMV, and the split of the
// reductions whose global value needs an all-reduce.
#pragma once
#include "kernels.cuh"
#include "incremental.cuh"

namespace pb {

constexpr uint32_t COL_ABSENT = 0xffffffffu;
constexpr uint32_t COL_REQ = 0x80000000u;  // tmp_col marker: (COL_REQ | request id), resolved after the exchange

struct ShardCounters {
    uint32_t n_out;     // keys routed to other ranks
    uint32_t overflow;
    uint32_t n_req;     // assembly look-up requests
    uint32_t pad;
};

/// Owner of a neighbour generated from a key THIS rank owns: a hop only rewrites the exciton register, which the
/// ownership hash ignores (owner_of, keys.cuh), so the neighbour stays here; only the ladder moves need the hash.
template <int W>
__device__ __forceinline__ uint32_t neighbor_owner(const ModelDev& m, int move, const Key<W>& kk, uint32_t rank, uint32_t P) {
    return move < MAX_NB ? rank : owner_of<W>(m, kk, P);
}

/// Expansion of one BFS order on a shard.  Neighbours owned by this rank take the local path of
/// expand_window_kernel (look-up, candidate + gap when absent); the others are appended to the outgoing list
/// with their destination rank.
template <int W>
static __global__ void __launch_bounds__(NT) expand_level_sharded_kernel(
    ModelDev m, uint32_t rank, uint32_t P, const uint32_t* __restrict__ table, uint32_t n,
    const uint32_t* __restrict__ frontier, uint32_t nf, uint32_t chunk, uint32_t* __restrict__ cand_keys,
    uint32_t* __restrict__ cand_gap, uint32_t cand_cap, uint32_t* __restrict__ gap_count, GrowCounters* ctr,
    uint32_t* __restrict__ out_keys, uint32_t* __restrict__ out_dest, uint32_t out_cap, ShardCounters* sc) {
    const uint64_t wbase = (uint64_t(blockIdx.x) * (NT / 32) + (threadIdx.x >> 5)) * 32ull * chunk + (threadIdx.x & 31);
    MoveCursors cur;
    cur.reset(0xffffffffu);
    for (uint64_t f = wbase; f < min(uint64_t(nf), uint64_t(wbase + 32ull * chunk)); f += 32) {
        const uint32_t row = frontier ? __ldg(frontier + f) : uint32_t(f);
        const Key<W> k = load_key<W>(table + size_t(row) * W);
        const uint32_t e = exciton_site<W>(m, k);
        if (e != cur.site) cur.reset(e);
        for_each_neighbor<W>(m, k, false, [&](int move, const Key<W>& kk, double, bool) {
            const uint32_t dest = neighbor_owner<W>(m, move, kk, rank, P);
            if (dest == rank) {
                uint32_t pos;
                if (!cursor_find<W>(table, n, cur, move, kk, pos)) {
                    const uint32_t slot = append_slot(&ctr->n_cand);
                    if (slot < cand_cap) {
                        store_key<W>(cand_keys + size_t(slot) * W, kk);
                        cand_gap[slot] = pos;
                        atomicAdd(gap_count + pos, 1u);
                    } else {
                        ctr->overflow = 1;
                    }
                }
            } else {
                const uint32_t slot = append_slot(&sc->n_out);
                if (slot < out_cap) {
                    store_key<W>(out_keys + size_t(slot) * W, kk);
                    out_dest[slot] = dest;
                } else {
                    sc->overflow = 1;
                }
            }
        });
    }
}

/// Routing scratch on the device (Engine::route_ctr): everything a routed exchange needs stays here until ONE read-back
/// brings the shard counters and both count vectors to the host together.
struct RouteBlock {
    uint32_t fill[64];     // arrival counters of route_place_kernel
    uint32_t displ[64];    // exclusive scan of counts
    ShardCounters sc;      // counters of the kernel that produced the routed list
    uint32_t counts[64];   // elements this rank sends to each peer
    uint32_t rcounts[64];  // elements each peer sends to this rank (all-to-all of counts, on the device)
};
/// what comes back to the host (the tail of RouteBlock)
struct RouteInfo {
    ShardCounters sc;
    uint32_t counts[64];
    uint32_t rcounts[64];
};

/// The length of a routed list lives on the device (a counter of the kernel that produced it), clamped to the buffer.
__device__ __forceinline__ uint32_t routed_count(const uint32_t* cnt_ptr, uint32_t cap) { return min(__ldg(cnt_ptr), cap); }

/// counts[dest[i]]++ (P is tiny: shared-memory histogram per CTA).
static __global__ void __launch_bounds__(NT) route_count_kernel(const uint32_t* __restrict__ dest,
                                                         const uint32_t* __restrict__ cnt_ptr, uint32_t cap, uint32_t P,
                                                         uint32_t* __restrict__ counts) {
    __shared__ uint32_t sh[64];
    const uint32_t cnt = routed_count(cnt_ptr, cap);
    if (threadIdx.x < 64) sh[threadIdx.x] = 0;
    __syncthreads();
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < cnt; i += gridDim.x * NT) atomicAdd(&sh[dest[i]], 1u);
    __syncthreads();
    if (threadIdx.x < P && sh[threadIdx.x]) atomicAdd(counts + threadIdx.x, sh[threadIdx.x]);
}

/// displ = exclusive scan of counts over the P <= 64 peers (one warp pair; no trip to the host).
static __global__ void route_scan_kernel(const uint32_t* __restrict__ counts, uint32_t P, uint32_t* __restrict__ displ) {
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (uint32_t p = 0; p < P; ++p) {
            displ[p] = acc;
            acc += counts[p];
        }
    }
}

/// pos[i] = displ[dest[i]] + arrival order inside the bucket; fill[] starts at zero.
static __global__ void __launch_bounds__(NT) route_place_kernel(const uint32_t* __restrict__ dest,
                                                         const uint32_t* __restrict__ cnt_ptr, uint32_t cap,
                                                         const uint32_t* __restrict__ displ,
                                                         uint32_t* __restrict__ fill, uint32_t* __restrict__ pos) {
    const uint32_t cnt = routed_count(cnt_ptr, cap);
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < cnt; i += gridDim.x * NT) {
        const uint32_t d = dest[i];
        pos[i] = displ[d] + atomicAdd(fill + d, 1u);
    }
}

template <int W>
static __global__ void __launch_bounds__(NT) route_scatter_keys_kernel(const uint32_t* __restrict__ keys,
                                                                const uint32_t* __restrict__ pos,
                                                                const uint32_t* __restrict__ cnt_ptr, uint32_t cap,
                                                                uint32_t* __restrict__ send) {
    const uint32_t cnt = routed_count(cnt_ptr, cap);
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < cnt; i += gridDim.x * NT)
        store_key<W>(send + size_t(pos[i]) * W, load_key<W>(keys + size_t(i) * W));
}

/// Keys received from other ranks during expansion: those absent from the local table become candidates.
template <int W>
static __global__ void __launch_bounds__(NT) classify_received_kernel(const uint32_t* __restrict__ table, uint32_t n,
                                                               const uint32_t* __restrict__ recv, uint32_t nr,
                                                               uint32_t* __restrict__ cand_keys,
                                                               uint32_t* __restrict__ cand_gap, uint32_t cand_cap,
                                                               uint32_t* __restrict__ gap_count, GrowCounters* ctr) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < nr; i += gridDim.x * NT) {
        const Key<W> k = load_key<W>(recv + size_t(i) * W);
        uint32_t pos;
        if (!find_row<W>(table, n, k, pos)) {
            const uint32_t slot = append_slot(&ctr->n_cand);
            if (slot < cand_cap) {
                store_key<W>(cand_keys + size_t(slot) * W, k);
                cand_gap[slot] = pos;
                atomicAdd(gap_count + pos, 1u);
            } else {
                ctr->overflow = 1;
            }
        }
    }
}

/// Assembly pass 1 on a shard: like assemble_window_kernel, but a neighbour owned by another rank becomes a
/// look-up request; its scratch column holds COL_REQ | request id until the replies arrive.  Entries stay
/// in ascending NEIGHBOUR-KEY order (the reference's summation order), whatever their final column.
template <int W>
static __global__ void __launch_bounds__(NT) assemble_rows_sharded_kernel(
    ModelDev m, uint32_t rank, uint32_t P, const uint32_t* __restrict__ table, uint32_t n, uint32_t chunk, int width,
    uint32_t* __restrict__ tmp_col, double* __restrict__ tmp_val, uint8_t* __restrict__ tmp_move,
    uint32_t* __restrict__ tmp_cnt, uint32_t* __restrict__ req_keys, uint32_t* __restrict__ req_dest, uint32_t req_cap,
    ShardCounters* sc) {
    const uint64_t wbase = (uint64_t(blockIdx.x) * (NT / 32) + (threadIdx.x >> 5)) * 32ull * chunk + (threadIdx.x & 31);
    MoveCursors cur;
    cur.reset(0xffffffffu);
    for (uint64_t ii = wbase; ii < min(uint64_t(n), uint64_t(wbase + 32ull * chunk)); ii += 32) {
        const uint32_t i = uint32_t(ii);
        const Key<W> k = load_key<W>(table + size_t(i) * W);
        const uint32_t e = exciton_site<W>(m, k);
        if (e != cur.site) cur.reset(e);
        int len = 0;
        uint32_t* tc = tmp_col + size_t(i) * width;
        double* tv = tmp_val + size_t(i) * width;
        uint8_t* tm = tmp_move + size_t(i) * width;
        for_each_neighbor<W>(m, k, true, [&](int move, const Key<W>& kk, double amp, bool is_diag) {
            uint32_t pos = i;
            bool keep = true;
            if (!is_diag) {
                const uint32_t dest = neighbor_owner<W>(m, move, kk, rank, P);
                if (dest == rank) {
                    keep = cursor_find<W>(table, n, cur, move, kk, pos);
                } else {
                    const uint32_t r = append_slot(&sc->n_req);
                    if (r < req_cap) {
                        store_key<W>(req_keys + size_t(r) * W, kk);
                        req_dest[r] = dest;
                    } else {
                        sc->overflow = 1;
                    }
                    pos = COL_REQ | r;
                }
            }
            if (keep) {
                tc[len] = pos;
                tv[len] = amp;
                tm[len] = uint8_t(move);
                ++len;
            }
        });
        tmp_cnt[i] = uint32_t(len);
    }
}

/// What the incremental table growth leaves behind for the assembly of the new table (Engine::grow_incremental_sharded):
/// where every new row came from, the previous space's CSR with the generator's move id of every entry, and the index
/// arithmetic old row -> new row.
struct AsmHint {
    const uint32_t* origin;    // [n_new] old row index, or ORIGIN_SIDE | side index
    const uint8_t* touched;    // [n_old] 1: the row has a local side key among its neighbours (its row is searched)
    const uint32_t* newidx;    // [n_old] new index of a surviving old row, IDX_NONE for a dropped one
    const uint32_t* row_ptr;   // previous space: CSR of the local rows ...
    const int32_t* col;
    const uint8_t* move;       // ... and the move id of every entry
    uint32_t n_old;
};
constexpr uint32_t ORIGIN_SIDE = 0x80000000u;

/// Marks the surviving old rows that have a LOCAL side key among their neighbours: one thread per (side key, move).
/// (Side keys of other ranks reach a row through the look-up requests, which every row issues for all its remote
/// neighbours anyway.)
template <int W>
static __global__ void __launch_bounds__(NT) inc_shard_touch_kernel(ModelDev m, uint32_t rank, uint32_t P,
                                                                    const uint32_t* __restrict__ table, uint32_t n, int order,
                                                                    int levels, const uint8_t* __restrict__ dist,
                                                                    const uint32_t* __restrict__ side_keys, int nslots,
                                                                    uint8_t* __restrict__ touched,
                                                                    const IncCounters* __restrict__ ctr) {
    const uint32_t side_n = ctr->side_n[levels];
    const uint64_t total = uint64_t(side_n) * uint32_t(nslots);
    for (uint64_t t = uint64_t(blockIdx.x) * NT + threadIdx.x; t < total; t += uint64_t(gridDim.x) * NT) {
        const uint32_t j = uint32_t(t / uint32_t(nslots));
        const int slot = int(t - uint64_t(j) * uint32_t(nslots));
        const Key<W> key = load_key<W>(side_keys + size_t(j) * W);
        int idx = 0;
        for_each_neighbor<W>(m, key, false, [&](int move, const Key<W>& kk, double, bool) {
            if (idx++ != slot) return;
            if (neighbor_owner<W>(m, move, kk, rank, P) != rank) return;
            uint32_t pos;
            if (find_row_in4<W>(table, 0, n, kk, pos) && dist[pos] <= uint8_t(order)) touched[pos] = 1;
        });
    }
}

/// Assembly pass 1 on a shard WITH the previous space as a hint, one thread per row of the new table.  A row that
/// survived from the previous table and has no local side key among its neighbours needs NO search: the previous
/// H_eff lists every local neighbour it had, tagged with the generator's move id, and the neighbour's new index is
/// index arithmetic (S[j] + add[j] when it survived).  Side keys and touched rows search the new table.  Neighbours
/// owned by other ranks become look-up requests exactly as in assemble_rows_sharded_kernel; same scratch layout.
template <int W>
static __global__ void __launch_bounds__(NT) assemble_rows_hinted_sharded_kernel(
    ModelDev m, uint32_t rank, uint32_t P, const uint32_t* __restrict__ table, uint32_t n, int width, AsmHint h,
    uint32_t* __restrict__ tmp_col, double* __restrict__ tmp_val, uint8_t* __restrict__ tmp_move,
    uint32_t* __restrict__ tmp_cnt, uint32_t* __restrict__ req_keys, uint32_t* __restrict__ req_dest, uint32_t req_cap,
    ShardCounters* sc) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        const Key<W> k = load_key<W>(table + size_t(i) * W);
        const uint32_t org = __ldg(h.origin + i);
        const bool hinted = !(org & ORIGIN_SIDE) && !__ldg(h.touched + org);
        // the previous row lists the neighbours that were in the previous table (any rank), each tagged with its move
        // id.  Everything the generator will ask about it is fetched up front with INDEPENDENT loads -- the row's
        // columns and move ids, then the new indices of its local columns -- so a row costs three exposed latencies,
        // not one per neighbour
        uint32_t ni[MAX_ROW];
        unsigned long long mpack = ~0ull;  // 4-bit move ids of the previous entries (0xf: none)
        if (hinted) {
            const uint32_t kb = __ldg(h.row_ptr + org);
            const uint32_t olen = min(__ldg(h.row_ptr + org + 1) - kb, uint32_t(MAX_ROW));
            uint32_t oc[MAX_ROW];
#pragma unroll
            for (int u = 0; u < MAX_ROW; ++u)
                if (uint32_t(u) < olen) {
                    oc[u] = uint32_t(__ldg(h.col + kb + u));
                    mpack = (mpack & ~(0xfull << (4 * u))) | ((unsigned long long)(__ldg(h.move + kb + u) & 0xf) << (4 * u));
                }
#pragma unroll
            for (int u = 0; u < MAX_ROW; ++u) {
                ni[u] = IDX_NONE;
                if (uint32_t(u) < olen && oc[u] < h.n_old) ni[u] = __ldg(h.newidx + oc[u]);
            }
        }
        int len = 0;
        uint32_t* tc = tmp_col + size_t(i) * width;
        double* tv = tmp_val + size_t(i) * width;
        uint8_t* tm = tmp_move + size_t(i) * width;
        for_each_neighbor<W>(m, k, true, [&](int move, const Key<W>& kk, double amp, bool is_diag) {
            uint32_t pos = i;
            bool keep = true;
            if (!is_diag) {
                const uint32_t dest = neighbor_owner<W>(m, move, kk, rank, P);
                if (dest == rank) {
                    if (hinted) {
                        // the previous entry with this move id, if any (a local neighbour: its column was local)
                        pos = IDX_NONE;
#pragma unroll
                        for (int u = 0; u < MAX_ROW; ++u)
                            if (int((mpack >> (4 * u)) & 0xf) == move) pos = ni[u];
                        keep = pos != IDX_NONE;
                    } else {
                        keep = find_row_in4<W>(table, 0, n, kk, pos);
                    }
                } else {
                    const uint32_t r = append_slot(&sc->n_req);
                    if (r < req_cap) {
                        store_key<W>(req_keys + size_t(r) * W, kk);
                        req_dest[r] = dest;
                    } else {
                        sc->overflow = 1;
                    }
                    pos = COL_REQ | r;
                }
            }
            if (keep) {
                tc[len] = pos;
                tv[len] = amp;
                tm[len] = uint8_t(move);
                ++len;
            }
        });
        tmp_cnt[i] = uint32_t(len);
    }
}

/// Owner side of the look-up exchange: answer[j] = local row of the requested key or COL_ABSENT;
/// found[j] = 1/0 (scanned afterwards to build the halo send list).
template <int W>
static __global__ void __launch_bounds__(NT) answer_requests_kernel(const uint32_t* __restrict__ table, uint32_t n,
                                                             const uint32_t* __restrict__ recv, uint32_t nr,
                                                             uint32_t* __restrict__ answer,
                                                             uint32_t* __restrict__ found) {
    for (uint32_t j = blockIdx.x * NT + threadIdx.x; j < nr; j += gridDim.x * NT) {
        const Key<W> k = load_key<W>(recv + size_t(j) * W);
        uint32_t pos;
        const bool f = find_row<W>(table, n, k, pos);
        answer[j] = f ? pos : COL_ABSENT;
        found[j] = f ? 1u : 0u;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) found[nr] = 0;
}

/// Per-peer bucket boundaries of an exclusive scan, picked on the device: out[p] = scan[offs.v[p]] for p = 0..P (the
/// requests of peer p occupy [offs.v[p], offs.v[p+1]) of the bucketed list); extra != nullptr: out[65] = *extra.
/// Replaces P + 1 four-byte copies to the host per list.
struct PeerOffsets {
    uint32_t v[65];
};
struct ShardAsmInfo {
    uint32_t found_at[66];  // [0..P] scan of the found flags at the requesters' bucket boundaries
    uint32_t halo_at[66];   // [0..P] scan of the reply flags at the owners' bucket boundaries; [65] = nnz
};
static __global__ void pick_boundaries_kernel(const uint32_t* __restrict__ scan, PeerOffsets offs, uint32_t P,
                                              const uint32_t* __restrict__ extra, uint32_t* __restrict__ out) {
    if (threadIdx.x <= P) out[threadIdx.x] = scan[offs.v[threadIdx.x]];
    if (threadIdx.x == 0 && extra != nullptr) out[65] = *extra;
}

/// (rows, non-zeros, code-failure flag) of this rank as doubles, for one device all-reduce at the end of the assembly.
static __global__ void shard_sizes_kernel(uint32_t n, uint32_t nnz, const uint32_t* __restrict__ fail, double* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    out[0] = double(n);
    out[1] = double(nnz);
    out[2] = (fail != nullptr && *fail != 0) ? 1.0 : 0.0;
}

/// send_idx[found_pos[j]] = answer[j] for found requests (order preserving).
static __global__ void __launch_bounds__(NT) build_send_list_kernel(const uint32_t* __restrict__ answer,
                                                             const uint32_t* __restrict__ found_pos, uint32_t nr,
                                                             uint32_t* __restrict__ send_idx) {
    for (uint32_t j = blockIdx.x * NT + threadIdx.x; j < nr; j += gridDim.x * NT)
        if (answer[j] != COL_ABSENT) send_idx[found_pos[j]] = answer[j];
}

/// Requester side: reply[] is in send (bucketed) order.  flag[p] = reply found; scanned into halo slots.
static __global__ void __launch_bounds__(NT) reply_flags_kernel(const uint32_t* __restrict__ reply, uint32_t nreq,
                                                         uint32_t* __restrict__ flag) {
    for (uint32_t p = blockIdx.x * NT + threadIdx.x; p < nreq; p += gridDim.x * NT)
        flag[p] = (reply[p] != COL_ABSENT) ? 1u : 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) flag[nreq] = 0;
}

/// Resolves the COL_REQ markers (found -> n_local + halo slot, absent -> dropped) and closes the gaps inside the
/// row's scratch: afterwards the first row_len[i] scratch entries of row i are its CSR entries, in neighbour-key order.
static __global__ void __launch_bounds__(NT) resolve_requests_kernel(uint32_t n, int width, uint32_t* __restrict__ tmp_col,
                                                              double* __restrict__ tmp_val,
                                                              uint8_t* __restrict__ tmp_move,
                                                              const uint32_t* __restrict__ tmp_cnt,
                                                              const uint32_t* __restrict__ req_pos,
                                                              const uint32_t* __restrict__ reply,
                                                              const uint32_t* __restrict__ halo_slot,
                                                              uint32_t* __restrict__ row_len) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        uint32_t* tc = tmp_col + size_t(i) * width;
        double* tv = tmp_val + size_t(i) * width;
        uint8_t* tm = tmp_move + size_t(i) * width;
        const uint32_t cnt = tmp_cnt[i];
        uint32_t len = 0;
        for (uint32_t s = 0; s < cnt; ++s) {
            const uint32_t c0 = tc[s];
            uint32_t c = c0;
            if (c != COL_ABSENT && (c & COL_REQ)) {
                const uint32_t p = req_pos[c & ~COL_REQ];
                c = (reply[p] != COL_ABSENT) ? n + halo_slot[p] : COL_ABSENT;
            }
            if (c != COL_ABSENT) {
                if (c != c0 || len != s) tc[len] = c;
                if (len != s) {
                    tv[len] = tv[s];
                    tm[len] = tm[s];
                }
                ++len;
            }
        }
        row_len[i] = len;
    }
}

/// Pass 2 on a shard: the gap-free scratch rows -> CSR.  A warp takes 32 consecutive rows, whose entries form ONE
/// contiguous run of the CSR arrays, and writes it with coalesced stores (assemble_compact_kernel's scheme).  code !=
/// nullptr: the value codes of the Taylor tile kernels are produced on the way (encode_csr_kernel's rule: index of the
/// value in the model's table; the diagonal entry 0xffff + diag[row] when the diagonals are not tabulated; *fail when
/// a value is not in the table).
static __global__ void __launch_bounds__(NT) assemble_compact_sharded_kernel(uint32_t n, int width,
                                                                      const uint32_t* __restrict__ tmp_col,
                                                                      const double* __restrict__ tmp_val,
                                                                      const uint8_t* __restrict__ tmp_move,
                                                                      const uint32_t* __restrict__ row_ptr,
                                                                      int32_t* __restrict__ col,
                                                                      double* __restrict__ val,
                                                                      uint8_t* __restrict__ move,
                                                                      const double* __restrict__ vtab, int vt_n,
                                                                      int vt_diag, uint16_t* __restrict__ code,
                                                                      double* __restrict__ diag,
                                                                      uint32_t* __restrict__ fail) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = uint64_t(gridDim.x) * (NT / 32);
    for (uint64_t base = (uint64_t(blockIdx.x) * (NT / 32) + (threadIdx.x >> 5)) * 32; base < n; base += nwarps * 32) {
        const uint64_t i = base + lane;
        const uint32_t rp = __ldg(row_ptr + (i < n ? i : n));  // rows past the end are empty
        const uint32_t rp0 = __shfl_sync(0xffffffffu, rp, 0);
        const uint32_t end = __ldg(row_ptr + (base + 32 < n ? base + 32 : n));
        const uint32_t total = end - rp0;
        for (uint32_t k0 = 0; k0 < total; k0 += 32) {
            const uint32_t k = k0 + lane;
            const uint32_t target = rp0 + (k < total ? k : total - 1);
            uint32_t r = 0;  // last row whose offset is <= target
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, rp, (r + step) & 31);
                if (v <= target) r += step;
            }
            const uint32_t off = target - __shfl_sync(0xffffffffu, rp, r);
            if (k < total) {
                const size_t src = size_t(base + r) * width + off;
                const uint32_t cc = __ldg(tmp_col + src);
                const double v = __ldg(tmp_val + src);
                col[target] = int32_t(cc);
                val[target] = v;
                move[target] = __ldg(tmp_move + src);
                if (code != nullptr) {
                    if (!vt_diag && cc == uint32_t(base + r)) {
                        diag[base + r] = v;
                        code[target] = uint16_t(0xffffu);
                    } else {
                        uint32_t cd = vt_find(vtab, vt_n, v);
                        if (cd == 0xfffeu) {
                            *fail = 1u;
                            cd = 0;
                        }
                        code[target] = uint16_t(cd);
                    }
                }
            }
        }
    }
}

// ================================================================================================
// Incremental TABLE growth on a shard (the expansion half of incremental.cuh, across ranks).  T_new = {k : dist(k, S)
// <= m}: the kept keys S are a subset of the previous table and the previous H_eff lists every edge among its keys on
// BOTH ranks of an edge, so the ball is grown in old index space: a row pulls through its CSR columns, halo columns
// included -- the owners' distances of the halo rows travel over the SpMV's halo lists, one byte per entry and level.
// Only the rows whose neighbourhood was not complete in the previous space and the keys they bring in ("side" keys)
// are expanded by key; a neighbour owned by another rank is routed to its owner, which lowers the distance of the
// row it finds (a push: the edge of a side key is not in the old H_eff) or takes the key as a candidate.
// ================================================================================================

/// dist[i] = 0 for kept rows, DIST_INF elsewhere (n local rows + the halo slots behind them).
static __global__ void __launch_bounds__(NT) inc_dist_from_keep_kernel(const uint32_t* __restrict__ keep, uint32_t n,
                                                                       uint32_t n_ext, uint8_t* __restrict__ dist) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n_ext; i += gridDim.x * NT)
        dist[i] = (i < n && keep[i]) ? uint8_t(0) : DIST_INF;
}

/// Halo pack of the distances: send[j] = dist[send_idx[j]].
static __global__ void __launch_bounds__(NT) halo_pack_u8_kernel(const uint8_t* __restrict__ dist,
                                                                 const uint32_t* __restrict__ send_idx, uint32_t cnt,
                                                                 uint8_t* __restrict__ send) {
    for (uint32_t j = blockIdx.x * NT + threadIdx.x; j < cnt; j += gridDim.x * NT) send[j] = dist[send_idx[j]];
}

/// inc_expand_kernel on a shard: a neighbour owned by this rank takes the local path (old table -> distance k+1; side
/// list -> known; else candidate with its insertion gap), one owned elsewhere is appended to the outgoing list.
template <int W>
static __global__ void __launch_bounds__(NT) inc_expand_sharded_kernel(
    ModelDev m, uint32_t rank, uint32_t P, const uint32_t* __restrict__ table, uint32_t n,
    const uint32_t* __restrict__ elist, const uint32_t* __restrict__ side_keys, const uint8_t* __restrict__ side_dist, int k,
    int nslots, uint8_t* dist, uint32_t* __restrict__ cand_keys, uint32_t* __restrict__ cand_gap, uint32_t cand_cap, int sh,
    uint32_t* __restrict__ bucket_count, IncCounters* ctr, uint32_t* __restrict__ out_keys, uint32_t* __restrict__ out_dest,
    uint32_t out_cap, ShardCounters* sc) {
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
        for_each_neighbor<W>(m, key, false, [&](int move, const Key<W>& kk, double, bool) {
            if (idx++ != slot) return;
            const uint32_t dest = neighbor_owner<W>(m, move, kk, rank, P);
            if (dest != rank) {
                const uint32_t o = append_slot(&sc->n_out);
                if (o < out_cap) {
                    store_key<W>(out_keys + size_t(o) * W, kk);
                    out_dest[o] = dest;
                } else {
                    sc->overflow = 1;
                }
                return;
            }
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

/// Keys another rank generated at level k and this rank owns: in the old table -> that row is within k+1; in the side
/// list -> known; else a candidate of this level.
template <int W>
static __global__ void __launch_bounds__(NT) inc_classify_received_kernel(
    const uint32_t* __restrict__ table, uint32_t n, const uint32_t* __restrict__ side_keys, int k,
    const uint32_t* __restrict__ recv, uint32_t nr, uint8_t* dist, uint32_t* __restrict__ cand_keys,
    uint32_t* __restrict__ cand_gap, uint32_t cand_cap, int sh, uint32_t* __restrict__ bucket_count, IncCounters* ctr) {
    const uint32_t side_n = ctr->side_n[k];
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < nr; i += gridDim.x * NT) {
        const Key<W> kk = load_key<W>(recv + size_t(i) * W);
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
    }
}

/// add[g] = number of side keys whose insertion gap is old row g (g = 0..n; slot n: behind the last row); add[] starts
/// at zero.
static __global__ void __launch_bounds__(NT) inc_shard_mark_kernel(const uint32_t* __restrict__ side_gap, int levels,
                                                                   const IncCounters* __restrict__ ctr,
                                                                   uint32_t* __restrict__ add) {
    const uint32_t side_n = ctr->side_n[levels];
    for (uint32_t j = blockIdx.x * NT + threadIdx.x; j < side_n; j += gridDim.x * NT) atomicAdd(add + side_gap[j], 1u);
}

/// v[i] = [old row i survives] + add[i] over i = 0..n, v[n + 1] = 0.  The exclusive scan of v numbers the new table.
static __global__ void __launch_bounds__(NT) inc_shard_count_kernel(uint32_t n, int m, const uint8_t* __restrict__ dist,
                                                                    const uint32_t* __restrict__ add,
                                                                    uint32_t* __restrict__ v) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i <= n; i += gridDim.x * NT)
        v[i] = add[i] + ((i < n && dist[i] <= uint8_t(m)) ? 1u : 0u);
    if (blockIdx.x == 0 && threadIdx.x == 0) v[n + 1] = 0;
}

/// Head of the counter block after the scan (over n + 2 slots, the last one zero: vscan[n + 1] is the total).
static __global__ void inc_shard_head_kernel(uint32_t n, const uint32_t* __restrict__ vscan, int levels, IncCounters* ctr) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const uint32_t side_n = ctr->side_n[levels];
    const uint32_t n_new = vscan[n + 1];
    ctr->h.side_total = side_n;
    ctr->h.n_new = n_new;
    ctr->h.n_keep = n_new - side_n;
}

/// The new table: surviving old rows and side keys at their merged positions; full = the row's neighbourhood was
/// generated (distance < m); origin = where the row came from (the assembly hint).  Old row i -> S[i] + add[i]; side
/// key j with gap g -> S[g] + (j - first side key of gap g).  A warp moves the keys of 32 consecutive old rows word by
/// word (coalesced reads; surviving neighbours land next to each other); the few side keys follow one per thread.
template <int W>
static __global__ void __launch_bounds__(NT) inc_shard_table_kernel(uint32_t n, int m, int levels,
                                                                    const uint8_t* __restrict__ dist,
                                                                    const uint32_t* __restrict__ table,
                                                                    const uint32_t* __restrict__ side_keys,
                                                                    const uint32_t* __restrict__ side_gap,
                                                                    const uint8_t* __restrict__ side_dist,
                                                                    const uint32_t* __restrict__ add,
                                                                    const uint32_t* __restrict__ S,
                                                                    const IncCounters* __restrict__ ctr,
                                                                    uint32_t* __restrict__ words_new,
                                                                    uint8_t* __restrict__ full_new,
                                                                    uint32_t* __restrict__ origin) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = uint64_t(gridDim.x) * (NT / 32);
    for (uint64_t base = (uint64_t(blockIdx.x) * (NT / 32) + (threadIdx.x >> 5)) * 32; base < n; base += nwarps * 32) {
        const uint64_t i = base + lane;
        uint32_t o = IDX_NONE;
        if (i < n) {
            const uint8_t d = dist[i];
            if (d <= uint8_t(m)) {
                o = S[i] + add[i];
                full_new[o] = d < uint8_t(m) ? 1 : 0;
                origin[o] = uint32_t(i);
            }
        }
        const uint32_t rows = uint32_t(min(uint64_t(32), uint64_t(n) - base));
        const uint32_t* src = table + size_t(base) * W;
#pragma unroll
        for (int t = 0; t < W; ++t) {
            const uint32_t q = uint32_t(t) * 32 + lane;  // word q of the run of 32 keys
            const uint32_t r = q / uint32_t(W);
            const uint32_t dst_row = __shfl_sync(0xffffffffu, o, int(r));
            if (r < rows && dst_row != IDX_NONE) words_new[size_t(dst_row) * W + (q - r * uint32_t(W))] = __ldg(src + q);
        }
    }
    const uint32_t side_n = ctr->side_n[levels];
    for (uint32_t j = blockIdx.x * NT + threadIdx.x; j < side_n; j += gridDim.x * NT) {
        const uint32_t g = side_gap[j];
        const uint32_t o = S[g] + (j - lower_bound_u32(side_gap, side_n, g));
        store_key<W>(words_new + size_t(o) * W, load_key<W>(side_keys + size_t(j) * W));
        full_new[o] = side_dist[j] < uint8_t(m) ? 1 : 0;
        origin[o] = ORIGIN_SIDE | j;
    }
}

/// remap_state (subspace.hpp:281-305) through the same index arithmetic: the coefficient of a surviving old row moves
/// to its new position, a side key starts at zero, a dropped row adds |c|^2 to the discarded weight (per-CTA partials
/// combined in CTA order -> out[0]).
static __global__ void __launch_bounds__(NT) inc_shard_remap_kernel(uint32_t n, int m, int levels,
                                                                    const uint8_t* __restrict__ dist,
                                                                    const uint32_t* __restrict__ side_gap,
                                                                    const uint32_t* __restrict__ add,
                                                                    const uint32_t* __restrict__ S,
                                                                    const IncCounters* __restrict__ ctr,
                                                                    const double2* __restrict__ c_old,
                                                                    double2* __restrict__ c_new,
                                                                    double* __restrict__ partials, unsigned* ticket,
                                                                    double* __restrict__ out) {
    __shared__ double smem[NT / 32];
    const uint32_t side_n = ctr->side_n[levels];
    const uint64_t total = uint64_t(n) + side_n;
    double acc[1] = {0.0};
    for (uint64_t t = uint64_t(blockIdx.x) * NT + threadIdx.x; t < total; t += uint64_t(gridDim.x) * NT) {
        if (t < n) {
            const uint32_t i = uint32_t(t);
            const double2 x = c_old[i];
            if (dist[i] <= uint8_t(m))
                c_new[S[i] + add[i]] = x;
            else
                acc[0] = __dadd_rn(acc[0], __dadd_rn(__dmul_rn(x.x, x.x), __dmul_rn(x.y, x.y)));
        } else {
            const uint32_t j = uint32_t(t - n);
            const uint32_t g = side_gap[j];
            c_new[S[g] + (j - lower_bound_u32(side_gap, side_n, g))] = make_double2(0.0, 0.0);
        }
    }
    double tot[1];
    if (grid_sum<1>(acc, partials, ticket, tot, smem) && threadIdx.x == 0) out[0] = tot[0];
}

/// add[i] -> new index of old row i (IDX_NONE when it was dropped): the assembly hint needs one gather per column.
static __global__ void __launch_bounds__(NT) inc_shard_newidx_kernel(uint32_t n, int m, const uint8_t* __restrict__ dist,
                                                                     const uint32_t* __restrict__ S, uint32_t* add) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT)
        add[i] = dist[i] <= uint8_t(m) ? S[i] + add[i] : IDX_NONE;
}

/// Halo pack: send[j] = x[send_idx[j]].
static __global__ void __launch_bounds__(NT) halo_pack_kernel(const double2* __restrict__ x,
                                                       const uint32_t* __restrict__ send_idx, uint32_t cnt,
                                                       double2* __restrict__ send) {
    for (uint32_t j = blockIdx.x * NT + threadIdx.x; j < cnt; j += gridDim.x * NT) send[j] = x[send_idx[j]];
}

/// Stop rule of propagator.hpp:76-84 on the globally reduced sums of one order.  tot[0..3] / tot[4..7] are the
/// deposits of the two launches of the order (rows without / with halo columns): |term|^2 = tot[0] + tot[4],
/// |c|^2 = tot[1] + tot[5].  Every rank holds the same all-reduced numbers, hence the same flags.
static __global__ void taylor_stop_kernel(TaylorCtl* ctl, const double* __restrict__ tot, int order, double rtol) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (ctl->done || ctl->bail) return;
    const double tn = __dsqrt_rn(__dadd_rn(tot[0], tot[4])), rn = __dsqrt_rn(__dadd_rn(tot[1], tot[5]));
    if (order > ctl->order_used) ctl->order_used = order;
    ctl->last_order = order;
    ctl->last_term_norm = tn;
    ctl->last_c_norm = rn;
    const int streak = (tn <= __dmul_rn(rtol, rn)) ? ctl->streak + 1 : 0;
    ctl->streak = streak;
    if (streak >= 2) ctl->done = 1;
}

/// Paired orders on shards: order - 1 ran deferred (|term_{k}|^2 in tot[3] + tot[7], c untouched), order caught up
/// (|c_k|^2 in tot[2] + tot[6], then the sums of its own order).  One all-reduce served both orders.
static __global__ void taylor_stop_pair_kernel(TaylorCtl* ctl, const double* __restrict__ tot, int order, double rtol) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (ctl->done || ctl->bail) return;
    {
        const double tn = __dsqrt_rn(__dadd_rn(tot[3], tot[7])), rn = __dsqrt_rn(__dadd_rn(tot[2], tot[6]));
        ctl->streak = (tn <= __dmul_rn(rtol, rn)) ? ctl->streak + 1 : 0;  // the streak was 0: this cannot stop the series
        ctl->deferred += 1;
    }
    const double tn = __dsqrt_rn(__dadd_rn(tot[0], tot[4])), rn = __dsqrt_rn(__dadd_rn(tot[1], tot[5]));
    if (order > ctl->order_used) ctl->order_used = order;
    ctl->last_order = order;
    ctl->last_term_norm = tn;
    ctl->last_c_norm = rn;
    const int streak = (tn <= __dmul_rn(rtol, rn)) ? ctl->streak + 1 : 0;
    ctl->streak = streak;
    if (streak >= 2) ctl->done = 1;
}

/// flag[i] = 1 when row i has a halo column (col >= n): it has to wait for the halo exchange.
static __global__ void __launch_bounds__(NT) row_has_halo_kernel(uint32_t n, const uint32_t* __restrict__ row_ptr,
                                                                 const int32_t* __restrict__ col,
                                                                 uint32_t* __restrict__ flag) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i <= n; i += gridDim.x * NT) {
        uint32_t f = 0;
        if (i < n) {
            const uint32_t kb = __ldg(row_ptr + i), ke = __ldg(row_ptr + i + 1);
            for (uint32_t e = kb; e < ke; ++e) f |= (uint32_t(__ldg(col + e)) >= n) ? 1u : 0u;
        }
        flag[i] = f;
    }
}

/// pos = exclusive scan of flag: row i goes to bnd[pos[i]] when flagged, else to intr[i - pos[i]].
static __global__ void __launch_bounds__(NT) split_rows_kernel(uint32_t n, const uint32_t* __restrict__ flag,
                                                               const uint32_t* __restrict__ pos,
                                                               uint32_t* __restrict__ intr, uint32_t* __restrict__ bnd) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        if (flag[i])
            bnd[pos[i]] = i;
        else
            intr[i - pos[i]] = i;
    }
}

/// Marks the locally owned keys among the globally selected tie keys (truncate_select, engine.hpp:137-142).
template <int W>
static __global__ void __launch_bounds__(NT) mark_selected_kernel(ModelDev m, uint32_t rank, uint32_t P,
                                                           const uint32_t* __restrict__ table, uint32_t n,
                                                           const uint32_t* __restrict__ sel, uint32_t ns,
                                                           uint32_t* __restrict__ keep) {
    for (uint32_t j = blockIdx.x * NT + threadIdx.x; j < ns; j += gridDim.x * NT) {
        const Key<W> k = load_key<W>(sel + size_t(j) * W);
        if (owner_of<W>(m, k, P) != rank) continue;
        uint32_t pos;
        if (find_row<W>(table, n, k, pos)) keep[pos] = 1u;
    }
}

/// Gathers the keys of flagged rows (order preserving): out[pos[i]] = table[i].  (= compact_rows_kernel)

/// Members of the cutoff's group a rank contributes to the single-CTA tail of the distributed selection, and the
/// staging layout of their exchange: per rank one count word + 2 words per member.  The ranks' slots are disjoint and
/// start from zero, so an all-reduce (sum) of the buffer IS the all-gather.
constexpr uint32_t SHARD_LIST_CAP = 1024;
constexpr uint32_t SHARD_STAGE_WORDS = 1 + 2 * SHARD_LIST_CAP;

/// Copies this rank's members into its slot (nothing when the global group is too large for the tail, or nothing is cut).
static __global__ void __launch_bounds__(NT) select_stage_kernel(const unsigned long long* __restrict__ list,
                                                          const SelectCtl* __restrict__ ctl, uint32_t rank,
                                                          uint32_t* __restrict__ stage) {
    if (ctl->support <= ctl->k || ctl->count_eq > SHARD_LIST_CAP) return;
    const uint32_t cnt = min(ctl->list_n, SHARD_LIST_CAP);
    uint32_t* slot = stage + size_t(rank) * SHARD_STAGE_WORDS;
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < cnt; i += gridDim.x * NT) {
        const unsigned long long b = list[i];
        slot[1 + 2 * i] = uint32_t(b);
        slot[2 + 2 * i] = uint32_t(b >> 32);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) slot[0] = cnt;
}

/// One CTA: the all-reduced slots -> one contiguous list (same order on every rank), ctl->list_n = its length.
static __global__ void __launch_bounds__(NT) select_union_kernel(const uint32_t* __restrict__ stage, uint32_t P,
                                                          unsigned long long* __restrict__ list, SelectCtl* ctl) {
    __shared__ uint32_t off[65];
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (uint32_t r = 0; r < P; ++r) {
            off[r] = acc;
            acc += min(stage[size_t(r) * SHARD_STAGE_WORDS], SHARD_LIST_CAP);
        }
        off[P] = acc;
        ctl->list_n = acc;
    }
    __syncthreads();
    for (uint32_t r = 0; r < P; ++r) {
        const uint32_t* slot = stage + size_t(r) * SHARD_STAGE_WORDS;
        const uint32_t cnt = off[r + 1] - off[r];
        for (uint32_t i = threadIdx.x; i < cnt; i += NT)
            list[off[r] + i] = (unsigned long long)slot[1 + 2 * i] | ((unsigned long long)slot[2 + 2 * i] << 32);
    }
}

/// Pick step of the radix select on an ALL-REDUCED histogram (one CTA); see select_pass_kernel.  gsum != nullptr (first
/// digit): the all-reduced sum of the weights and support count are stored first.
static __global__ void __launch_bounds__(NT) select_pick_global_kernel(uint32_t* __restrict__ hist, int width, SelectCtl* ctl,
                                                                const double* __restrict__ gsum = nullptr) {
    __shared__ uint32_t wsum[NT / 32];
    if (gsum != nullptr) {
        if (threadIdx.x == 0) {
            ctl->norm2 = gsum[0];
            ctl->support = (unsigned long long)gsum[1];
        }
        __syncthreads();
    }
    constexpr int PER = SEL_BINS / NT;
    uint32_t loc[PER];
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        loc[j] = hist[SEL_BINS - 1 - (threadIdx.x * PER + j)];
        s += loc[j];
    }
    uint32_t tot;
    const uint32_t before = block_exclusive_scan_u32(s, wsum, tot);
    const unsigned long long k = ctl->k;
    const unsigned long long prefix = ctl->prefix;
    if (k > before && k <= (unsigned long long)before + s) {
        unsigned long long kk = k - before, gt = ctl->count_gt + before;
        int j = 0;
        for (; j < PER - 1; ++j) {
            if (kk <= loc[j]) break;
            kk -= loc[j];
            gt += loc[j];
        }
        const uint32_t d = SEL_BINS - 1 - (threadIdx.x * PER + j);
        ctl->count_eq = loc[j];
        ctl->prefix = (prefix << width) | (unsigned long long)d;
        ctl->k = kk;
        ctl->count_gt = gt;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < SEL_BINS; i += NT) hist[i] = 0;
}

}  // namespace pb
