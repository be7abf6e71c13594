// kernels.cuh -- the sm_100a kernels of the paces adapt-evolve-truncate step.
//
// Invariant shared by all of them: a basis table is ALWAYS held in canonical order (rows strictly
// ascending in word-lexicographic order), exactly like the reference's PackedBasisTable with
// sorted == true.  Consequences: (1) CSR column order == neighbour-key order, which fixes the
// floating-point summation order of every SpMV row to the reference's (SURVEY hard part 1);
// (2) uploads/downloads are plain copies; (3) neighbour look-ups are binary searches whose upper
// levels are shared by a warp working on consecutive rows (monotone moves -> monotone answers);
// (4) the x-gather of the SpMV is nearly coalesced for the same reason.
//
// Arithmetic that must match the reference bit for bit uses __dmul_rn/__dadd_rn/__dsqrt_rn so no FMA
// is ever contracted (the reference is built without -march, i.e. without FMA: proj/CMakeLists.txt:6-8).
#pragma once
#include "keys.cuh"
#include "primitives.cuh"
#include "taylor.cuh"

namespace pb {

// ================================================================================================
// K1  expansion: candidates of one BFS order
// ================================================================================================
struct GrowCounters {
    uint32_t n_cand;         // candidates not present in the table (with duplicates)
    uint32_t overflow;       // candidate buffer too small
    unsigned long long emitted;  // matrix elements emitted (transcript growth, subspace.hpp:117-123)
    uint32_t n_new;          // unique new keys (after segment dedup)
    uint32_t max_seg;        // longest gap segment seen (diagnostic)
};

// The expansion kernel itself (expand_window_kernel) lives in window.cuh.

// ================================================================================================
// K2  dedup: counting sort by insertion gap, then exact dedup + ranking inside each (tiny) gap segment
// ================================================================================================

/// The dedup kernels work on SEGMENTS of candidates: segment id = insertion gap >> sh.  sh = 0 (the full expansion:
/// one segment per gap, mean length 1-3) or a coarse bucket of 2^sh table rows (the incremental adapt phase: a few
/// 1e4 candidates against a table of millions of rows -- no table-sized counter arrays).  Inside a segment candidates
/// are ordered by KEY, which also orders them by gap (the gap is monotone in the key).  The candidate count is read
/// from device memory and clamped to nc_cap (an overflowing expansion leaves a larger count behind).
/// perm[seg_start[seg] + k] = candidate id, k = arrival order inside the segment (gap_fill starts at zero).
static __global__ void __launch_bounds__(NT) place_candidates_kernel(const uint32_t* __restrict__ cand_gap,
                                                              const uint32_t* __restrict__ nc_ptr, uint32_t nc_cap, int sh,
                                                              const uint32_t* __restrict__ seg_start,
                                                              uint32_t* __restrict__ gap_fill,
                                                              uint32_t* __restrict__ perm) {
    const uint32_t nc = min(*nc_ptr, nc_cap);  // the count stays on the device: no host round trip before the merge
    for (uint32_t c = blockIdx.x * NT + threadIdx.x; c < nc; c += gridDim.x * NT) {
        const uint32_t g = cand_gap[c] >> sh;
        const uint32_t r = atomicAdd(gap_fill + g, 1u);
        perm[seg_start[g] + r] = c;
    }
}

constexpr uint32_t SEG_DUP = 0xffffffffu;

/// One thread per placed slot s.  Inside its gap segment a candidate is a duplicate if an equal key sits
/// at a smaller slot (which copy survives is irrelevant: they are the same key).  seg_rank[s] = SEG_DUP
/// for dropped duplicates, 0 otherwise; gap_kept[g] += 1 per survivor.
template <int W>
static __global__ void __launch_bounds__(NT) segment_dedup_kernel(const uint32_t* __restrict__ cand_keys,
                                                           const uint32_t* __restrict__ cand_gap,
                                                           const uint32_t* __restrict__ perm,
                                                           const uint32_t* __restrict__ nc_ptr, uint32_t nc_cap, int sh,
                                                           const uint32_t* __restrict__ seg_start,
                                                           uint32_t* __restrict__ seg_rank,
                                                           uint32_t* __restrict__ gap_kept, GrowCounters* ctr) {
    const uint32_t nc = min(*nc_ptr, nc_cap);
    for (uint32_t s = blockIdx.x * NT + threadIdx.x; s < nc; s += gridDim.x * NT) {
        const uint32_t c = perm[s];
        const uint32_t g = cand_gap[c] >> sh;
        const uint32_t s0 = seg_start[g], s1 = seg_start[g + 1];
        const Key<W> k = load_key<W>(cand_keys + size_t(c) * W);
        bool dup = false;
        // early-exit compares: two different candidates of one gap usually differ within the first words read
        for (uint32_t t = s0; t < s && !dup; ++t) dup = row_cmp<W>(cand_keys + size_t(perm[t]) * W, k) == 0;
        seg_rank[s] = dup ? SEG_DUP : 0u;
        if (!dup) atomicAdd(gap_kept + g, 1u);
        if (ctr && s == s0 && s1 - s0 > 32) atomicMax(&ctr->max_seg, s1 - s0);
    }
}

/// Survivors get rank = number of surviving smaller keys in their segment = canonical position inside
/// the gap.  Readers only test a slot for SEG_DUP, which a concurrent rank write never produces.
template <int W>
static __global__ void __launch_bounds__(NT) segment_rank_kernel(const uint32_t* __restrict__ cand_keys,
                                                          const uint32_t* __restrict__ cand_gap,
                                                          const uint32_t* __restrict__ perm,
                                                          const uint32_t* __restrict__ nc_ptr, uint32_t nc_cap, int sh,
                                                          const uint32_t* __restrict__ seg_start,
                                                          volatile uint32_t* seg_rank) {
    const uint32_t nc = min(*nc_ptr, nc_cap);
    for (uint32_t s = blockIdx.x * NT + threadIdx.x; s < nc; s += gridDim.x * NT) {
        if (seg_rank[s] == SEG_DUP) continue;
        const uint32_t c = perm[s];
        const uint32_t g = cand_gap[c] >> sh;
        const uint32_t s0 = seg_start[g], s1 = seg_start[g + 1];
        if (s1 - s0 == 1) continue;  // alone in its gap: rank 0 already stored
        const Key<W> k = load_key<W>(cand_keys + size_t(c) * W);
        uint32_t rank = 0;
        for (uint32_t t = s0; t < s1; ++t) {
            if (t == s || seg_rank[t] == SEG_DUP) continue;
            if (row_cmp<W>(cand_keys + size_t(perm[t]) * W, k) < 0) ++rank;
        }
        seg_rank[s] = rank;
    }
}

/// Writes the merged table: old row i moves to i + (#new keys in gaps <= i); a surviving candidate in
/// gap g with rank r goes to g + kept_before[g] + r.  Also emits the next frontier (ascending row
/// indices of the new keys in the merged table).   (sort_unique_rows + diff_rows + merge_rows,
/// basis_codec.hpp:247-321, in one pass.)
template <int W>
static __global__ void __launch_bounds__(NT) merge_old_rows_kernel(const uint32_t* __restrict__ table, uint32_t n,
                                                            const uint32_t* __restrict__ kept_before,
                                                            uint32_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        const Key<W> k = load_key<W>(table + size_t(i) * W);
        store_key<W>(out + size_t(i + kept_before[i + 1]) * W, k);
    }
}

template <int W>
static __global__ void __launch_bounds__(NT) merge_new_rows_kernel(const uint32_t* __restrict__ cand_keys,
                                                            const uint32_t* __restrict__ cand_gap,
                                                            const uint32_t* __restrict__ perm,
                                                            const uint32_t* __restrict__ seg_rank,
                                                            const uint32_t* __restrict__ nc_ptr,
                                                            const uint32_t* __restrict__ kept_before,
                                                            uint32_t* __restrict__ out,
                                                            uint32_t* __restrict__ next_frontier) {
    const uint32_t nc = *nc_ptr;
    for (uint32_t s = blockIdx.x * NT + threadIdx.x; s < nc; s += gridDim.x * NT) {
        const uint32_t r = seg_rank[s];
        if (r == SEG_DUP) continue;
        const uint32_t c = perm[s];
        const uint32_t g = cand_gap[c];
        const uint32_t ord = kept_before[g] + r;  // index among all new keys, canonical order
        const uint32_t pos = g + ord;
        const Key<W> k = load_key<W>(cand_keys + size_t(c) * W);
        store_key<W>(out + size_t(pos) * W, k);
        next_frontier[ord] = pos;
    }
}

// ================================================================================================
// K3  row-wise assembly of H_eff
// ================================================================================================
constexpr int MAX_ROW = 2 * 3 + 3;  // hops (<= 6) + 2 ladder + diagonal

// Pass 1 (assemble_window_kernel) lives in window.cuh.

/// Pass 2: compact the fixed-width scratch into CSR (row_ptr from the scan of row_len).  A warp takes 32
/// consecutive rows: their entries form ONE contiguous run of the CSR arrays, so the lanes write it with
/// coalesced stores; the source row of an entry is found by a 5-step search over the 32 row offsets held in
/// registers (shuffles).
static __global__ void __launch_bounds__(NT) assemble_compact_kernel(uint32_t n, int width, const uint32_t* __restrict__ tmp_col,
                                                              const double* __restrict__ tmp_val,
                                                              const uint32_t* __restrict__ row_ptr,
                                                              int32_t* __restrict__ col, double* __restrict__ val) {
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
                col[target] = int32_t(__ldg(tmp_col + src));
                val[target] = __ldg(tmp_val + src);
            }
        }
    }
}

// ================================================================================================
// K4  fused Taylor order: taylor.cuh / taylor.cu (own translation unit)
// ================================================================================================
/// Value codes of a model-built H_eff (taylor.cuh, TaylorCodes), one thread per row: code[k] = index of val[k] in the
/// model's table of matrix elements; the diagonal entry of a row (col == row) whose values are not tabulated is coded
/// 0xffff and its value copied to diag[row].  A value that is not in the table raises *fail: the space then keeps
/// using `val`.  The row count is read from the device when n_ptr != nullptr (incremental adapt: the host does not
/// know it yet).
static __global__ void __launch_bounds__(NT) encode_csr_kernel(uint32_t n_host, const uint32_t* __restrict__ n_ptr,
                                                               const uint32_t* __restrict__ row_ptr,
                                                               const int32_t* __restrict__ col,
                                                               const double* __restrict__ val,
                                                               const double* __restrict__ vtab, int vt_n, int vt_diag,
                                                               uint16_t* __restrict__ code, double* __restrict__ diag,
                                                               uint32_t* __restrict__ fail) {
    const uint32_t n = n_ptr ? *n_ptr : n_host;
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        const uint32_t kb = __ldg(row_ptr + i), ke = __ldg(row_ptr + i + 1);
        for (uint32_t k = kb; k < ke; ++k) {
            const double v = __ldg(val + k);
            if (!vt_diag && uint32_t(__ldg(col + k)) == i) {
                diag[i] = v;
                code[k] = uint16_t(0xffffu);
                continue;
            }
            uint32_t cd = vt_find(vtab, vt_n, v);
            if (cd == 0xfffeu) {
                *fail = 1u;
                cd = 0;
            }
            code[k] = uint16_t(cd);
        }
    }
}

/// The 8-byte values of a coded H_eff, for whoever still wants them (CSR export, <H>, the row kernels): val[k] = the
/// table entry of code[k], or the row's diag for 0xffff.
static __global__ void __launch_bounds__(NT) decode_csr_kernel(uint32_t n, const uint32_t* __restrict__ row_ptr,
                                                               const uint16_t* __restrict__ code,
                                                               const double* __restrict__ diag,
                                                               const double* __restrict__ vtab,
                                                               double* __restrict__ val) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        const uint32_t kb = __ldg(row_ptr + i), ke = __ldg(row_ptr + i + 1);
        for (uint32_t k = kb; k < ke; ++k) {
            const uint32_t cd = __ldg(code + k);
            val[k] = cd == 0xffffu ? __ldg(diag + i) : __ldg(vtab + cd);
        }
    }
}

/// Plain y = H x (csr_matvec, subspace.hpp:35-43).
static __global__ void __launch_bounds__(NT) spmv_kernel(uint32_t n, const uint32_t* __restrict__ row_ptr,
                                                  const int32_t* __restrict__ col, const double* __restrict__ val,
                                                  const double2* __restrict__ x, double2* __restrict__ y) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        const uint32_t kb = __ldg(row_ptr + i), ke = __ldg(row_ptr + i + 1);
        double ar = 0.0, ai = 0.0;
        for (uint32_t k = kb; k < ke; ++k) {
            const double v = __ldg(val + k);
            const double2 xx = __ldg(x + __ldg(col + k));
            ar = __dadd_rn(ar, __dmul_rn(v, xx.x));
            ai = __dadd_rn(ai, __dmul_rn(v, xx.y));
        }
        y[i] = make_double2(ar, ai);
    }
}

// ================================================================================================
// K5  <x|H|x> (csr_expectation, subspace.hpp:46-55) fused with |x|^2 and the finiteness check of
//     expmv (propagator.hpp:55-57).  out[0] = <x|H|x>, out[1] = sum |x|^2, out[2] = #non-finite.
// ================================================================================================
static __global__ void __launch_bounds__(NT) expectation_kernel(uint32_t n, const uint32_t* __restrict__ row_ptr,
                                                         const int32_t* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double2* __restrict__ x, double* __restrict__ partials,
                                                         unsigned* ticket, double* __restrict__ out) {
    __shared__ double smem[NT / 32];
    double acc[3] = {0.0, 0.0, 0.0};
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        const uint32_t kb = __ldg(row_ptr + i), ke = __ldg(row_ptr + i + 1);
        double ar = 0.0, ai = 0.0;
        for (uint32_t k = kb; k < ke; ++k) {
            const double v = __ldg(val + k);
            const double2 xx = __ldg(x + __ldg(col + k));
            ar = __dadd_rn(ar, __dmul_rn(v, xx.x));
            ai = __dadd_rn(ai, __dmul_rn(v, xx.y));
        }
        const double2 xi = __ldg(x + i);
        // real(conj(x) * row) = xr*rr - (-xi)*ri
        acc[0] = __dadd_rn(acc[0], __dsub_rn(__dmul_rn(xi.x, ar), __dmul_rn(-xi.y, ai)));
        acc[1] = __dadd_rn(acc[1], __dadd_rn(__dmul_rn(xi.x, xi.x), __dmul_rn(xi.y, xi.y)));
        if (!isfinite(xi.x) || !isfinite(xi.y)) acc[2] = acc[2] + 1.0;
    }
    double tot[3];
    if (grid_sum<3>(acc, partials, ticket, tot, smem) && threadIdx.x == 0) {
        out[0] = tot[0];
        out[1] = tot[1];
        out[2] = tot[2];
    }
}

// ================================================================================================
// K6  truncation: weights, exact q_nom-th largest by radix select on the double's bit pattern,
//     flags, order-preserving compaction   (truncate_select, engine.hpp:107-156)
// ================================================================================================
struct SelectCtl {
    unsigned long long prefix;    // bit pattern of the cutoff being built, top digits first
    unsigned long long k;         // rank still wanted inside the current prefix group (1-based from the top)
    unsigned long long count_gt;  // weights strictly above the cutoff
    unsigned long long count_eq;  // weights equal to the cutoff
    unsigned long long support;   // weights > 0
    unsigned ticket;
    unsigned list_n;              // candidates gathered for the single-CTA tail (select_gather_kernel)
    double norm2;                 // sum of weights
    unsigned tail_done;           // 1: prefix is the full 64-bit cutoff (select_tail_kernel finished the digits)
    unsigned pad;
};

/// w_i = re^2 + im^2 (std::norm), sum and support count.
static __global__ void __launch_bounds__(NT) weights_kernel(const double2* __restrict__ c, uint32_t n, double* __restrict__ w,
                                                     double* __restrict__ partials, SelectCtl* ctl) {
    __shared__ double smem[NT / 32];
    double acc[2] = {0.0, 0.0};
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        const double2 x = c[i];
        const double ww = __dadd_rn(__dmul_rn(x.x, x.x), __dmul_rn(x.y, x.y));
        w[i] = ww;
        acc[0] = __dadd_rn(acc[0], ww);
        if (ww > 0.0) acc[1] = acc[1] + 1.0;  // exact for counts < 2^53
    }
    double tot[2];
    if (grid_sum<2>(acc, partials, &ctl->ticket, tot, smem) && threadIdx.x == 0) {
        ctl->norm2 = tot[0];
        ctl->support = (unsigned long long)tot[1];
    }
}

/// Radix select, one pass: histogram of the `width`-bit digit at `shift` over the weights whose higher
/// bits equal ctl->prefix (positive doubles order like their bit patterns, so the selection is exact),
/// then -- in the last CTA to finish -- the pick: walk the bins from the top until the wanted rank k falls
/// inside one, extend the prefix by that digit, and clear the histogram for the next pass.
constexpr int SEL_BITS = 11;
constexpr int SEL_BINS = 1 << SEL_BITS;

static __global__ void __launch_bounds__(NT) select_pass_kernel(const double* __restrict__ w, uint32_t n, int shift, int width,
                                                         SelectCtl* ctl, uint32_t* __restrict__ hist, int fuse_pick) {
    __shared__ uint32_t sh[SEL_BINS];
    __shared__ uint32_t wsum[NT / 32];
    __shared__ bool is_last;
    if (fuse_pick == 2 && ctl->support <= ctl->k) return;  // single-GPU pipeline: nothing is cut
    for (int i = threadIdx.x; i < SEL_BINS; i += NT) sh[i] = 0;
    __syncthreads();
    const unsigned long long prefix = ctl->prefix;
    const uint32_t dmask = (1u << width) - 1u;
    const int hi_shift = shift + width;
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        const double ww = w[i];
        if (!(ww > 0.0)) continue;
        const unsigned long long bits = (unsigned long long)__double_as_longlong(ww);
        if (hi_shift >= 64 || (bits >> hi_shift) == prefix) atomicAdd(&sh[uint32_t(bits >> shift) & dmask], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < SEL_BINS; i += NT) {
        const uint32_t v = sh[i];
        if (v) atomicAdd(hist + i, v);
    }
    if (!fuse_pick) return;  // sharded: the histogram is all-reduced, then select_pick_global_kernel
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(&ctl->ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    // pick: bins in DESCENDING order, thread t owns descending positions [t*PER, (t+1)*PER)
    constexpr int PER = SEL_BINS / NT;
    uint32_t loc[PER];
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        loc[j] = __ldcg(hist + (SEL_BINS - 1 - (threadIdx.x * PER + j)));
        s += loc[j];
    }
    uint32_t tot;
    const uint32_t before = block_exclusive_scan_u32(s, wsum, tot);  // weights in higher bins owned by earlier threads
    const unsigned long long k = ctl->k;
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
    if (threadIdx.x == 0) ctl->ticket = 0;
}

/// Pick step shared by the select kernels: the calling CTA (NT threads) walks the `width`-bit histogram from
/// the top bin down until the wanted rank ctl->k falls inside a bin, extends ctl->prefix by that digit and
/// updates k / count_gt / count_eq.  Bins are read from `bins` (global or shared).
__device__ __forceinline__ void select_pick_block(const uint32_t* bins, int width, SelectCtl* ctl, uint32_t* wsum) {
    constexpr int PER = SEL_BINS / NT;
    uint32_t loc[PER];
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        loc[j] = bins[SEL_BINS - 1 - (threadIdx.x * PER + j)];
        s += loc[j];
    }
    uint32_t tot;
    const uint32_t before = block_exclusive_scan_u32(s, wsum, tot);  // weights in higher bins owned by earlier threads
    const unsigned long long k = ctl->k;
    const unsigned long long prefix = ctl->prefix;
    __syncthreads();  // everyone has read k / prefix before the owner rewrites them
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
}

/// Adds one to sh[digit] for every active lane, one shared-memory atomic per distinct digit in the warp (weights
/// cluster in a few exponents, so plain per-lane atomics would serialise 32 ways on the top digit).
__device__ __forceinline__ void hist_add_aggregated(uint32_t* sh, uint32_t digit) {
    const unsigned peers = __match_any_sync(__activemask(), digit);
    if ((threadIdx.x & 31) == uint32_t(__ffs(peers) - 1)) atomicAdd(&sh[digit], uint32_t(__popc(peers)));
}

/// Selection pass 1 fused with the weights: w_i = re^2 + im^2 (std::norm, engine.hpp:113-116), their sum, the
/// support count, and the histogram of the top 11 bits (sign + exponent) of the positive weights.  The last CTA
/// to finish stores norm2 / support and, when support > q_nom (= ctl->k on entry), picks the first digit.
/// gsum != nullptr (a shard): the sums go to gsum[0..1] and the histogram stays as it is -- both are all-reduced over
/// the ranks before select_pick_global_kernel picks the digit.
static __global__ void __launch_bounds__(NT) weights_hist_kernel(const double2* __restrict__ c, uint32_t n,
                                                          double* __restrict__ w, double* __restrict__ partials,
                                                          SelectCtl* ctl, uint32_t* __restrict__ hist,
                                                          double* __restrict__ gsum = nullptr) {
    __shared__ uint32_t sh[SEL_BINS];
    __shared__ double smem[NT / 32];
    __shared__ uint32_t wsum[NT / 32];
    for (int i = threadIdx.x; i < SEL_BINS; i += NT) sh[i] = 0;
    __syncthreads();
    double acc[2] = {0.0, 0.0};
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        const double2 x = c[i];
        const double ww = __dadd_rn(__dmul_rn(x.x, x.x), __dmul_rn(x.y, x.y));
        w[i] = ww;
        acc[0] = __dadd_rn(acc[0], ww);
        if (ww > 0.0) {
            acc[1] = acc[1] + 1.0;  // exact for counts < 2^53
            hist_add_aggregated(sh, uint32_t((unsigned long long)__double_as_longlong(ww) >> 53));
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < SEL_BINS; i += NT) {
        const uint32_t v = sh[i];
        if (v) atomicAdd(hist + i, v);
    }
    __threadfence();  // the histogram contributions are visible before this CTA takes its ticket (inside grid_sum)
    double tot[2];
    if (!grid_sum<2>(acc, partials, &ctl->ticket, tot, smem)) return;
    if (gsum != nullptr) {
        if (threadIdx.x == 0) {
            gsum[0] = tot[0];
            gsum[1] = tot[1];
        }
        return;
    }
    const unsigned long long support = (unsigned long long)tot[1];
    if (threadIdx.x == 0) {
        ctl->norm2 = tot[0];
        ctl->support = support;
    }
    __syncthreads();
    if (support > ctl->k) {
        for (int i = threadIdx.x; i < SEL_BINS; i += NT) sh[i] = __ldcg(hist + i);
        __syncthreads();
        select_pick_block(sh, 11, ctl, wsum);
    }
    for (int i = threadIdx.x; i < SEL_BINS; i += NT) hist[i] = 0;
}

constexpr uint32_t SEL_LIST_CAP = 1u << 16;

/// After the first two digits (22 bits) the group that still contains the cutoff is almost always tiny: gather
/// its members' bit patterns so one CTA can finish the remaining 42 bits.  Does nothing when the group is larger
/// than the list (massive exact ties): the host then falls back to full passes.
static __global__ void __launch_bounds__(NT) select_gather_kernel(const double* __restrict__ w, uint32_t n, int hi_shift,
                                                           SelectCtl* ctl, unsigned long long* __restrict__ list,
                                                           uint32_t cap = SEL_LIST_CAP) {
    if (ctl->support <= ctl->k) return;  // nothing is cut (after a pick the wanted rank is below the support)
    if (ctl->count_eq > cap) return;
    const unsigned long long prefix = ctl->prefix;
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        const double ww = w[i];
        if (!(ww > 0.0)) continue;
        const unsigned long long bits = (unsigned long long)__double_as_longlong(ww);
        if ((bits >> hi_shift) == prefix) list[append_slot(&ctl->list_n)] = bits;
    }
}

/// Single CTA: remaining digits (shifts 31, 20, 9, 0; widths 11, 11, 11, 9) over the gathered list.
static __global__ void __launch_bounds__(NT) select_tail_kernel(const unsigned long long* __restrict__ list, SelectCtl* ctl,
                                                         uint32_t cap = SEL_LIST_CAP) {
    __shared__ uint32_t sh[SEL_BINS];
    __shared__ uint32_t wsum[NT / 32];
    const uint32_t cnt = ctl->list_n;
    if (cnt == 0 || ctl->count_eq > cap) return;
    const int shifts[4] = {31, 20, 9, 0};
    const int widths[4] = {11, 11, 11, 9};
    for (int p = 0; p < 4; ++p) {
        for (int i = threadIdx.x; i < SEL_BINS; i += NT) sh[i] = 0;
        __syncthreads();
        const unsigned long long prefix = ctl->prefix;
        const int hi_shift = shifts[p] + widths[p];
        const uint32_t dmask = (1u << widths[p]) - 1u;
        for (uint32_t i = threadIdx.x; i < cnt; i += NT) {
            const unsigned long long bits = list[i];
            if ((bits >> hi_shift) == prefix) atomicAdd(&sh[uint32_t(bits >> shifts[p]) & dmask], 1u);
        }
        __syncthreads();
        select_pick_block(sh, widths[p], ctl, wsum);
    }
    if (threadIdx.x == 0) ctl->tail_done = 1;
}

/// mode 0: keep every supported row (w > 0).  mode 1: keep w > cutoff, and w == cutoff too when
/// keep_ties; otherwise the ties are flagged separately for the host-side Fisher-Yates draw.
/// keep (uint32 flags, n + 1 entries) and dist0 (the incremental adapt phase's BFS distances: 0 = kept, 255 = not)
/// are both optional.
static __global__ void __launch_bounds__(NT) select_flags_kernel(const double* __restrict__ w, uint32_t n, int mode,
                                                          const SelectCtl* __restrict__ ctl, int keep_ties,
                                                          uint32_t* __restrict__ keep, uint32_t* __restrict__ tie,
                                                          uint8_t* __restrict__ dist0) {
    const unsigned long long cut = ctl->prefix;
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        const double ww = w[i];
        uint32_t kf = 0, tf = 0;
        if (ww > 0.0) {
            if (mode == 0) {
                kf = 1;
            } else {
                const unsigned long long bits = (unsigned long long)__double_as_longlong(ww);
                if (bits > cut)
                    kf = 1;
                else if (bits == cut) {
                    if (keep_ties)
                        kf = 1;
                    else
                        tf = 1;
                }
            }
        }
        if (keep) keep[i] = kf;
        if (dist0) dist0[i] = kf ? 0 : 255;
        if (tie) tie[i] = tf;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (keep) keep[n] = 0;
        if (tie) tie[n] = 0;
    }
}

/// idx[pos[i]] = i for flagged i (order preserving).
static __global__ void __launch_bounds__(NT) compact_index_kernel(const uint32_t* __restrict__ flag,
                                                           const uint32_t* __restrict__ pos, uint32_t n,
                                                           uint32_t* __restrict__ idx) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT)
        if (flag[i]) idx[pos[i]] = i;
}

static __global__ void set_flags_kernel(const uint32_t* __restrict__ idx, uint32_t cnt, uint32_t* __restrict__ flag,
                                        uint8_t* __restrict__ dist0) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        if (flag) flag[idx[i]] = 1;
        if (dist0) dist0[idx[i]] = 0;
    }
}

/// out[pos[i]] = table[i] for flagged rows: ascending indices of a sorted parent stay sorted
/// (engine.hpp:146-155).
template <int W>
static __global__ void __launch_bounds__(NT) compact_rows_kernel(const uint32_t* __restrict__ table,
                                                          const uint32_t* __restrict__ flag,
                                                          const uint32_t* __restrict__ pos, uint32_t n,
                                                          uint32_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        if (flag[i]) store_key<W>(out + size_t(pos[i]) * W, load_key<W>(table + size_t(i) * W));
    }
}

// K7 (remap_window_kernel) lives in window.cuh.

// ================================================================================================
// K8  observables: norm^2 + exciton density (observables.hpp:26-37), dipole overlap (:99-112),
//     phonon numbers (:84-95)
// ================================================================================================

/// The table is sorted and the exciton register is the most significant field, so the rows of one
/// site are contiguous: a CTA's chunk touches only a few sites and reduces each with the fixed tree.
/// block_part[(blockIdx, site)] partial sums are combined in CTA order by density_finish_kernel.
template <int W>
static __global__ void __launch_bounds__(NT) density_kernel(ModelDev m, const uint32_t* __restrict__ table,
                                                     const double2* __restrict__ c, uint32_t n,
                                                     uint32_t rows_per_block, double* __restrict__ block_part) {
    __shared__ double smem[NT / 32];
    __shared__ uint32_t s_lo, s_hi;
    const uint32_t r0 = blockIdx.x * rows_per_block;
    const uint32_t r1 = min(n, r0 + rows_per_block);
    if (r0 >= r1) return;
    if (threadIdx.x == 0) {
        s_lo = exciton_site<W>(m, load_key<W>(table + size_t(r0) * W));
        s_hi = exciton_site<W>(m, load_key<W>(table + size_t(r1 - 1) * W));
    }
    __syncthreads();
    const uint32_t lo = s_lo, hi = s_hi;
    for (uint32_t site = lo; site <= hi; ++site) {
        double acc = 0.0;
        for (uint32_t i = r0 + threadIdx.x; i < r1; i += NT) {
            const uint32_t e = exciton_site<W>(m, load_key<W>(table + size_t(i) * W));
            if (e == site) {
                const double2 x = c[i];
                acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(x.x, x.x), __dmul_rn(x.y, x.y)));
            }
        }
        const double t = block_sum(acc, smem);
        if (threadIdx.x == 0) block_part[size_t(blockIdx.x) * m.L + site] = t;
    }
}

/// density[site] = sum over CTAs in ascending order; one thread per site.  block_part must be zeroed
/// before density_kernel.
static __global__ void density_finish_kernel(const double* __restrict__ block_part, uint32_t nblocks, int L,
                                      double* __restrict__ density) {
    const int site = blockIdx.x * blockDim.x + threadIdx.x;
    if (site >= L) return;
    double acc = 0.0;
    for (uint32_t b = 0; b < nblocks; ++b) acc = __dadd_rn(acc, block_part[size_t(b) * L + site]);
    density[site] = acc;
}

/// amp = (1/sqrt(L)) sum_j c[find_row(|j; vacuum>)], summed in ascending j by one thread after the
/// L look-ups ran in parallel.
template <int W>
static __global__ void dipole_kernel(ModelDev m, const uint32_t* __restrict__ table, const double2* __restrict__ c,
                              uint32_t n, double2* __restrict__ found, double* __restrict__ out) {
    for (int j = threadIdx.x; j < m.L; j += blockDim.x) {
        Key<W> k;
#pragma unroll
        for (int i = 0; i < W; ++i) k.w[i] = 0;
        set_bits<W>(k, 0, m.b0, uint32_t(j));
        uint32_t pos;
        found[j] = find_row<W>(table, n, k, pos) ? c[pos] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double ar = 0.0, ai = 0.0;
        for (int j = 0; j < m.L; ++j) {
            ar = __dadd_rn(ar, found[j].x);
            ai = __dadd_rn(ai, found[j].y);
        }
        const double s = __dsqrt_rn(double(m.L));
        out[0] = __ddiv_rn(ar, s);
        out[1] = __ddiv_rn(ai, s);
    }
}

/// n_j = sum_i |c_i|^2 * occ_j(i); per-CTA partials for all L sites, combined by density_finish_kernel.
template <int W>
static __global__ void __launch_bounds__(NT) phonon_numbers_kernel(ModelDev m, const uint32_t* __restrict__ table,
                                                            const double2* __restrict__ c, uint32_t n,
                                                            uint32_t rows_per_block, double* __restrict__ block_part) {
    __shared__ double smem[NT / 32];
    const uint32_t r0 = blockIdx.x * rows_per_block;
    const uint32_t r1 = min(n, r0 + rows_per_block);
    for (int j = 0; j < m.L; ++j) {
        double acc = 0.0;
        for (uint32_t i = r0 + threadIdx.x; i < r1; i += NT) {
            const double2 x = c[i];
            const double w = __dadd_rn(__dmul_rn(x.x, x.x), __dmul_rn(x.y, x.y));
            if (w != 0.0) {
                const uint32_t occ = phonon_occ<W>(m, load_key<W>(table + size_t(i) * W), j);
                acc = __dadd_rn(acc, __dmul_rn(w, double(occ)));
            }
        }
        const double t = block_sum(acc, smem);
        if (threadIdx.x == 0) block_part[size_t(blockIdx.x) * m.L + j] = t;
    }
}

/// apply_terms for a batch of keys (lattice_models.hpp:212-267), canonical neighbour order.
template <int W>
static __global__ void apply_terms_kernel(ModelDev m, const uint32_t* __restrict__ keys, uint32_t n, int cap,
                                   uint32_t* __restrict__ out_keys, double* __restrict__ out_amps,
                                   int* __restrict__ count) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const Key<W> k = load_key<W>(keys + size_t(i) * W);
        int len = 0;
        for_each_neighbor<W>(m, k, true, [&](int, const Key<W>& kk, double amp, bool) {
            if (len < cap) {
                store_key<W>(out_keys + (size_t(i) * cap + len) * W, kk);
                out_amps[size_t(i) * cap + len] = amp;
            }
            ++len;
        });
        count[i] = len;
    }
}

/// bad[0] != 0 unless the rows are strictly ascending (PackedBasisTable::sorted, basis_codec.hpp:211).
template <int W>
static __global__ void __launch_bounds__(NT) check_sorted_kernel(const uint32_t* __restrict__ table, uint32_t n,
                                                          uint32_t* __restrict__ bad) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i + 1 < n; i += gridDim.x * NT) {
        const Key<W> a = load_key<W>(table + size_t(i) * W), b = load_key<W>(table + size_t(i + 1) * W);
        if (key_cmp<W>(a, b) >= 0) bad[0] = 1u;
    }
}

/// flag[0] = 1 unless the two word arrays are bitwise identical (host-buffer step: is the state the caller hands
/// in the one this context produced last?).
static __global__ void __launch_bounds__(NT) words_differ_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                                                          uint64_t n_words, uint32_t* __restrict__ flag) {
    bool diff = false;
    for (uint64_t i = uint64_t(blockIdx.x) * NT + threadIdx.x; i < n_words; i += uint64_t(gridDim.x) * NT)
        diff |= (a[i] != b[i]);
    if (diff) flag[0] = 1u;
}

/// L2 flush for benchmarking: streams a buffer larger than L2.
static __global__ void flush_kernel(double* __restrict__ buf, size_t n) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        buf[i] = buf[i] + 1.0;
}

}  // namespace pb
