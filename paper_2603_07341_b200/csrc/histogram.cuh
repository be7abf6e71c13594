// histogram.cuh -- weight_histogram (observables.hpp:114-176) on the device: a hand-written stable LSD radix sort of
// the weights' bit patterns (descending), a fixed-tree prefix sum of the sorted weights for the cumulative-weight
// marks, a grid reduction for the log-log tail slope and a gather of the sampled curve.  Only the sampled points and
// a 64-byte result block cross PCIe.
//
// Positive IEEE doubles order like their bit patterns, so sorting ~bits ascending sorts the weights descending and
// sends the zeros (bits == 0) to the end, where the support count cuts them off.
#pragma once
#include "kernels.cuh"

namespace pb {

constexpr int RS_BITS = 8;
constexpr int RS_BINS = 1 << RS_BITS;
constexpr int RS_IPT = 8;                 // keys per thread and tile
constexpr int RS_TILE = NT * RS_IPT;      // keys per CTA

/// keys[i] = ~bits(w_i) (ascending key order == descending weight order).
static __global__ void __launch_bounds__(NT) rs_make_keys_kernel(const double* __restrict__ w, uint32_t n,
                                                          unsigned long long* __restrict__ keys) {
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT)
        keys[i] = ~(unsigned long long)__double_as_longlong(w[i]);
}

/// Pass 1 of a radix pass: digit counts of tile b -> counts[d * ntiles + b] (digit-major, so ONE exclusive scan over
/// the whole array yields, for every (digit, tile), the output offset of that tile's first key with that digit).
static __global__ void __launch_bounds__(NT) rs_count_kernel(const unsigned long long* __restrict__ keys, uint32_t n, int shift,
                                                      uint32_t ntiles, uint32_t* __restrict__ counts) {
    __shared__ uint32_t sh[RS_BINS];
    sh[threadIdx.x] = 0;  // NT == RS_BINS
    __syncthreads();
    const uint64_t base = uint64_t(blockIdx.x) * RS_TILE;
#pragma unroll
    for (int r = 0; r < RS_IPT; ++r) {
        const uint64_t i = base + uint64_t(r) * NT + threadIdx.x;
        if (i < n) hist_add_aggregated(sh, uint32_t(keys[i] >> shift) & (RS_BINS - 1));
    }
    __syncthreads();
    counts[size_t(threadIdx.x) * ntiles + blockIdx.x] = sh[threadIdx.x];
}

/// Pass 2: stable scatter.  The tile is walked in rounds of NT consecutive keys; inside a round the warps take their
/// turn in order, and inside a warp the lanes of equal digit are ranked by lane index (match_any), so keys of equal
/// digit leave the tile in their input order.
static __global__ void __launch_bounds__(NT) rs_scatter_kernel(const unsigned long long* __restrict__ keys, uint32_t n,
                                                        int shift, uint32_t ntiles,
                                                        const uint32_t* __restrict__ offsets,
                                                        unsigned long long* __restrict__ out) {
    __shared__ uint32_t next[RS_BINS];  // output position of the tile's next key with that digit
    next[threadIdx.x] = offsets[size_t(threadIdx.x) * ntiles + blockIdx.x];
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t base = uint64_t(blockIdx.x) * RS_TILE;
    for (int r = 0; r < RS_IPT; ++r) {
        const uint64_t i = base + uint64_t(r) * NT + threadIdx.x;
        const bool live = i < n;
        const unsigned long long k = live ? keys[i] : 0ull;
        const uint32_t d = uint32_t(k >> shift) & (RS_BINS - 1);
        const unsigned act = __ballot_sync(0xffffffffu, live);
        unsigned peers = 0;
        if (live) peers = __match_any_sync(act, d);
        const uint32_t before = __popc(peers & ((1u << lane) - 1u));
        for (int w = 0; w < NT / 32; ++w) {
            if (int(warp) == w && live) {
                uint32_t pos = 0;
                const int leader = __ffs(peers) - 1;
                if (int(lane) == leader) {
                    pos = next[d];
                    next[d] = pos + __popc(peers);
                }
                pos = __shfl_sync(peers, pos, leader);
                out[pos + before] = k;
            }
            __syncthreads();
        }
    }
}

/// Sum of each tile of the sorted weights (w_i = bits(~key_i)), fixed tree.
static __global__ void __launch_bounds__(NT) wh_tile_sums_kernel(const unsigned long long* __restrict__ keys, uint32_t m,
                                                          double* __restrict__ tile_sum) {
    __shared__ double smem[NT / 32];
    const uint64_t base = uint64_t(blockIdx.x) * RS_TILE + uint64_t(threadIdx.x) * RS_IPT;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < RS_IPT; ++j)
        if (base + j < m) s = __dadd_rn(s, __longlong_as_double((long long)~keys[base + j]));
    const double t = block_sum(s, smem);
    if (threadIdx.x == 0) tile_sum[blockIdx.x] = t;
}

/// One CTA: tile_sum -> exclusive prefix (in place), total in *total_out.  Thread t owns a contiguous run of tiles.
static __global__ void __launch_bounds__(NT) wh_scan_tiles_kernel(double* __restrict__ tile_sum, uint32_t ntiles,
                                                           double* __restrict__ total_out) {
    __shared__ double part[NT];
    const uint32_t per = (ntiles + NT - 1) / NT;
    const uint32_t b = threadIdx.x * per, e = min(ntiles, b + per);
    double s = 0.0;
    for (uint32_t i = b; i < e; ++i) s = __dadd_rn(s, tile_sum[i]);
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double run = 0.0;
        for (int i = 0; i < NT; ++i) {
            const double v = part[i];
            part[i] = run;
            run = __dadd_rn(run, v);
        }
        *total_out = run;
    }
    __syncthreads();
    double run = part[threadIdx.x];
    for (uint32_t i = b; i < e; ++i) {
        const double v = tile_sum[i];
        tile_sum[i] = run;
        run = __dadd_rn(run, v);
    }
}

struct WeightHistDev {
    double total;                  // sum of the sorted weights
    unsigned long long below[4];   // #{i : running_i < fraction_j * total - 1e-15 * total}
    double sums[4];                // sx, sy, sxx, sxy over the tail ranks
    unsigned ticket;
    unsigned pad;
};

/// Cumulative-weight marks (observables.hpp:133-146): running_i = inclusive prefix of the descending weights; the
/// mark of fraction f is the first rank whose running sum reaches f*total - 1e-15*total, i.e. 1 + the number of
/// ranks below it (the running sums ascend).  Fused with the tail regression sums (:149-163) over ranks >= lo.
static __global__ void __launch_bounds__(NT) wh_marks_slope_kernel(const unsigned long long* __restrict__ keys, uint32_t m,
                                                            const double* __restrict__ tile_prefix, uint32_t lo,
                                                            double* __restrict__ partials, WeightHistDev* res) {
    __shared__ double smem[NT / 32];
    __shared__ double wtot[NT / 32];
    __shared__ unsigned long long cnt_sh[4];
    if (threadIdx.x < 4) cnt_sh[threadIdx.x] = 0;
    const double total = res->total;
    const double frac[4] = {0.50, 0.90, 0.99, 0.9999};
    double thr[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) thr[j] = __dsub_rn(__dmul_rn(frac[j], total), __dmul_rn(1e-15, total));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    uint32_t below[4] = {0, 0, 0, 0};
    for (uint32_t tile = blockIdx.x; uint64_t(tile) * RS_TILE < m; tile += gridDim.x) {
        const uint64_t base = uint64_t(tile) * RS_TILE + uint64_t(threadIdx.x) * RS_IPT;
        double v[RS_IPT];
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < RS_IPT; ++j) {
            v[j] = (base + j < m) ? __longlong_as_double((long long)~keys[base + j]) : 0.0;
            s = __dadd_rn(s, v[j]);
        }
        // exclusive prefix of the per-thread sums inside the tile: warp scan, then the warp totals in order
        double inc = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc = __dadd_rn(inc, t);
        }
        __syncthreads();
        if (lane == 31) wtot[warp] = inc;
        __syncthreads();
        double woff = 0.0;
        for (int i = 0; i < warp; ++i) woff = __dadd_rn(woff, wtot[i]);
        double run = __dadd_rn(tile_prefix[tile], __dadd_rn(woff, __dsub_rn(inc, s)));
#pragma unroll
        for (int j = 0; j < RS_IPT; ++j) {
            if (base + j >= m) break;
            run = __dadd_rn(run, v[j]);
#pragma unroll
            for (int q = 0; q < 4; ++q) below[q] += (run < thr[q]) ? 1u : 0u;
            if (base + j >= lo) {
                const double x = log(double(base + j + 1)), y = log(v[j]);
                acc[0] = __dadd_rn(acc[0], x);
                acc[1] = __dadd_rn(acc[1], y);
                acc[2] = __dadd_rn(acc[2], __dmul_rn(x, x));
                acc[3] = __dadd_rn(acc[3], __dmul_rn(x, y));
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t b = below[q];
        for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
        if (lane == 0 && b) atomicAdd(&cnt_sh[q], (unsigned long long)b);
    }
    __syncthreads();
    if (threadIdx.x < 4 && cnt_sh[threadIdx.x]) atomicAdd(&res->below[threadIdx.x], cnt_sh[threadIdx.x]);
    double tot[4];
    if (grid_sum<4>(acc, partials, &res->ticket, tot, smem) && threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) res->sums[j] = tot[j];
    }
}

/// Sampled curve (observables.hpp:166-174): point k sits at rank i = k*(m-1)/(npts-1).
static __global__ void __launch_bounds__(NT) wh_sample_kernel(const unsigned long long* __restrict__ keys, uint64_t m,
                                                       uint64_t npts, uint64_t cnt, unsigned long long* __restrict__ rank,
                                                       double* __restrict__ weight) {
    for (uint64_t k = uint64_t(blockIdx.x) * NT + threadIdx.x; k < cnt; k += uint64_t(gridDim.x) * NT) {
        const uint64_t i = npts == 1 ? 0 : k * (m - 1) / (npts - 1);
        rank[k] = i + 1;
        weight[k] = __longlong_as_double((long long)~keys[i]);
    }
}

}  // namespace pb
