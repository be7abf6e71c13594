// primitives.cuh -- device-wide building blocks shared by the paces kernels: deterministic block
// reductions with last-block finalisation, a single-pass exclusive scan, and warp-aggregated appends.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>

namespace pb {
namespace cg = cooperative_groups;

constexpr int NT = 256;  // threads per CTA for the streaming kernels

// ------------------------------------------------------------------------------------------------
// deterministic sums: fixed-shape tree inside a CTA, per-CTA partials in global memory, fixed-order
// final pass by the last CTA to arrive.  For a given (n, grid) the result is bit-reproducible.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

/// Sum over the CTA; result valid in every thread.  smem: NT/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* smem) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) smem[warp] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) t = __dadd_rn(t, smem[i]);
    return t;
}

/// Publishes K per-CTA partial sums and elects the last CTA; in that CTA (return value true in all
/// its threads) total[] holds the grid-wide sums in every thread.  partials: K * gridDim.x doubles.
template <int K>
__device__ __forceinline__ bool grid_sum(const double (&v)[K], double* partials, unsigned* ticket, double (&total)[K],
                                         double* smem) {
    __shared__ bool is_last;
    double b[K];
#pragma unroll
    for (int j = 0; j < K; ++j) b[j] = block_sum(v[j], smem);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < K; ++j) partials[size_t(j) * gridDim.x + blockIdx.x] = b[j];
        __threadfence();
        const unsigned t = atomicAdd(ticket, 1u);
        is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!is_last) return false;
    __threadfence();
#pragma unroll
    for (int j = 0; j < K; ++j) {
        double acc = 0.0;
        for (unsigned i = threadIdx.x; i < gridDim.x; i += NT)
            acc = __dadd_rn(acc, __ldcg(partials + size_t(j) * gridDim.x + i));
        total[j] = block_sum(acc, smem);
    }
    if (threadIdx.x == 0) *ticket = 0;
    return true;
}

// ------------------------------------------------------------------------------------------------
// exclusive scan of uint32.  Callers pass n+1 elements with in[n] == 0 so out[n] is the total.  out may alias in.
// ------------------------------------------------------------------------------------------------

__device__ __forceinline__ uint32_t block_exclusive_scan_u32(uint32_t v, uint32_t* smem, uint32_t& block_total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    __syncthreads();
    if (lane == 31) smem[warp] = inc;
    __syncthreads();
    uint32_t woff = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) {
        const uint32_t s = smem[i];
        if (i < warp) woff += s;
        tot += s;
    }
    block_total = tot;
    return woff + inc - v;
}

// ------------------------------------------------------------------------------------------------
// single-pass exclusive scan (decoupled look-back): every element is read once and written once.  Tiles are
// handed out through an atomic ticket so a tile's predecessors are always already running; each tile publishes
// its aggregate, looks back over the published aggregates / inclusive prefixes of earlier tiles (one warp, 32
// tiles per round) and then publishes its own inclusive prefix.  status[] and *ticket must be zero on entry.
// ------------------------------------------------------------------------------------------------
constexpr int LB_IPT = 16;
constexpr int LB_TILE = NT * LB_IPT;
constexpr unsigned long long LB_AGG = 1ull << 62, LB_PREFIX = 2ull << 62, LB_FLAGS = 3ull << 62;

/// Decoupled look-back step of a single-pass scan, for kernels that fuse the scan with their own work: the CTA that
/// owns tile `tile` (tiles are handed out through an atomic ticket, so every predecessor is already running) publishes
/// its aggregate `total`, waits for the inclusive prefix of the tiles before it and publishes its own.  Returns the
/// exclusive prefix of the tile in every thread.  status[] must be zero on entry; contains a CTA barrier.
__device__ __forceinline__ uint32_t lookback_exclusive_prefix(unsigned long long* status, uint32_t tile, uint32_t total,
                                                             uint32_t* s_prefix) {
    if (threadIdx.x == 0) {
        // 64-bit aligned stores are single transactions: flag and value arrive together
        *reinterpret_cast<volatile unsigned long long*>(status + tile) = (tile == 0 ? LB_PREFIX : LB_AGG) | total;
        if (tile == 0) *s_prefix = 0;
    }
    if (tile > 0 && threadIdx.x < 32) {
        const uint32_t lane = threadIdx.x;
        uint32_t prefix = 0;
        int64_t idx = int64_t(tile) - 1;
        for (;;) {
            const int64_t j = idx - lane;
            unsigned long long st = LB_PREFIX;  // before tile 0: an empty inclusive prefix
            if (j >= 0) {
                do {
                    st = *reinterpret_cast<volatile unsigned long long*>(status + j);
                } while ((st & LB_FLAGS) == 0);
            }
            const unsigned done = __ballot_sync(0xffffffffu, (st & LB_FLAGS) == LB_PREFIX);
            const int stop = done ? __ffs(done) - 1 : 32;  // nearest tile that already knows its inclusive prefix
            uint32_t part = (int(lane) <= stop) ? uint32_t(st) : 0u;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            prefix += part;
            if (done) break;
            idx -= 32;
        }
        if (lane == 0) {
            *reinterpret_cast<volatile unsigned long long*>(status + tile) = LB_PREFIX | (uint32_t)(prefix + total);
            *s_prefix = prefix;
        }
    }
    __syncthreads();
    return *s_prefix;
}

static __global__ void __launch_bounds__(NT) scan_lookback_kernel(const uint32_t* in, uint64_t n, uint32_t* out,
                                                           unsigned long long* status, unsigned* ticket) {
    __shared__ uint32_t smem[NT / 32];
    __shared__ uint32_t s_tile, s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t base = uint64_t(tile) * LB_TILE + uint64_t(threadIdx.x) * LB_IPT;
    uint32_t v[LB_IPT];
    if (base + LB_IPT <= n) {
        const uint4* p = reinterpret_cast<const uint4*>(in + base);
#pragma unroll
        for (int i = 0; i < LB_IPT / 4; ++i) {
            const uint4 x = p[i];
            v[4 * i] = x.x, v[4 * i + 1] = x.y, v[4 * i + 2] = x.z, v[4 * i + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < LB_IPT; ++i) v[i] = (base + i < n) ? in[base + i] : 0u;
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < LB_IPT; ++i) s += v[i];
    uint32_t total;
    const uint32_t toff = block_exclusive_scan_u32(s, smem, total);
    uint32_t run = lookback_exclusive_prefix(status, tile, total, &s_prefix) + toff;
    if (base + LB_IPT <= n) {
        uint4* q = reinterpret_cast<uint4*>(out + base);
#pragma unroll
        for (int i = 0; i < LB_IPT / 4; ++i) {
            uint4 x;
            x.x = run, run += v[4 * i];
            x.y = run, run += v[4 * i + 1];
            x.z = run, run += v[4 * i + 2];
            x.w = run, run += v[4 * i + 3];
            q[i] = x;
        }
    } else {
#pragma unroll
        for (int i = 0; i < LB_IPT; ++i) {
            if (base + i < n) out[base + i] = run;
            run += v[i];
        }
    }
}

/// Warp-aggregated append: returns a unique slot in [0, ...) from *counter for each calling thread.
__device__ __forceinline__ uint32_t append_slot(uint32_t* counter) {
    cg::coalesced_group g = cg::coalesced_threads();
    uint32_t base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(counter, g.size());
    base = g.shfl(base, 0);
    return base + g.thread_rank();
}

}  // namespace pb
