// primitives.cuh -- device-wide building blocks shared by the paces kernels: deterministic block
// reductions with last-block finalisation, a three-kernel exclusive scan, and warp-aggregated appends.
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
// exclusive scan of uint32 (three kernels: tile sums -> spine -> apply).  Callers pass n+1 elements
// with in[n] == 0 so out[n] is the total.  out may alias in.
// ------------------------------------------------------------------------------------------------
constexpr int SCAN_IPT = 8;
constexpr int SCAN_TILE = NT * SCAN_IPT;

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

__global__ void __launch_bounds__(NT) scan_tile_sums_kernel(const uint32_t* __restrict__ in, uint64_t n,
                                                            uint32_t* __restrict__ tile_sums) {
    __shared__ uint32_t smem[NT / 32];
    const uint64_t base = uint64_t(blockIdx.x) * SCAN_TILE + uint64_t(threadIdx.x) * SCAN_IPT;
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_IPT; ++i)
        if (base + i < n) s += in[base + i];
    uint32_t tot;
    block_exclusive_scan_u32(s, smem, tot);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) scan_spine_kernel(uint32_t* __restrict__ tile_sums, uint32_t ntiles) {
    __shared__ uint32_t wsum[32];
    __shared__ uint32_t carry_s;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t base = 0; base < ntiles; base += 1024) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t v = (i < ntiles) ? tile_sums[i] : 0;
        uint32_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        uint32_t woff = 0, tot = 0;
        for (int w = 0; w < 32; ++w) {
            const uint32_t s = wsum[w];
            if (w < warp) woff += s;
            tot += s;
        }
        const uint32_t carry = carry_s;
        if (i < ntiles) tile_sums[i] = carry + woff + inc - v;
        __syncthreads();
        if (threadIdx.x == 0) carry_s = carry + tot;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(NT) scan_apply_kernel(const uint32_t* in, uint64_t n,
                                                        const uint32_t* __restrict__ tile_off, uint32_t* out) {
    __shared__ uint32_t smem[NT / 32];
    const uint64_t base = uint64_t(blockIdx.x) * SCAN_TILE + uint64_t(threadIdx.x) * SCAN_IPT;
    uint32_t v[SCAN_IPT];
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_IPT; ++i) {
        v[i] = (base + i < n) ? in[base + i] : 0;
        s += v[i];
    }
    uint32_t tot;
    uint32_t run = block_exclusive_scan_u32(s, smem, tot) + tile_off[blockIdx.x];
#pragma unroll
    for (int i = 0; i < SCAN_IPT; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
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
