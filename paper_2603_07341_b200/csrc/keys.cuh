// keys.cuh -- packed basis keys on the device: bit fields, lexicographic order, sorted-table search
// and the closed-form Holstein / tight-binding neighbour generator.
//
// Key format (reference basis_codec.hpp:17-26, 90-128): site i gets bit_width(d_i - 1) bits, payloads
// packed back to back MSB-first into W 32-bit words, site 0 (the exciton register) in the top bits of
// word 0; a payload that straddles a word boundary keeps its high bits in the earlier word; padding
// bits are zero.  Word-lexicographic order equals occupation-vector order (basis_codec.hpp:188-194).
//
// Everything is templated on W (words per key) so a key lives in registers; runtime word indices are
// resolved with unrolled selects instead of dynamic indexing (which would spill the key to local memory).
#pragma once
#include <cstdint>

namespace pb {

constexpr int MAX_NB = 6;  // 2 * ndim hop partners per site

/// Model constants in device-readable form (closed form of the term list).
/// Layout: site 0 = exciton register with b0 bits at offset 0; phonon register j has bp bits at
/// offset b0 + j*bp (HamiltonianTermSet::phonon_slot, lattice_models.hpp:123-124).
struct ModelDev {
    int kind;        // 0 tight-binding, 1 holstein
    int L;           // lattice sites
    int nph;         // phonon registers (0 for tight binding)
    int b0;          // bits of the exciton register
    int bp;          // bits per phonon register
    int W;           // words per key
    uint32_t d_pho;  // phonon cutoff dimension
    int max_deg;     // max hop partners of a site
    const double* eps;     // [L]   onsite energies (0 where the term is absent)
    const double* omega;   // [L]   phonon frequencies (0 where absent)
    const double* g;       // [L]   vibronic couplings (0 where absent)
    const int* nb_site;    // [L*MAX_NB] hop partners sorted ascending, -1 padded; zero-amplitude bonds removed
    const double* nb_amp;  // [L*MAX_NB] bond amplitude J
    const double* omega_n;  // [nph << bp] omega[j] * double(n), the product the diagonal sums (same IEEE multiply)
    // exact shortcut for the diagonal: when eps == 0 everywhere and every omega[j] is the same integer-valued w,
    // sum_j w*n_j is a sum of small integers -- exact in ANY order -- so it equals w * (total phonon number), and
    // the total is sum_b 2^b * popcount(key & mask_b) with mask_b = bit b of every phonon register.
    int diag_uniform;            // 1: shortcut valid
    double omega_u;              // the common omega
    const uint32_t* diag_masks;  // [bp * W] multi-word masks, bit plane b at diag_masks + b*W
    int wfirst[17];        // wfirst[w] = first phonon register whose leading bit lies in key word >= w (nph past the end)
    // value codes (taylor.cuh, TaylorCodes): the distinct matrix elements the generator below can produce, ascending
    // bit patterns; vt_n == 0: the model has too many (no codes).  vt_diag: the diagonal elements are tabulated too
    // (diag_uniform models); otherwise a diagonal entry is coded CODE_DIAG and its value kept per row.
    const double* vtab;
    int vt_n;
    int vt_diag;
};

/// Code of matrix element v: its index in the table, or 0xfffe (CODE_FAIL) when it is not there.
__device__ __forceinline__ uint32_t vt_find(const double* __restrict__ vtab, int vt_n, double v) {
    const unsigned long long key = (unsigned long long)__double_as_longlong(v);
    int lo = 0, hi = vt_n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((unsigned long long)__double_as_longlong(__ldg(vtab + mid)) < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return (lo < vt_n && (unsigned long long)__double_as_longlong(__ldg(vtab + lo)) == key) ? uint32_t(lo) : 0xfffeu;
}

template <int W>
struct Key {
    uint32_t w[W];
};

template <int W>
__device__ __forceinline__ Key<W> load_key(const uint32_t* __restrict__ p) {
    Key<W> k;
#pragma unroll
    for (int i = 0; i < W; ++i) k.w[i] = __ldg(p + i);
    return k;
}

template <int W>
__device__ __forceinline__ void store_key(uint32_t* __restrict__ p, const Key<W>& k) {
#pragma unroll
    for (int i = 0; i < W; ++i) p[i] = k.w[i];
}

template <int W>
__device__ __forceinline__ bool key_equal(const Key<W>& a, const Key<W>& b) {
    bool eq = true;
#pragma unroll
    for (int i = 0; i < W; ++i) eq = eq && (a.w[i] == b.w[i]);
    return eq;
}

/// -1 / 0 / +1 for a < b / a == b / a > b in word-lexicographic order (row_less, basis_codec.hpp:188-194).
template <int W>
__device__ __forceinline__ int key_cmp(const Key<W>& a, const Key<W>& b) {
    int r = 0;
#pragma unroll
    for (int i = W - 1; i >= 0; --i) {
        if (a.w[i] != b.w[i]) r = (a.w[i] < b.w[i]) ? -1 : 1;
    }
    return r;
}

/// Compares a table row in global memory against a key, reading only as many words as needed.
template <int W>
__device__ __forceinline__ int row_cmp(const uint32_t* __restrict__ row, const Key<W>& k) {
#pragma unroll
    for (int i = 0; i < W; ++i) {
        const uint32_t v = __ldg(row + i);
        if (v != k.w[i]) return (v < k.w[i]) ? -1 : 1;
    }
    return 0;
}

/// Branch-free "row < key" with all words loaded up front (independent loads, no early-exit divergence).
template <int W>
__device__ __forceinline__ bool row_less_key(const uint32_t* __restrict__ row, const Key<W>& k) {
    uint32_t v[W];
#pragma unroll
    for (int i = 0; i < W; ++i) v[i] = __ldg(row + i);
    bool lt = false;
#pragma unroll
    for (int i = W - 1; i >= 0; --i) lt = (v[i] < k.w[i]) || (v[i] == k.w[i] && lt);
    return lt;
}

/// Lower bound of k in table[lo, hi): uniform trip count (depends only on hi - lo), conditional moves
/// instead of branches, so a warp never diverges inside the search.
template <int W>
__device__ __forceinline__ bool find_row_in(const uint32_t* __restrict__ table, uint32_t lo, uint32_t hi,
                                            const Key<W>& k, uint32_t& pos) {
    const uint32_t end = hi;
    uint32_t len = hi - lo;
    while (len > 0) {
        const uint32_t half = len >> 1;
        const uint32_t mid = lo + half;
        const bool lt = row_less_key<W>(table + size_t(mid) * W, k);
        lo = lt ? mid + 1 : lo;
        len = lt ? len - half - 1 : half;
    }
    pos = lo;
    return lo < end && row_cmp<W>(table + size_t(lo) * W, k) == 0;
}

/// The same lower bound by 4-ary steps: three pivots per round, loaded independently, so a search over n rows is
/// ~log4(n) dependent memory latencies instead of log2(n).  For the sparse look-ups of the incremental adapt phase
/// (a few 1e4 threads, each one search in a multi-million-row table: pure latency chains).
template <int W>
__device__ __forceinline__ bool find_row_in4(const uint32_t* __restrict__ table, uint32_t lo, uint32_t hi,
                                             const Key<W>& k, uint32_t& pos) {
    const uint32_t end = hi;
    while (hi - lo >= 4) {
        const uint32_t s = (hi - lo) >> 2;
        const uint32_t p1 = lo + s, p2 = p1 + s, p3 = p2 + s;
        const bool l1 = row_less_key<W>(table + size_t(p1) * W, k);
        const bool l2 = row_less_key<W>(table + size_t(p2) * W, k);
        const bool l3 = row_less_key<W>(table + size_t(p3) * W, k);
        // rows are sorted: l1 >= l2 >= l3
        const uint32_t nlo = l3 ? p3 + 1 : (l2 ? p2 + 1 : (l1 ? p1 + 1 : lo));
        const uint32_t nhi = !l1 ? p1 : (!l2 ? p2 : (!l3 ? p3 : hi));
        lo = nlo;
        hi = nhi;
    }
    uint32_t len = hi - lo;
    while (len > 0) {
        const uint32_t half = len >> 1;
        const uint32_t mid = lo + half;
        const bool lt = row_less_key<W>(table + size_t(mid) * W, k);
        lo = lt ? mid + 1 : lo;
        len = lt ? len - half - 1 : half;
    }
    pos = lo;
    return lo < end && row_cmp<W>(table + size_t(lo) * W, k) == 0;
}

/// Binary search in a sorted table (find_row, basis_codec.hpp:334-348).  Returns true and the row
/// index when present; otherwise false and the insertion point (number of rows < key).
template <int W>
__device__ __forceinline__ bool find_row(const uint32_t* __restrict__ table, uint32_t n, const Key<W>& k,
                                         uint32_t& pos) {
    return find_row_in<W>(table, 0, n, k, pos);
}

/// 64-bit mix of a key (splitmix-style), used for shard ownership.
template <int W>
__host__ __device__ __forceinline__ uint64_t key_hash_words(const uint32_t* w) {
    uint64_t h = 0x9E3779B97F4A7C15ull;
#pragma unroll
    for (int i = 0; i < W; ++i) {
        h = (h ^ w[i]) * 0xBF58476D1CE4E5B9ull;
        h ^= h >> 29;
    }
    h *= 0x94D049BB133111EBull;
    h ^= h >> 32;
    return h;
}

/// b-bit field at bit offset off (get_site, basis_codec.hpp:90-108).  b in [0, 32].
template <int W>
__device__ __forceinline__ uint32_t get_bits(const Key<W>& k, int off, int b) {
    if (b == 0) return 0;
    const int wi = off >> 5;
    uint32_t hi = 0, lo = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) {
        if (i == wi) hi = k.w[i];
        if (i == wi + 1) lo = k.w[i];
    }
    const uint64_t win = (uint64_t(hi) << 32) | lo;
    const int sh = 64 - (off & 31) - b;
    const uint64_t mask = (b >= 32) ? 0xffffffffull : ((1ull << b) - 1);
    return uint32_t((win >> sh) & mask);
}

/// Overwrites the b-bit field at bit offset off (set_site, basis_codec.hpp:111-128).
template <int W>
__device__ __forceinline__ void set_bits(Key<W>& k, int off, int b, uint32_t value) {
    if (b == 0) return;
    const int wi = off >> 5;
    const int sh = 64 - (off & 31) - b;
    const uint64_t mask = ((b >= 32) ? 0xffffffffull : ((1ull << b) - 1)) << sh;
    const uint64_t val = (uint64_t(value) << sh) & mask;
    const uint32_t mhi = uint32_t(mask >> 32), mlo = uint32_t(mask);
    const uint32_t vhi = uint32_t(val >> 32), vlo = uint32_t(val);
#pragma unroll
    for (int i = 0; i < W; ++i) {
        if (i == wi) k.w[i] = (k.w[i] & ~mhi) | vhi;
        if (i == wi + 1) k.w[i] = (k.w[i] & ~mlo) | vlo;
    }
}

template <int W>
__device__ __forceinline__ uint32_t exciton_site(const ModelDev& m, const Key<W>& k) {
    return m.b0 == 0 ? 0u : (k.w[0] >> (32 - m.b0));
}

template <int W>
__device__ __forceinline__ uint32_t phonon_occ(const ModelDev& m, const Key<W>& k, int j) {
    return get_bits<W>(k, m.b0 + j * m.bp, m.bp);
}

/// Shard owner of a key: hash of its PHONON part (exciton register masked to zero) mod P.  Hop neighbours
/// keep the phonon configuration, so they live on the same rank; only ladder neighbours travel
/// (halo 0.5-0.9 columns per row instead of 1.8-2.2 with a whole-key hash).
template <int W>
__device__ __forceinline__ uint32_t owner_of(const ModelDev& m, const Key<W>& k, uint32_t P) {
    Key<W> z = k;
    if (m.b0 > 0) z.w[0] = (m.b0 >= 32) ? 0u : (z.w[0] & (0xffffffffu >> m.b0));
    return uint32_t(key_hash_words<W>(z.w) % P);
}

/// Diagonal element: eps[e] first, then omega[j]*n_j for ascending j, separate multiply and add
/// (apply_terms accumulation order, lattice_models.hpp:228-235 over the term order of :160-171).
/// Registers with n_j == 0 contribute +0.0 and are skipped; whole zero words are skipped at once.
template <int W>
__device__ __forceinline__ double diagonal_element(const ModelDev& m, const Key<W>& k, uint32_t e) {
    if (m.diag_uniform) {
        uint32_t total = 0;
        for (int b = 0; b < m.bp; ++b) {
            uint32_t cnt = 0;
#pragma unroll
            for (int i = 0; i < W; ++i) cnt += __popc(k.w[i] & __ldg(m.diag_masks + b * W + i));
            total += cnt << b;
        }
        return __dmul_rn(m.omega_u, double(total));  // exact: integers below 2^53
    }
    double diag = 0.0;
    const double ee = __ldg(m.eps + e);
    if (ee != 0.0) diag = __dadd_rn(diag, ee);
    if (m.nph > 0 && m.bp > 0) {
        const uint64_t fmask = (m.bp >= 32) ? 0xffffffffull : ((1ull << m.bp) - 1);
        // word by word (compile-time word index, so the key stays in registers); registers are visited in
        // ascending j because register j starts at bit b0 + j*bp
#pragma unroll
        for (int wi = 0; wi < W; ++wi) {
            const uint32_t cur = k.w[wi];
            const uint32_t nxt = (wi + 1 < W) ? k.w[wi + 1] : 0u;
            if ((cur | nxt) == 0u) continue;  // every register starting in this word is empty
            const uint64_t win = (uint64_t(cur) << 32) | nxt;
            const int j1 = m.wfirst[wi + 1];
            for (int j = m.wfirst[wi]; j < j1; ++j) {
                const int sh = 64 - (m.b0 + j * m.bp - 32 * wi) - m.bp;
                const uint32_t n = uint32_t((win >> sh) & fmask);
                // omega[j] * double(n) from the table; a zero product (omega[j] == 0: the term does not exist,
                // lattice_models.hpp:169) adds +0.0, which leaves diag unchanged bit for bit
                if (n != 0) diag = __dadd_rn(diag, __ldg(m.omega_n + (size_t(j) << m.bp) + n));
            }
        }
    }
    return diag;
}

constexpr int MOVE_LOWER = MAX_NB;      // stable move ids: 0..MAX_NB-1 = hop to the d-th partner of the site
constexpr int MOVE_RAISE = MAX_NB + 1;
constexpr int MOVE_DIAG = MAX_NB + 2;
constexpr int N_MOVES = MAX_NB + 2;     // off-diagonal moves

/// Neighbour generator in CANONICAL (ascending key) order:
///   hops to partners t < e (ascending t) | lower n_e | diagonal | raise n_e | hops to t > e (ascending t)
/// A hop rewrites the most significant field, so t < e sorts before every key with site0 = e; the
/// ladder moves keep site0 and change one later field.  F is called as f(move, key', amp, is_diag) with
/// the stable move id above.  Every move is strictly order-preserving on keys that share the exciton
/// site (it adds a fixed multi-word constant), which the cursor searches below rely on.
/// Amplitudes follow lattice_models.hpp:236-248: g*sqrt(double(n+1)) (dropped at the cutoff
/// n+1 == d_pho), g*sqrt(double(n)), bond J; sqrt is the correctly rounded IEEE one.
template <int W, class F>
__device__ __forceinline__ void for_each_neighbor(const ModelDev& m, const Key<W>& k, bool with_diag, F&& f) {
    const uint32_t e = exciton_site<W>(m, k);
    const int* nbs = m.nb_site + size_t(e) * MAX_NB;
    const double* nba = m.nb_amp + size_t(e) * MAX_NB;
    int d = 0;
    for (; d < MAX_NB; ++d) {
        const int t = __ldg(nbs + d);
        if (t < 0 || uint32_t(t) > e) break;
        Key<W> kk = k;
        set_bits<W>(kk, 0, m.b0, uint32_t(t));
        f(d, kk, __ldg(nba + d), false);
    }
    uint32_t n = 0;
    double ge = 0.0;
    if (m.nph > 0) {
        n = phonon_occ<W>(m, k, int(e));
        ge = __ldg(m.g + e);
    }
    if (ge != 0.0 && n >= 1) {
        Key<W> kk = k;
        set_bits<W>(kk, m.b0 + int(e) * m.bp, m.bp, n - 1);
        f(MOVE_LOWER, kk, __dmul_rn(ge, __dsqrt_rn(double(n))), false);
    }
    if (with_diag) {
        const double diag = diagonal_element<W>(m, k, e);
        if (diag != 0.0) f(MOVE_DIAG, k, diag, true);
    }
    if (ge != 0.0 && n + 1 < m.d_pho) {
        Key<W> kk = k;
        set_bits<W>(kk, m.b0 + int(e) * m.bp, m.bp, n + 1);
        f(MOVE_RAISE, kk, __dmul_rn(ge, __dsqrt_rn(double(n + 1))), false);
    }
    for (; d < MAX_NB; ++d) {
        const int t = __ldg(nbs + d);
        if (t < 0) break;
        Key<W> kk = k;
        set_bits<W>(kk, 0, m.b0, uint32_t(t));
        f(d, kk, __ldg(nba + d), false);
    }
}

/// Forward search from a cursor: the answer (lower bound of k) is known to be >= start.  Gallops
/// 1, 2, 4, ... rows ahead, then bisects.  When a thread walks consecutive sorted rows, the targets of
/// one move are increasing, so the next answer is usually within a few rows of the previous one: a
/// handful of cache-local probes instead of log2(n) scattered ones (a per-thread merge join).
template <int W>
__device__ __forceinline__ bool gallop_find(const uint32_t* __restrict__ table, uint32_t n, uint32_t start,
                                            const Key<W>& k, uint32_t& pos) {
    uint32_t lo = start, hi = start, step = 1;
    while (hi < n) {
        const int c = row_cmp<W>(table + size_t(hi) * W, k);
        if (c == 0) {
            pos = hi;
            return true;
        }
        if (c > 0) break;
        lo = hi + 1;
        hi = (n - hi > step) ? hi + step : n;
        step <<= 1;
    }
    return find_row_in<W>(table, lo, hi < n ? hi : n, k, pos);
}

/// Per-thread cursors, one per move; CUR_NONE = no previous answer (do a full binary search).
constexpr uint32_t CUR_NONE = 0xffffffffu;
struct MoveCursors {
    uint32_t c[N_MOVES];
    uint32_t site;
    __device__ __forceinline__ void reset(uint32_t e) {
#pragma unroll
        for (int i = 0; i < N_MOVES; ++i) c[i] = CUR_NONE;
        site = e;
    }
};

/// Look-up of the `move` neighbour of a row that a thread visits in ascending order.
template <int W>
__device__ __forceinline__ bool cursor_find(const uint32_t* __restrict__ table, uint32_t n, MoveCursors& cur, int move,
                                            const Key<W>& k, uint32_t& pos) {
    uint32_t start = 0;
#pragma unroll
    for (int i = 0; i < N_MOVES; ++i)
        if (i == move) start = cur.c[i];
    const bool found = (start == CUR_NONE) ? find_row<W>(table, n, k, pos) : gallop_find<W>(table, n, start, k, pos);
    const uint32_t next = found ? pos + 1 : pos;
#pragma unroll
    for (int i = 0; i < N_MOVES; ++i)
        if (i == move) cur.c[i] = next;
    return found;
}

}  // namespace pb
