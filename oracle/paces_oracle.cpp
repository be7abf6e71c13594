// paces_oracle.cpp -- CPU restatement of the paces adapt-evolve-truncate step.
//
// TEST INFRASTRUCTURE ONLY (see oracle_abi.h): the checker for the CUDA path,
// never a fallback for it.  Written from the behaviour of the reference, not
// from its text; each function cites the reference lines it follows
// (paths relative to /root/reference/proj/include/paces/).
//
// PARITY PINNED: tests/test_oracle_port.py checks every entry point of this
// file bit-for-bit against oracle/_ref/libpaces_ref.so (the unmodified
// reference headers) where that library is present, and against the golden
// fixtures under tests/golden/ (generated from the reference by
// tests/golden/make_golden.py) everywhere.
//
// Where this restatement deliberately takes a different route to the same
// bits (all verified in the tests):
//   * neighbour generation is closed-form per key (exciton register -> its
//     incident bonds and its own ladder) instead of a scan over the whole
//     term list, emitting in the same order as the term list would;
//   * H_eff is assembled row by row (row i = in-table neighbours of key i,
//     sorted by column) instead of transcript -> Hermitian closure -> global
//     sort -> duplicate collapse;
//   * all complex arithmetic is written out on (re, im) doubles in the exact
//     operation order libstdc++'s std::complex produces without FMA.
//
// Build: oracle/Makefile (g++ -std=c++20 -O3 -fopenmp, no -march, no
// -ffast-math; -ffp-contract=off is implied on baseline x86-64 but is passed
// anyway by the pragma below).

#pragma GCC optimize("fp-contract=off")

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "oracle_abi.h"

namespace {

using u32 = std::uint32_t;
using u64 = std::uint64_t;
using i64 = std::int64_t;

struct Fail : std::runtime_error {
    using std::runtime_error::runtime_error;
};

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// common.hpp:30-49 -- PACES_MAX_MEMORY_BYTES cap, re-read on every call.
void need_memory(u64 bytes, const char* what) {
    const char* env = std::getenv("PACES_MAX_MEMORY_BYTES");
    if (!env || !*env) return;
    char* end = nullptr;
    const unsigned long long cap = std::strtoull(env, &end, 10);
    if (end == env) throw Fail(std::string("PACES_MAX_MEMORY_BYTES is not a number: ") + env);
    if (cap != 0 && bytes > cap)
        throw Fail(std::string("memory cap exceeded: ") + what + " needs " + std::to_string(bytes) +
                   " bytes, PACES_MAX_MEMORY_BYTES=" + std::to_string(cap));
}

// ---------------------------------------------------------------------------
// key layout (basis_codec.hpp:39-77): site i takes bit_width(d_i - 1) bits,
// packed MSB-first from the top of word 0; straddling payloads put their high
// bits in the earlier word (:90-128).
// ---------------------------------------------------------------------------
struct Layout {
    std::vector<u32> dims, bits, offs;
    u32 total_bits = 0, words = 1;

    void build(std::vector<u32> d) {
        if (d.empty()) throw Fail("site layout needs at least one site");
        dims = std::move(d);
        u32 off = 0;
        for (std::size_t i = 0; i < dims.size(); ++i) {
            if (dims[i] < 1) throw Fail("site dimension must be >= 1 at site " + std::to_string(i));
            u32 b = 0;
            while (b < 32 && (u64(1) << b) < dims[i]) ++b;  // ceil(log2 d), 0 for d == 1
            bits.push_back(b);
            offs.push_back(off);
            off += b;
        }
        total_bits = off;
        words = std::max<u32>(1, (off + 31) / 32);
    }
    std::size_t sites() const { return dims.size(); }

    u32 get(const u32* row, std::size_t s) const {
        const u32 b = bits[s];
        if (b == 0) return 0;
        // read the b-bit field starting at absolute bit offs[s] (bit 0 = MSB of word 0)
        const u32 w = offs[s] >> 5, sh = offs[s] & 31;
        u64 window = u64(row[w]) << 32;
        if (sh + b > 32) window |= row[w + 1];
        return u32((window << sh) >> (64 - b));
    }
    void set(u32* row, std::size_t s, u32 v) const {
        const u32 b = bits[s];
        if (b == 0) return;
        const u32 w = offs[s] >> 5, sh = offs[s] & 31;
        const bool two = sh + b > 32;
        u64 window = u64(row[w]) << 32;
        if (two) window |= row[w + 1];
        const u64 mask = ((u64(1) << b) - 1) << (64 - sh - b);
        window = (window & ~mask) | (u64(v) << (64 - sh - b));
        row[w] = u32(window >> 32);
        if (two) row[w + 1] = u32(window);
    }
};

inline bool key_less(const u32* a, const u32* b, u32 w) {
    for (u32 i = 0; i < w; ++i)
        if (a[i] != b[i]) return a[i] < b[i];
    return false;
}
inline bool key_eq(const u32* a, const u32* b, u32 w) { return std::memcmp(a, b, 4 * w) == 0; }

// lower-bound search in a sorted flat table; returns rows if absent (basis_codec.hpp:334-348)
std::size_t locate(const u32* table, std::size_t rows, u32 w, const u32* key) {
    std::size_t lo = 0, hi = rows;
    while (lo < hi) {
        const std::size_t mid = lo + (hi - lo) / 2;
        if (key_less(table + mid * w, key, w))
            lo = mid + 1;
        else
            hi = mid;
    }
    return (lo < rows && key_eq(table + lo * w, key, w)) ? lo : rows;
}

bool strictly_sorted(const u32* t, std::size_t rows, u32 w) {
    for (std::size_t i = 1; i < rows; ++i)
        if (!key_less(t + (i - 1) * w, t + i * w, w)) return false;
    return true;
}

// sort + unique on flat rows (basis_codec.hpp:247-270)
void sort_unique(std::vector<u32>& rows, u32 w) {
    const std::size_t n = rows.size() / w;
    if (n <= 1) return;
    std::vector<u32> idx(n);
    std::iota(idx.begin(), idx.end(), 0u);
    const u32* base = rows.data();
    std::sort(idx.begin(), idx.end(),
              [=](u32 a, u32 b) { return key_less(base + std::size_t(a) * w, base + std::size_t(b) * w, w); });
    std::vector<u32> out;
    out.reserve(rows.size());
    for (std::size_t k = 0; k < n; ++k) {
        const u32* r = base + std::size_t(idx[k]) * w;
        if (!out.empty() && key_eq(out.data() + out.size() - w, r, w)) continue;
        out.insert(out.end(), r, r + w);
    }
    rows.swap(out);
}

// ---------------------------------------------------------------------------
// model (lattice_models.hpp:25-66 geometry, :140-189 term order)
// ---------------------------------------------------------------------------
struct Bond {
    u32 a, b;
    double j;
};

struct Model {
    int kind = 1;  // 0 tight binding, 1 holstein
    int ndim = 1;
    u32 ext[3] = {1, 1, 1};
    u32 nsites = 1;
    u32 d_pho = 1;
    std::vector<double> eps, omega, g;  // per site (broadcast applied)
    std::vector<Bond> bonds;            // x-then-y-then-z per site, row-major sites, J == 0 dropped
    std::vector<std::vector<u32>> incident;  // bond ids touching a site, ascending bond id
    Layout lay;
    u32 n_terms = 0;

    u32 site_index(u32 x, u32 y, u32 z) const { return (z * ext[1] + y) * ext[0] + x; }
};

std::vector<double> spread(const double* v, int n, std::size_t want, const char* name) {
    if (n == 0) return std::vector<double>(want, 0.0);
    if (n == 1) return std::vector<double>(want, v[0]);
    if (std::size_t(n) != want)
        throw Fail(std::string(name) + ": expected 1 or " + std::to_string(want) + " values, got " + std::to_string(n));
    return std::vector<double>(v, v + n);
}

// apply_terms, lattice_models.hpp:212-267, for the two exciton model kinds.
// Emission order equals the reference's term-list order: hops in bond order,
// raise, lower, and the diagonal last (only when nonzero).  Returns count.
struct Emit {
    std::vector<u32> keys;
    std::vector<double> amps;
    void clear() {
        keys.clear();
        amps.clear();
    }
};

void check_key(const Model& m, const u32* key) {  // unpack_state validation, basis_codec.hpp:155-165
    for (std::size_t s = 0; s < m.lay.sites(); ++s) {
        const u32 v = m.lay.get(key, s);
        if (v >= m.lay.dims[s])
            throw Fail("unpack: corrupt row, decoded value " + std::to_string(v) + " >= dim " +
                       std::to_string(m.lay.dims[s]) + " at site " + std::to_string(s));
    }
}

void neighbours(const Model& m, const u32* key, Emit& out) {
    const u32 w = m.lay.words;
    check_key(m, key);
    const u32 e = m.lay.get(key, 0);
    double diag = 0.0;
    if (m.eps[e] != 0.0) diag += m.eps[e];  // only site e's diagonal_exciton term fires (:229-231)
    auto push = [&](std::size_t slot, u32 value, double amp) {
        const std::size_t base = out.keys.size();
        out.keys.insert(out.keys.end(), key, key + w);
        m.lay.set(out.keys.data() + base, slot, value);
        out.amps.push_back(amp);
    };
    for (u32 b : m.incident[e]) {  // hop terms precede the phonon terms in the list (:162-171)
        const Bond& bd = m.bonds[b];
        push(0, bd.a == e ? bd.b : bd.a, bd.j);
    }
    if (m.kind == 1) {
        for (u32 j = 0; j < m.nsites; ++j) {
            const u32 nj = m.lay.get(key, 1 + j);
            if (m.omega[j] != 0.0) diag += m.omega[j] * double(nj);  // :232-234
            if (j == e && m.g[j] != 0.0) {                           // :235-244
                if (nj + 1 < m.d_pho) push(1 + j, nj + 1, m.g[j] * std::sqrt(double(nj + 1)));
                if (nj >= 1) push(1 + j, nj - 1, m.g[j] * std::sqrt(double(nj)));
            }
        }
    }
    if (diag != 0.0) {  // :263-266
        out.keys.insert(out.keys.end(), key, key + w);
        out.amps.push_back(diag);
    }
}

// ---------------------------------------------------------------------------
// CSR + space
// ---------------------------------------------------------------------------
struct Csr {
    i64 n = 0;
    std::vector<i64> row_ptr;
    std::vector<std::int32_t> col;
    std::vector<double> val;
};

struct Space {
    std::vector<u32> table;  // sorted, flat
    std::size_t rows = 0;
    Csr h;
    std::size_t q_nom = 0;
};

// grow_subspace (subspace.hpp:195-249): breadth-first ball of order m around
// the seeds; H_eff = restriction of H to the ball.  Row-wise assembly: because
// every key's terms are applied exactly once and the last frontier is filtered
// to in-table targets, row i holds exactly the in-table neighbours of key i;
// the reference's (r, c) sort makes columns ascending within a row.
Space grow(const Model& m, const u32* seeds, std::size_t nseeds, int order) {
    const u32 w = m.lay.words;
    if (nseeds == 0) throw Fail("grow_subspace: empty seed set");
    if (!strictly_sorted(seeds, nseeds, w)) throw Fail("grow_subspace: seed keys must be sorted");
    if (order < 0) throw Fail("grow_subspace: neighbor order must be >= 0");

    std::vector<u32> table(seeds, seeds + nseeds * w), frontier = table;
    u64 emitted = 0;
    for (int k = 0; k < order && !frontier.empty(); ++k) {
        const std::size_t nf = frontier.size() / w;
        std::vector<u32> cand;
        {
            const std::size_t chunk = 4096, nchunks = (nf + chunk - 1) / chunk;
            std::vector<std::vector<u32>> parts(nchunks);
#pragma omp parallel for schedule(dynamic)
            for (std::size_t c = 0; c < nchunks; ++c) {
                Emit e;
                for (std::size_t i = c * chunk; i < std::min(nf, (c + 1) * chunk); ++i) {
                    e.clear();
                    neighbours(m, frontier.data() + i * w, e);
                    parts[c].insert(parts[c].end(), e.keys.begin(), e.keys.end());
                }
            }
            for (auto& p : parts) cand.insert(cand.end(), p.begin(), p.end());
        }
        emitted += cand.size() / w;
        sort_unique(cand, w);
        // frontier = cand \ table ; table = table U frontier (basis_codec.hpp:273-321)
        std::vector<u32> fresh, merged;
        merged.reserve(table.size() + cand.size());
        std::size_t i = 0, j = 0;
        const std::size_t na = cand.size() / w, nb = table.size() / w;
        while (i < na || j < nb) {
            const u32* a = i < na ? cand.data() + i * w : nullptr;
            const u32* b = j < nb ? table.data() + j * w : nullptr;
            if (b == nullptr || (a != nullptr && key_less(a, b, w))) {
                fresh.insert(fresh.end(), a, a + w);
                merged.insert(merged.end(), a, a + w);
                ++i;
            } else if (a == nullptr || key_less(b, a, w)) {
                merged.insert(merged.end(), b, b + w);
                ++j;
            } else {
                merged.insert(merged.end(), b, b + w);
                ++i;
                ++j;
            }
        }
        frontier.swap(fresh);
        table.swap(merged);
        // transcript footprint the reference checks (subspace.hpp:215-217)
        need_memory((table.size() + emitted * w * 2) * sizeof(u32) + emitted * sizeof(double), "subspace growth");
    }

    Space sp;
    sp.rows = table.size() / w;
    sp.q_nom = nseeds;
    sp.table = std::move(table);

    const std::size_t n = sp.rows;
    std::vector<u32> len(n, 0);
    struct Ent {
        std::int32_t c;
        double v;
    };
    std::vector<std::vector<Ent>> rows(n);
#pragma omp parallel
    {
        Emit e;
#pragma omp for schedule(dynamic, 1024)
        for (std::size_t i = 0; i < n; ++i) {
            e.clear();
            neighbours(m, sp.table.data() + i * w, e);
            auto& r = rows[i];
            for (std::size_t k = 0; k < e.amps.size(); ++k) {
                const std::size_t c = locate(sp.table.data(), n, w, e.keys.data() + k * w);
                if (c < n) r.push_back({std::int32_t(c), e.amps[k]});
            }
            std::sort(r.begin(), r.end(), [](const Ent& a, const Ent& b) { return a.c < b.c; });
        }
    }
    sp.h.n = i64(n);
    sp.h.row_ptr.assign(n + 1, 0);
    for (std::size_t i = 0; i < n; ++i) sp.h.row_ptr[i + 1] = sp.h.row_ptr[i] + i64(rows[i].size());
    need_memory(u64(sp.h.row_ptr[n]) * 2 * 16, "matrix assembly buffer");  // subspace.hpp:152
    sp.h.col.resize(sp.h.row_ptr[n]);
    sp.h.val.resize(sp.h.row_ptr[n]);
    for (std::size_t i = 0; i < n; ++i) {
        i64 p = sp.h.row_ptr[i];
        for (const Ent& en : rows[i]) {
            sp.h.col[p] = en.c;
            sp.h.val[p] = en.v;
            ++p;
        }
    }
    return sp;
}

// ---------------------------------------------------------------------------
// sparse kernels on split (re, im) arithmetic
// ---------------------------------------------------------------------------
// csr_matvec, subspace.hpp:35-43: acc starts at 0, entries in stored order,
// real x complex = two real products.
void matvec(const Csr& a, const double* x, double* y) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < a.n; ++i) {
        double ar = 0.0, ai = 0.0;
        for (i64 k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
            const std::size_t c = std::size_t(a.col[k]);
            ar = ar + a.val[k] * x[2 * c];
            ai = ai + a.val[k] * x[2 * c + 1];
        }
        y[2 * i] = ar;
        y[2 * i + 1] = ai;
    }
}

// csr_expectation, subspace.hpp:46-55: serial; Re(conj(x_i) * row_i) = xr*rr - (-xi)*ri.
double expectation(const Csr& a, const double* x) {
    double acc = 0.0;
    for (i64 i = 0; i < a.n; ++i) {
        double rr = 0.0, ri = 0.0;
        for (i64 k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
            const std::size_t c = std::size_t(a.col[k]);
            rr = rr + a.val[k] * x[2 * c];
            ri = ri + a.val[k] * x[2 * c + 1];
        }
        acc += x[2 * i] * rr + x[2 * i + 1] * ri;
    }
    return acc;
}

double norm2_serial(const double* c, std::size_t n) {  // subspace.hpp:91-95, propagator.hpp:39-43
    double acc = 0.0;
    for (std::size_t i = 0; i < n; ++i) acc += c[2 * i] * c[2 * i] + c[2 * i + 1] * c[2 * i + 1];
    return acc;
}

struct ExpmvOut {
    int order = 0;
    double last = 0;
};

// expmv, propagator.hpp:52-92.  scale = (0, -dt_sub/n); scale*h = (0*hr - b*hi, 0*hi + b*hr).
ExpmvOut taylor(const Csr& a, double* c, double dt, double rtol, int max_order, int substeps) {
    if (!(dt > 0)) throw Fail("propagator: dt must be > 0");
    if (!(rtol > 0) || !(rtol < 1)) throw Fail("propagator: rtol must be in (0, 1)");
    if (max_order < 1) throw Fail("propagator: max_order must be >= 1");
    if (substeps < 1) throw Fail("propagator: substeps must be >= 1");
    const std::size_t n = std::size_t(a.n);
    for (std::size_t i = 0; i < 2 * n; ++i)
        if (!std::isfinite(c[i])) throw Fail("expmv: non-finite input coefficient");
    const double dt_sub = dt / substeps;
    std::vector<double> term(2 * n), h(2 * n);
    ExpmvOut res;
    for (int s = 0; s < substeps; ++s) {
        std::copy(c, c + 2 * n, term.begin());
        int streak = 0;
        bool done = false;
        for (int k = 1; k <= max_order; ++k) {
            matvec(a, term.data(), h.data());
            const double b = -dt_sub / double(k);
#pragma omp parallel for schedule(static)
            for (std::size_t i = 0; i < n; ++i) {
                const double hr = h[2 * i], hi = h[2 * i + 1];
                const double tr = 0.0 * hr - b * hi;
                const double ti = 0.0 * hi + b * hr;
                term[2 * i] = tr;
                term[2 * i + 1] = ti;
                c[2 * i] = c[2 * i] + tr;
                c[2 * i + 1] = c[2 * i + 1] + ti;
            }
            const double tn = std::sqrt(norm2_serial(term.data(), n));
            const double rn = std::sqrt(norm2_serial(c, n));
            res.order = std::max(res.order, k);
            res.last = tn;
            streak = (tn <= rtol * rn) ? streak + 1 : 0;
            if (streak >= 2) {
                done = true;
                break;
            }
        }
        if (!done)
            throw Fail("expmv: Taylor series did not converge within max_order=" + std::to_string(max_order) +
                       "; reduce dt or increase substeps");
    }
    return res;
}

// ---------------------------------------------------------------------------
// truncate-select (engine.hpp:107-156) and remap (subspace.hpp:281-305)
// ---------------------------------------------------------------------------
std::vector<std::size_t> select_rows(const double* c, std::size_t rows, std::size_t q_nom, u64 seed) {
    if (q_nom < 1) throw Fail("truncate_select: q_nom must be >= 1");
    std::vector<std::size_t> support;
    for (std::size_t i = 0; i < rows; ++i)
        if (c[2 * i] * c[2 * i] + c[2 * i + 1] * c[2 * i + 1] > 0) support.push_back(i);
    if (support.empty()) throw Fail("truncate_select: state has no support");
    if (support.size() <= q_nom) return support;

    std::vector<double> wts(support.size());
    for (std::size_t k = 0; k < support.size(); ++k) {
        const std::size_t i = support[k];
        wts[k] = c[2 * i] * c[2 * i] + c[2 * i + 1] * c[2 * i + 1];
    }
    std::vector<double> tmp = wts;
    std::nth_element(tmp.begin(), tmp.begin() + (q_nom - 1), tmp.end(), std::greater<double>());
    const double cut = tmp[q_nom - 1];
    std::vector<std::size_t> keep, ties;
    for (std::size_t k = 0; k < support.size(); ++k) {
        if (wts[k] > cut)
            keep.push_back(support[k]);
        else if (wts[k] == cut)
            ties.push_back(support[k]);
    }
    const std::size_t need = q_nom - keep.size();
    std::mt19937_64 rng(seed);  // Fisher-Yates from the top, only when a strict subset is needed (:137-141)
    for (std::size_t i = ties.size(); i > 1 && need < ties.size(); --i) {
        const std::size_t j = std::size_t(rng() % i);
        std::swap(ties[i - 1], ties[j]);
    }
    keep.insert(keep.end(), ties.begin(), ties.begin() + need);
    std::sort(keep.begin(), keep.end());
    return keep;
}

double remap(const u32* sw, const double* sc, std::size_t srows, const u32* dw, std::size_t drows, u32 w,
             double* out) {
    if (!strictly_sorted(sw, srows, w)) throw Fail("remap: state table must be sorted");
    std::fill(out, out + 2 * drows, 0.0);
    double lost = 0.0;
    std::size_t j = 0;
    for (std::size_t i = 0; i < srows; ++i) {
        const u32* key = sw + i * w;
        while (j < drows && key_less(dw + j * w, key, w)) ++j;
        if (j < drows && key_eq(dw + j * w, key, w)) {
            out[2 * j] = sc[2 * i];
            out[2 * j + 1] = sc[2 * i + 1];
            ++j;
        } else {
            lost += sc[2 * i] * sc[2 * i] + sc[2 * i + 1] * sc[2 * i + 1];
        }
    }
    return lost;
}

// ---------------------------------------------------------------------------
// observables (observables.hpp:26-112)
// ---------------------------------------------------------------------------
void density(const Model& m, const u32* words, const double* c, std::size_t rows, double* p) {
    std::fill(p, p + m.nsites, 0.0);
    for (std::size_t i = 0; i < rows; ++i) {
        const double wt = c[2 * i] * c[2 * i] + c[2 * i + 1] * c[2 * i + 1];
        if (wt == 0.0) continue;
        p[m.lay.get(words + i * m.lay.words, 0)] += wt;
    }
}

void dipole(const Model& m, const u32* words, const double* c, std::size_t rows, double* amp) {
    if (!strictly_sorted(words, rows, m.lay.words)) throw Fail("find_row requires a sorted table");
    std::vector<u32> key(m.lay.words);
    double ar = 0.0, ai = 0.0;
    for (u32 j = 0; j < m.nsites; ++j) {
        std::fill(key.begin(), key.end(), 0u);
        m.lay.set(key.data(), 0, j);
        const std::size_t idx = locate(words, rows, m.lay.words, key.data());
        if (idx < rows) {
            ar += c[2 * idx];
            ai += c[2 * idx + 1];
        }
    }
    const double s = std::sqrt(double(m.nsites));
    amp[0] = ar / s;
    amp[1] = ai / s;
}

void phonons(const Model& m, const u32* words, const double* c, std::size_t rows, double* out) {
    if (m.kind != 1) throw Fail("phonon numbers: not a Holstein model");
    std::fill(out, out + m.nsites, 0.0);
    for (std::size_t i = 0; i < rows; ++i) {
        const double wt = c[2 * i] * c[2 * i] + c[2 * i + 1] * c[2 * i + 1];
        if (wt == 0.0) continue;
        for (u32 j = 0; j < m.nsites; ++j) out[j] += wt * double(m.lay.get(words + i * m.lay.words, 1 + j));
    }
}

double spread_rmsd(const Model& m, const double* p) {  // observables.hpp:49-70
    double wsum = 0, mean[3] = {0, 0, 0};
    auto coords = [&](u32 idx, u32* c) {
        c[0] = idx % m.ext[0];
        c[1] = (idx / m.ext[0]) % m.ext[1];
        c[2] = idx / (m.ext[0] * m.ext[1]);
    };
    u32 c[3];
    for (u32 i = 0; i < m.nsites; ++i) {
        coords(i, c);
        wsum += p[i];
        for (int a = 0; a < 3; ++a) mean[a] += p[i] * double(c[a]);
    }
    if (wsum <= 0) throw Fail("rmsd: zero-norm state");
    for (int a = 0; a < 3; ++a) mean[a] /= wsum;
    double var = 0;
    for (u32 i = 0; i < m.nsites; ++i) {
        coords(i, c);
        double r2 = 0;
        for (int a = 0; a < 3; ++a) {
            const double dx = double(c[a]) - mean[a];
            r2 += dx * dx;
        }
        var += (p[i] / wsum) * r2;
    }
    return std::sqrt(var);
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
struct po_model {
    Model m;
};
struct po_space {
    Space s;
};
struct po_run {
    const po_model* model = nullptr;
    po_run_cfg cfg{};
    std::vector<u32> words;  // current table (sorted)
    std::vector<double> coeff;
    double t = 0;
    Csr h;
    u64 steps_done = 0;
    po_phase_times times{};
};

extern "C" {

const char* po_last_error(void) { return g_err.c_str(); }
const char* po_impl_name(void) { return "port"; }
void po_set_threads(int n) {
#ifdef _OPENMP
    if (n >= 1) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
int po_get_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
uint64_t po_mix_seed(uint64_t x) {  // splitmix64 finaliser, common.hpp:76-81
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

int po_model_create(int kind, int ndim, const uint32_t* extents, const double* eps, int n_eps, const double* hop,
                    int n_hop, const double* omega, int n_omega, const double* g, int n_g, uint32_t d_pho,
                    po_model** out) {
    return guarded([&] {
        if (kind != 0 && kind != 1) throw Fail("model kind must be tight_binding (0) or holstein (1)");
        if (ndim < 1 || ndim > 3) throw Fail("lattice must have 1 to 3 extents");
        auto pm = std::make_unique<po_model>();
        Model& m = pm->m;
        m.kind = kind;
        m.ndim = ndim;
        for (int i = 0; i < ndim; ++i) {
            if (extents[i] == 0) throw Fail("lattice extent must be positive");
            m.ext[i] = extents[i];
        }
        m.nsites = m.ext[0] * m.ext[1] * m.ext[2];
        // bonds: x-then-y-then-z per site, sites row-major (lattice_models.hpp:54-65)
        std::vector<std::pair<u32, u32>> all;
        for (u32 z = 0; z < m.ext[2]; ++z)
            for (u32 y = 0; y < m.ext[1]; ++y)
                for (u32 x = 0; x < m.ext[0]; ++x) {
                    const u32 here = m.site_index(x, y, z);
                    if (x + 1 < m.ext[0]) all.emplace_back(here, m.site_index(x + 1, y, z));
                    if (y + 1 < m.ext[1]) all.emplace_back(here, m.site_index(x, y + 1, z));
                    if (z + 1 < m.ext[2]) all.emplace_back(here, m.site_index(x, y, z + 1));
                }
        m.eps = spread(eps, n_eps, m.nsites, "eps");
        const auto hops = spread(hop, n_hop, all.size(), "J");
        std::vector<u32> dims{m.nsites};
        if (kind == 1) {
            if (d_pho < 1) throw Fail("d_pho must be >= 1");
            m.d_pho = d_pho;
            dims.insert(dims.end(), m.nsites, d_pho);
            m.omega = spread(omega, n_omega, m.nsites, "omega0");
            m.g = spread(g, n_g, m.nsites, "g");
        } else {
            m.omega.assign(m.nsites, 0.0);
            m.g.assign(m.nsites, 0.0);
        }
        m.lay.build(dims);
        m.incident.assign(m.nsites, {});
        for (std::size_t b = 0; b < all.size(); ++b) {
            if (hops[b] == 0.0) continue;  // zero parameters dropped at build time (:163)
            const u32 id = u32(m.bonds.size());
            m.bonds.push_back({all[b].first, all[b].second, hops[b]});
            m.incident[all[b].first].push_back(id);
            m.incident[all[b].second].push_back(id);
        }
        m.n_terms = u32(m.bonds.size());
        for (u32 j = 0; j < m.nsites; ++j) {
            m.n_terms += m.eps[j] != 0.0;
            if (kind == 1) m.n_terms += (m.omega[j] != 0.0) + (m.g[j] != 0.0);
        }
        *out = pm.release();
    });
}
void po_model_destroy(po_model* m) { delete m; }

int po_model_info(const po_model* m, uint32_t* layout_sites, uint32_t* words_per_row, uint32_t* lattice_sites,
                  uint32_t* n_terms, uint32_t* total_bits) {
    if (layout_sites) *layout_sites = u32(m->m.lay.sites());
    if (words_per_row) *words_per_row = m->m.lay.words;
    if (lattice_sites) *lattice_sites = m->m.nsites;
    if (n_terms) *n_terms = m->m.n_terms;
    if (total_bits) *total_bits = m->m.lay.total_bits;
    return 0;
}
int po_model_dims(const po_model* m, uint32_t* dims) {
    std::copy(m->m.lay.dims.begin(), m->m.lay.dims.end(), dims);
    return 0;
}

int po_pack(const po_model* m, const uint32_t* occ, uint32_t* words) {  // basis_codec.hpp:131-145
    return guarded([&] {
        const Layout& l = m->m.lay;
        std::fill(words, words + l.words, 0u);
        for (std::size_t s = 0; s < l.sites(); ++s) {
            if (occ[s] >= l.dims[s])
                throw Fail("pack: occupation " + std::to_string(occ[s]) + " out of range at site " + std::to_string(s) +
                           " (dim " + std::to_string(l.dims[s]) + ")");
            l.set(words, s, occ[s]);
        }
    });
}
int po_unpack(const po_model* m, const uint32_t* words, uint32_t* occ) {
    return guarded([&] {
        check_key(m->m, words);
        for (std::size_t s = 0; s < m->m.lay.sites(); ++s) occ[s] = m->m.lay.get(words, s);
    });
}

int po_apply_terms(const po_model* m, const uint32_t* key, uint32_t* out_keys, double* out_amps, int cap, int* count) {
    return guarded([&] {
        Emit e;
        neighbours(m->m, key, e);
        if (int(e.amps.size()) > cap) throw Fail("po_apply_terms: output capacity too small");
        std::copy(e.keys.begin(), e.keys.end(), out_keys);
        std::copy(e.amps.begin(), e.amps.end(), out_amps);
        *count = int(e.amps.size());
    });
}

int po_grow(const po_model* m, const uint32_t* seeds, uint64_t rows, int order, po_space** out) {
    return guarded([&] {
        auto s = std::make_unique<po_space>();
        s->s = grow(m->m, seeds, rows, order);
        *out = s.release();
    });
}
int po_space_info(const po_space* s, uint64_t* q_true, uint64_t* nnz, uint64_t* q_nom) {
    if (q_true) *q_true = s->s.rows;
    if (nnz) *nnz = s->s.h.val.size();
    if (q_nom) *q_nom = s->s.q_nom;
    return 0;
}
int po_space_get(const po_space* s, uint32_t* words, int64_t* row_ptr, int32_t* col, double* val) {
    if (words) std::copy(s->s.table.begin(), s->s.table.end(), words);
    if (row_ptr) std::copy(s->s.h.row_ptr.begin(), s->s.h.row_ptr.end(), row_ptr);
    if (col) std::copy(s->s.h.col.begin(), s->s.h.col.end(), col);
    if (val) std::copy(s->s.h.val.begin(), s->s.h.val.end(), val);
    return 0;
}
void po_space_destroy(po_space* s) { delete s; }

int po_truncate_select(const po_model* m, const uint32_t* words, const double* coeff, uint64_t rows, uint64_t q_nom,
                       uint64_t seed, uint32_t* out_words, uint64_t* kept) {
    return guarded([&] {
        const u32 w = m->m.lay.words;
        if (!strictly_sorted(words, rows, w)) throw Fail("truncate_select: state table must be sorted");
        const auto keep = select_rows(coeff, rows, q_nom, seed);
        for (std::size_t k = 0; k < keep.size(); ++k)
            std::copy(words + keep[k] * w, words + (keep[k] + 1) * w, out_words + k * w);
        *kept = keep.size();
    });
}

int po_remap(const po_model* m, const uint32_t* src_words, const double* src_coeff, uint64_t src_rows,
             const uint32_t* dst_words, uint64_t dst_rows, double* out_coeff, double* discarded) {
    return guarded(
        [&] { *discarded = remap(src_words, src_coeff, src_rows, dst_words, dst_rows, m->m.lay.words, out_coeff); });
}

static Csr wrap_csr(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val) {
    Csr a;
    a.n = n;
    a.row_ptr.assign(row_ptr, row_ptr + n + 1);
    a.col.assign(col, col + row_ptr[n]);
    a.val.assign(val, val + row_ptr[n]);
    return a;
}

int po_csr_matvec(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val, const double* x,
                  double* y) {
    return guarded([&] { matvec(wrap_csr(n, row_ptr, col, val), x, y); });
}
int po_csr_expectation(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val, const double* x,
                       double* out) {
    return guarded([&] { *out = expectation(wrap_csr(n, row_ptr, col, val), x); });
}
int po_expmv(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val, double* c, double dt,
             double rtol, int max_order, int substeps, int* order_used, double* last_term_norm) {
    return guarded([&] {
        const ExpmvOut r = taylor(wrap_csr(n, row_ptr, col, val), c, dt, rtol, max_order, substeps);
        if (order_used) *order_used = r.order;
        if (last_term_norm) *last_term_norm = r.last;
    });
}

int po_state_norm(const double* coeff, uint64_t rows, double* out) {
    *out = std::sqrt(norm2_serial(coeff, rows));
    return 0;
}
int po_exciton_density(const po_model* m, const uint32_t* words, const double* coeff, uint64_t rows, double* p) {
    return guarded([&] { density(m->m, words, coeff, rows, p); });
}
int po_dipole_amplitude(const po_model* m, const uint32_t* words, const double* coeff, uint64_t rows, double* amp) {
    return guarded([&] { dipole(m->m, words, coeff, rows, amp); });
}
int po_phonon_numbers(const po_model* m, const uint32_t* words, const double* coeff, uint64_t rows, double* n_out) {
    return guarded([&] { phonons(m->m, words, coeff, rows, n_out); });
}

// weight_histogram, observables.hpp:123-176: descending |c|^2 curve; counts reaching 50/90/99/99.99 % of the total
// (serial running sum, tolerance 1e-15*total); least-squares slope of log w vs log rank over the last nine
// deciles; curve sampled at ranks k*(n-1)/(npts-1).
int po_weight_histogram(const double* coeff, uint64_t rows, uint64_t bins, po_weight_hist* out, uint64_t* rank,
                        double* weight, uint64_t cap, uint64_t* npts_out) {
    return guarded([&] {
        std::vector<double> w;
        w.reserve(rows);
        for (uint64_t i = 0; i < rows; ++i) {
            const double v = coeff[2 * i] * coeff[2 * i] + coeff[2 * i + 1] * coeff[2 * i + 1];  // std::norm
            if (v > 0) w.push_back(v);
        }
        if (w.empty()) throw Fail("weight histogram: empty state");
        std::sort(w.begin(), w.end(), std::greater<double>());
        const size_t n = w.size();
        double total = 0.0;
        for (double v : w) total += v;
        uint64_t marks[4] = {n, n, n, n};
        const double frac[4] = {0.50, 0.90, 0.99, 0.9999};
        double running = 0;
        size_t done = 0;
        for (size_t i = 0; i < n && done < 4; ++i) {
            running += w[i];
            while (done < 4 && running >= frac[done] * total - 1e-15 * total) marks[done++] = i + 1;
        }
        out->support = n;
        out->q50 = marks[0];
        out->q90 = marks[1];
        out->q99 = marks[2];
        out->q9999 = marks[3];
        out->tail_exponent = 0;
        const size_t lo = n / 10;
        if (n - lo >= 2) {
            double sx = 0, sy = 0, sxx = 0, sxy = 0;
            size_t cnt = 0;
            for (size_t i = lo; i < n; ++i) {
                const double x = std::log(double(i + 1)), y = std::log(w[i]);
                sx += x;
                sy += y;
                sxx += x * x;
                sxy += x * y;
                ++cnt;
            }
            const double denom = cnt * sxx - sx * sx;
            out->tail_exponent = denom != 0 ? (cnt * sxy - sx * sy) / denom : 0.0;
        }
        const size_t npts = (bins == 0 || n <= bins) ? n : size_t(bins);
        *npts_out = npts;
        for (size_t k = 0; k < npts && k < cap; ++k) {
            const size_t i = npts == 1 ? 0 : k * (n - 1) / (npts - 1);
            rank[k] = i + 1;
            weight[k] = w[i];
        }
    });
}

// initialize(), engine.hpp:165-251
int po_run_begin(const po_model* pm, const po_run_cfg* c, po_run** out) {
    return guarded([&] {
        const Model& m = pm->m;
        // RunConfig::validate, engine.hpp:48-58
        if (c->m < 0 || c->m_init < c->m) throw Fail("run: need m_init >= m >= 0");
        if (c->q_nom < 1) throw Fail("run: q_nom must be >= 1");
        if (c->t_max < 0) throw Fail("run: t_max must be >= 0");
        if (c->cadence < 1) throw Fail("run: cadence must be >= 1");
        if (!(c->dt > 0)) throw Fail("propagator: dt must be > 0");
        if (!(c->rtol > 0) || !(c->rtol < 1)) throw Fail("propagator: rtol must be in (0, 1)");
        if (c->max_order < 1) throw Fail("propagator: max_order must be >= 1");
        if (c->substeps < 1) throw Fail("propagator: substeps must be >= 1");

        const u32 w = m.lay.words;
        const std::size_t ls = m.lay.sites();
        std::vector<std::vector<u32>> occs;
        std::vector<double> ar, ai;
        if (c->init_kind == 0) {
            i64 site = c->init_site;
            if (site < 0) site = m.site_index(m.ext[0] / 2, m.ext[1] / 2, m.ext[2] / 2);
            if (site >= i64(m.nsites)) throw Fail("initial state: site index out of range");
            std::vector<u32> occ(ls, 0);
            occ[0] = u32(site);
            occs.push_back(occ);
            ar.push_back(1.0);
            ai.push_back(0.0);
        } else if (c->init_kind == 1) {
            std::vector<u32> occ(ls, 0);
            for (u32 j = 0; j < m.nsites; ++j) {
                occ[0] = j;
                occs.push_back(occ);
                ar.push_back(1.0 / std::sqrt(double(m.nsites)));
                ai.push_back(0.0);
            }
        } else {
            if (c->n_entries == 0) throw Fail("initial state: empty explicit list");
            for (u64 e = 0; e < c->n_entries; ++e) {
                occs.emplace_back(c->entry_occ + e * ls, c->entry_occ + (e + 1) * ls);
                ar.push_back(c->entry_amp[2 * e]);
                ai.push_back(c->entry_amp[2 * e + 1]);
            }
        }
        std::vector<u32> keys(occs.size() * w);
        for (std::size_t k = 0; k < occs.size(); ++k) {
            if (po_pack(pm, occs[k].data(), keys.data() + k * w) != 0) throw Fail(g_err);
        }
        std::vector<std::size_t> idx(occs.size());
        std::iota(idx.begin(), idx.end(), std::size_t(0));
        std::sort(idx.begin(), idx.end(),
                  [&](std::size_t a, std::size_t b) { return key_less(keys.data() + a * w, keys.data() + b * w, w); });
        std::vector<u32> seeds;
        std::vector<double> sc;
        for (std::size_t k = 0; k < idx.size(); ++k) {
            if (k > 0 && key_eq(keys.data() + idx[k] * w, keys.data() + idx[k - 1] * w, w))
                throw Fail("initial state: duplicate basis key");
            seeds.insert(seeds.end(), keys.begin() + idx[k] * w, keys.begin() + (idx[k] + 1) * w);
            sc.push_back(ar[idx[k]]);
            sc.push_back(ai[idx[k]]);
        }
        const double n2 = norm2_serial(sc.data(), idx.size());
        if (n2 <= 0) throw Fail("initial state: not normalizable");
        const double nrm = std::sqrt(n2);
        for (double& v : sc) v /= nrm;  // complex / real = componentwise division

        Space sp = grow(m, seeds.data(), idx.size(), c->m_init);
        auto r = std::make_unique<po_run>();
        r->model = pm;
        r->cfg = *c;
        r->cfg.entry_occ = nullptr;
        r->cfg.entry_amp = nullptr;
        r->coeff.resize(2 * sp.rows);
        const double lost = remap(seeds.data(), sc.data(), idx.size(), sp.table.data(), sp.rows, w, r->coeff.data());
        if (lost != 0) throw Fail("initialize: seed keys lost during growth");
        r->words = std::move(sp.table);
        r->h = std::move(sp.h);
        r->t = 0;
        *out = r.release();
    });
}

// one pass of run()'s loop body, engine.hpp:333-368 with step() = :268-291
int po_run_step(po_run* r, po_diag* out) {
    return guarded([&] {
        const Model& m = r->model->m;
        const po_run_cfg& c = r->cfg;
        const u32 w = m.lay.words;
        const u64 s = r->steps_done + 1;
        const std::size_t rows = r->words.size() / w;
        po_diag d{};
        d.step = s;
        const double t0 = now_s();
        d.norm_pre = std::sqrt(norm2_serial(r->coeff.data(), rows));
        if (s == 1) {
            d.norm_post = d.norm_pre;
            d.q_true = rows;
            const double ta = now_s();
            d.energy = expectation(r->h, r->coeff.data());
            const double tb = now_s();
            std::vector<double> psi = r->coeff;
            const ExpmvOut e = taylor(r->h, psi.data(), c.dt, c.rtol, c.max_order, c.substeps);
            const double tc = now_s();
            d.taylor_order = e.order;
            d.delta_norm_expmv = std::sqrt(norm2_serial(psi.data(), rows)) - d.norm_post;
            r->coeff.swap(psi);
            r->times.expectation += tb - ta;
            r->times.expmv += tc - tb;
            r->times.spmv_nnz += u64(e.order) * r->h.val.size();
        } else {
            const double ta = now_s();
            const auto keep = select_rows(r->coeff.data(), rows, c.q_nom, po_mix_seed(c.seed + s));
            std::vector<u32> kept(keep.size() * w);
            for (std::size_t k = 0; k < keep.size(); ++k)
                std::copy(r->words.begin() + keep[k] * w, r->words.begin() + (keep[k] + 1) * w, kept.begin() + k * w);
            const double tb = now_s();
            Space next = grow(m, kept.data(), keep.size(), c.m);
            need_memory(u64(next.rows) * 16 * 4, "state vectors");
            const double tc = now_s();
            std::vector<double> psi(2 * next.rows);
            d.discarded_weight = remap(r->words.data(), r->coeff.data(), rows, next.table.data(), next.rows, w, psi.data());
            const double td = now_s();
            d.norm_post = std::sqrt(norm2_serial(psi.data(), next.rows));
            d.q_true = next.rows;
            d.energy = expectation(next.h, psi.data());
            const double te = now_s();
            const ExpmvOut e = taylor(next.h, psi.data(), c.dt, c.rtol, c.max_order, c.substeps);
            const double tf = now_s();
            d.taylor_order = e.order;
            d.delta_norm_expmv = std::sqrt(norm2_serial(psi.data(), next.rows)) - d.norm_post;
            r->coeff.swap(psi);
            r->words = std::move(next.table);
            r->h = std::move(next.h);
            r->times.select += tb - ta;
            r->times.grow += tc - tb;
            r->times.remap += td - tc;
            r->times.expectation += te - td;
            r->times.expmv += tf - te;
            r->times.spmv_nnz += u64(e.order) * r->h.val.size();
        }
        r->t = r->t + c.dt;
        d.t = r->t;
        r->times.total += now_s() - t0;
        r->steps_done = s;
        if (out) *out = d;
    });
}

int po_run_info(const po_run* r, uint64_t* rows, uint64_t* nnz, double* t, uint64_t* steps_done) {
    if (rows) *rows = r->words.size() / r->model->m.lay.words;
    if (nnz) *nnz = r->h.val.size();
    if (t) *t = r->t;
    if (steps_done) *steps_done = r->steps_done;
    return 0;
}
int po_run_state(const po_run* r, uint32_t* words, double* coeff) {
    if (words) std::copy(r->words.begin(), r->words.end(), words);
    if (coeff) std::copy(r->coeff.begin(), r->coeff.end(), coeff);
    return 0;
}
int po_run_csr(const po_run* r, int64_t* row_ptr, int32_t* col, double* val) {
    if (row_ptr) std::copy(r->h.row_ptr.begin(), r->h.row_ptr.end(), row_ptr);
    if (col) std::copy(r->h.col.begin(), r->h.col.end(), col);
    if (val) std::copy(r->h.val.begin(), r->h.val.end(), val);
    return 0;
}

// detail::observe, engine.hpp:299-311
int po_run_observe(const po_run* r, double* norm, double* energy, double* rmsd_out, double* xbar, double* amp,
                   double* dens) {
    return guarded([&] {
        const Model& m = r->model->m;
        const std::size_t rows = r->words.size() / m.lay.words;
        const double nrm = std::sqrt(norm2_serial(r->coeff.data(), rows));
        if (norm) *norm = nrm;
        const double n2 = std::pow(nrm, 2);  // observables.hpp:78
        if (n2 == 0.0) throw Fail("energy: zero-norm state");
        if (energy) *energy = expectation(r->h, r->coeff.data()) / n2;
        std::vector<double> p(m.nsites);
        density(m, r->words.data(), r->coeff.data(), rows, p.data());
        if (rmsd_out) *rmsd_out = spread_rmsd(m, p.data());
        if (xbar) {
            double acc = 0;
            for (u32 i = 0; i < m.nsites; ++i) acc += double(i) * p[i];
            *xbar = acc;
        }
        if (amp) dipole(m, r->words.data(), r->coeff.data(), rows, amp);
        if (dens) std::copy(p.begin(), p.end(), dens);
    });
}
void po_run_destroy(po_run* r) { delete r; }

// run(), engine.hpp:318-375: ceil(t_max/dt - 1e-9) steps, stop at the first failing step
int po_run_all(const po_model* m, const po_run_cfg* c, po_diag* diag, uint64_t cap, uint64_t* n_diag,
               po_run** final_out) {
    po_run* r = nullptr;
    if (po_run_begin(m, c, &r) != 0) return 1;
    const u64 nsteps = c->t_max <= 0 ? 0 : u64(std::ceil(c->t_max / c->dt - 1e-9));
    u64 done = 0;
    int rc = 0;
    for (u64 s = 1; s <= nsteps; ++s) {
        po_diag d;
        if (po_run_step(r, &d) != 0) {
            g_err = "step " + std::to_string(s) + ": " + g_err;
            rc = 1;
            break;
        }
        if (done < cap) diag[done] = d;
        ++done;
    }
    if (n_diag) *n_diag = done;
    if (final_out)
        *final_out = r;
    else
        po_run_destroy(r);
    return rc;
}

int po_run_times(const po_run* r, po_phase_times* out) {
    *out = r->times;
    return 0;
}

}  // extern "C"
