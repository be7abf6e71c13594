// host_model.hpp -- host-side model description: lattice geometry, parameter broadcast, key layout,
// pack/unpack and the seed state.  Mirrors build_model (reference lattice_models.hpp:140-189),
// SiteLayout (basis_codec.hpp:39-77), pack_state/unpack_state (:131-172) and
// detail::build_seed_state (engine.hpp:165-229) for the two exciton model kinds.
#pragma once
#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace pb {

struct PacesError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

using cplx = std::complex<double>;

struct HostModel {
    int kind = 1;  // 0 tight binding, 1 holstein
    int ndim = 1;
    std::array<uint32_t, 3> extents{1, 1, 1};
    uint32_t L = 1;
    uint32_t d_pho = 1;
    std::vector<double> eps, omega, g;                   // [L] after broadcast (omega, g empty for tight binding)
    std::vector<std::pair<uint32_t, uint32_t>> bonds;    // (low, high), reference enumeration order
    std::vector<double> hop;                             // per bond
    // layout
    std::vector<uint32_t> dims;
    std::vector<uint8_t> bits;
    std::vector<uint32_t> offsets;
    uint32_t total_bits = 0, W = 1;
    int b0 = 0, bp = 0;
    uint32_t n_terms = 0;

    uint32_t index(uint32_t x, uint32_t y, uint32_t z) const { return (z * extents[1] + y) * extents[0] + x; }
    size_t layout_sites() const { return dims.size(); }
};

inline int bits_for_dim(uint32_t d) {
    if (d <= 1) return 0;
    int b = 0;
    uint32_t v = d - 1;
    while (v) {
        ++b;
        v >>= 1;
    }
    return b;
}

inline std::vector<double> broadcast(const double* v, int nv, size_t n, const char* name) {
    if (nv <= 0 || v == nullptr) return std::vector<double>(n, 0.0);
    if (nv == 1) return std::vector<double>(n, v[0]);
    if (size_t(nv) != n)
        throw PacesError(std::string(name) + ": expected 1 or " + std::to_string(n) + " values, got " +
                         std::to_string(nv));
    return std::vector<double>(v, v + nv);
}

inline HostModel build_host_model(int kind, int ndim, const uint32_t* extents, const double* eps, int n_eps,
                                  const double* hop, int n_hop, const double* omega, int n_omega, const double* g,
                                  int n_g, uint32_t d_pho) {
    HostModel m;
    if (kind != 0 && kind != 1) throw PacesError("dynamics runs support exciton models (tb, holstein) only");
    if (ndim < 1 || ndim > 3 || extents == nullptr) throw PacesError("lattice must have 1 to 3 extents");
    m.kind = kind;
    m.ndim = ndim;
    for (int i = 0; i < ndim; ++i) {
        if (extents[i] == 0) throw PacesError("lattice extent must be positive");
        m.extents[i] = extents[i];
    }
    m.L = m.extents[0] * m.extents[1] * m.extents[2];
    for (uint32_t z = 0; z < m.extents[2]; ++z)
        for (uint32_t y = 0; y < m.extents[1]; ++y)
            for (uint32_t x = 0; x < m.extents[0]; ++x) {
                const uint32_t here = m.index(x, y, z);
                if (x + 1 < m.extents[0]) m.bonds.emplace_back(here, m.index(x + 1, y, z));
                if (y + 1 < m.extents[1]) m.bonds.emplace_back(here, m.index(x, y + 1, z));
                if (z + 1 < m.extents[2]) m.bonds.emplace_back(here, m.index(x, y, z + 1));
            }
    m.eps = broadcast(eps, n_eps, m.L, "eps");
    m.hop = broadcast(hop, n_hop, m.bonds.size(), "J");
    m.dims.push_back(m.L);
    if (kind == 1) {
        if (d_pho < 1) throw PacesError("d_pho must be >= 1");
        m.d_pho = d_pho;
        m.dims.insert(m.dims.end(), m.L, d_pho);
        m.omega = broadcast(omega, n_omega, m.L, "omega0");
        m.g = broadcast(g, n_g, m.L, "g");
    } else {
        m.d_pho = 1;
    }
    uint32_t off = 0;
    for (size_t i = 0; i < m.dims.size(); ++i) {
        const int b = bits_for_dim(m.dims[i]);
        m.bits.push_back(uint8_t(b));
        m.offsets.push_back(off);
        off += uint32_t(b);
    }
    m.total_bits = off;
    m.W = std::max<uint32_t>(1, (off + 31) / 32);
    m.b0 = m.bits[0];
    m.bp = (kind == 1) ? bits_for_dim(d_pho) : 0;
    for (double e : m.eps) m.n_terms += (e != 0.0);
    for (double h : m.hop) m.n_terms += (h != 0.0);
    for (double o : m.omega) m.n_terms += (o != 0.0);
    for (double x : m.g) m.n_terms += (x != 0.0);
    return m;
}

inline uint32_t host_get_site(const HostModel& m, const uint32_t* row, size_t site) {
    const uint32_t b = m.bits[site];
    if (b == 0) return 0;
    const uint32_t off = m.offsets[site];
    const uint32_t wi = off / 32, bit = off % 32;
    const uint64_t hi = row[wi], lo = (wi + 1 < m.W) ? row[wi + 1] : 0;
    const uint64_t win = (hi << 32) | lo;
    const uint64_t mask = (b >= 32) ? 0xffffffffull : ((1ull << b) - 1);
    return uint32_t((win >> (64 - bit - b)) & mask);
}

inline void host_set_site(const HostModel& m, uint32_t* row, size_t site, uint32_t value) {
    const uint32_t b = m.bits[site];
    if (b == 0) return;
    const uint32_t off = m.offsets[site];
    const uint32_t wi = off / 32, bit = off % 32;
    const int sh = int(64 - bit - b);
    const uint64_t mask = ((b >= 32) ? 0xffffffffull : ((1ull << b) - 1)) << sh;
    const uint64_t val = (uint64_t(value) << sh) & mask;
    row[wi] = uint32_t((row[wi] & ~uint32_t(mask >> 32)) | uint32_t(val >> 32));
    if (wi + 1 < m.W) row[wi + 1] = uint32_t((row[wi + 1] & ~uint32_t(mask)) | uint32_t(val));
}

inline void host_pack(const HostModel& m, const uint32_t* occ, size_t n_occ, uint32_t* out) {
    if (n_occ != m.layout_sites())
        throw PacesError("pack: occupation vector length " + std::to_string(n_occ) + " does not match site count " +
                         std::to_string(m.layout_sites()));
    std::fill(out, out + m.W, 0u);
    for (size_t i = 0; i < n_occ; ++i) {
        if (occ[i] >= m.dims[i])
            throw PacesError("pack: occupation " + std::to_string(occ[i]) + " out of range at site " +
                             std::to_string(i) + " (dim " + std::to_string(m.dims[i]) + ")");
        host_set_site(m, out, i, occ[i]);
    }
}

inline void host_unpack(const HostModel& m, const uint32_t* row, uint32_t* occ) {
    for (size_t i = 0; i < m.layout_sites(); ++i) {
        const uint32_t v = host_get_site(m, row, i);
        if (v >= m.dims[i])
            throw PacesError("unpack: corrupt row, decoded value " + std::to_string(v) + " >= dim " +
                             std::to_string(m.dims[i]) + " at site " + std::to_string(i));
        occ[i] = v;
    }
}

inline bool host_row_less(const uint32_t* a, const uint32_t* b, uint32_t w) {
    for (uint32_t i = 0; i < w; ++i)
        if (a[i] != b[i]) return a[i] < b[i];
    return false;
}

/// Shard owner: identical arithmetic to owner_of() in keys.cuh (hash of the key with the exciton register zeroed).
inline uint32_t host_owner(const HostModel& m, const uint32_t* key, uint32_t P) {
    uint64_t h = 0x9E3779B97F4A7C15ull;
    for (uint32_t i = 0; i < m.W; ++i) {
        uint32_t w = key[i];
        if (i == 0 && m.b0 > 0) w = (m.b0 >= 32) ? 0u : (w & (0xffffffffu >> m.b0));
        h = (h ^ w) * 0xBF58476D1CE4E5B9ull;
        h ^= h >> 29;
    }
    h *= 0x94D049BB133111EBull;
    h ^= h >> 32;
    return uint32_t(h % P);
}

/// Strictly ascending rows (PackedBasisTable::sorted).
inline bool host_rows_sorted(const uint32_t* words, uint64_t rows, uint32_t w) {
    for (uint64_t i = 1; i < rows; ++i)
        if (!host_row_less(words + (i - 1) * w, words + i * w, w)) return false;
    return true;
}

/// Seed keys + amplitudes, sorted by key, duplicates rejected, normalised (engine.hpp:165-229).
inline void build_seed_state(const HostModel& m, int init_kind, int64_t init_site, uint64_t n_entries,
                             const uint32_t* entry_occ, const double* entry_amp, std::vector<uint32_t>& words,
                             std::vector<cplx>& amps) {
    const size_t ls = m.layout_sites();
    std::vector<std::vector<uint32_t>> occs;
    std::vector<cplx> a0;
    if (init_kind == 0) {
        int64_t site = init_site;
        if (site < 0) site = m.index(m.extents[0] / 2, m.extents[1] / 2, m.extents[2] / 2);
        if (site >= int64_t(m.L)) throw PacesError("initial state: site index out of range");
        std::vector<uint32_t> occ(ls, 0);
        occ[0] = uint32_t(site);
        occs.push_back(occ);
        a0.push_back(1.0);
    } else if (init_kind == 1) {
        std::vector<uint32_t> occ(ls, 0);
        for (uint32_t j = 0; j < m.L; ++j) {
            occ[0] = j;
            occs.push_back(occ);
            a0.push_back(1.0 / std::sqrt(double(m.L)));
        }
    } else if (init_kind == 2) {
        if (n_entries == 0 || !entry_occ || !entry_amp) throw PacesError("initial state: empty explicit list");
        for (uint64_t k = 0; k < n_entries; ++k) {
            occs.emplace_back(entry_occ + k * ls, entry_occ + (k + 1) * ls);
            a0.emplace_back(entry_amp[2 * k], entry_amp[2 * k + 1]);
        }
    } else {
        throw PacesError("initial state: unknown kind");
    }
    const size_t n = occs.size();
    std::vector<uint32_t> raw(n * m.W);
    for (size_t k = 0; k < n; ++k) host_pack(m, occs[k].data(), occs[k].size(), raw.data() + k * m.W);
    std::vector<size_t> idx(n);
    std::iota(idx.begin(), idx.end(), size_t(0));
    std::sort(idx.begin(), idx.end(),
              [&](size_t a, size_t b) { return host_row_less(raw.data() + a * m.W, raw.data() + b * m.W, m.W); });
    words.clear();
    amps.clear();
    for (size_t k = 0; k < n; ++k) {
        const uint32_t* r = raw.data() + idx[k] * m.W;
        if (k > 0 && std::equal(r, r + m.W, raw.data() + idx[k - 1] * m.W))
            throw PacesError("initial state: duplicate basis key");
        words.insert(words.end(), r, r + m.W);
        amps.push_back(a0[idx[k]]);
    }
    double n2 = 0;
    for (const cplx& a : amps) n2 += std::norm(a);
    if (n2 <= 0) throw PacesError("initial state: not normalizable");
    for (cplx& a : amps) a /= std::sqrt(n2);
}

}  // namespace pb
