"""GPU parity tests (run on the B200 box with -m gpu).  Every call goes through the C ABI of
libpaces_b200.so; the checker is the CPU oracle (oracle/libpaces_oracle.so, pinned to the reference by
tests/test_oracle_port.py) and the committed golden fixtures generated from the unmodified reference.

Bars: subspace tables, CSR structure and CSR values bit-exact; q_true, nnz, Taylor order equal; coefficients
bit-exact (the kernels reproduce the reference's summation order without FMA); norms, energy, discarded
weight, density and dipole amplitude within 1e-10 relative (parallel reductions reassociate the serial sums).
"""
import numpy as np
import pytest

from cases import CASES

pytestmark = pytest.mark.gpu

RTOL = 1e-10


def _close(a, b, rtol=RTOL, atol=0.0):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return bool(np.all(np.abs(a - b) <= atol + rtol * np.maximum(np.abs(a), np.abs(b))))


@pytest.fixture(scope="module")
def gpu():
    import paper_2603_07341_b200 as pb

    return pb


def _ctx(gpu, model_kw):
    return gpu.Context(gpu.ModelDef(**model_kw))


def _check_diag(d, g, name, s):
    for k in ("step", "q_true", "taylor_order"):
        assert d[k] == g[k], (name, s, k, d[k], g[k])
    assert _close(d["t"], g["t"], 1e-14), (name, s, "t")
    for k in ("norm_pre", "norm_post"):
        assert _close(d[k], g[k]), (name, s, k, d[k], g[k])
    # energy is a signed sum that can cancel to ~0: compare on the scale of the terms (|<H>| <= ||H|| ~ O(10))
    assert _close(d["energy"], g["energy"], RTOL, 1e-12), (name, s, "energy", d["energy"], g["energy"])
    assert _close(d["discarded_weight"], g["discarded_weight"], 1e-9, 1e-30), (name, s, d["discarded_weight"],
                                                                                g["discarded_weight"])
    # a difference of two norms ~1: reassociated sums move it by a few ulp of 1 per 1e5 rows (reference bound on
    # the quantity itself: |delta| <= 1e-12, acceptance C2)
    assert abs(d["delta_norm_expmv"] - g["delta_norm_expmv"]) <= 1e-12, (name, s, "delta_norm_expmv")


@pytest.mark.parametrize("name", list(CASES))
def test_trajectory_matches_reference_golden(gpu, golden, name):
    """Full initialize + step loop against the fixtures produced by the unmodified reference."""
    from oracle.pyoracle import fnv1a64

    case, g = CASES[name], golden[name]
    ctx = _ctx(gpu, case["model"])
    assert dict(sites=ctx.layout_sites, words=ctx.words, bits=ctx.total_bits, terms=ctx.n_terms) == g["layout"]
    run = ctx.run(**case["run"])
    rows, nnz, _, _ = run.info()
    w, c = run.state()
    rp, col, val = run.csr()
    assert (rows, nnz, fnv1a64(w), fnv1a64(c)) == (g["init"]["q_true"], g["init"]["nnz"], g["init"]["table"],
                                                   g["init"]["coeff"])
    assert (fnv1a64(col), fnv1a64(val)) == (g["init"]["col"], g["init"]["val"])
    for s in range(1, case["steps"] + 1):
        d = run.step()
        if str(s) in g["snaps"]:
            gs = g["snaps"][str(s)]
            w, c = run.state()
            rp, col, val = run.csr()
            assert int(rp[-1]) == gs["nnz"]
            assert fnv1a64(w) == gs["table"], (name, s, "table")
            assert (fnv1a64(rp), fnv1a64(col), fnv1a64(val)) == (gs["row_ptr"], gs["col"], gs["val"]), (name, s, "csr")
            assert fnv1a64(c) == gs["coeff"], (name, s, "coefficients not bit-identical")
            _check_diag(d, gs["diag"], name, s)
    ob = run.observe()
    fo = g["final_observe"]
    assert _close([ob["amp"].real, ob["amp"].imag], fo["amp"], RTOL, 1e-16)
    assert _close(ob["density"], fo["density"])
    for k in ("norm", "energy", "rmsd", "xbar"):
        assert _close(ob[k], fo[k], RTOL, 1e-12), k
    assert ctx.kernel_launches > 0


@pytest.mark.parametrize("name", ["cfg1_holstein_L4_d8", "disordered_4x3_d7", "cube_2x2x2_d16", "tb_chain_31"])
def test_every_step_against_oracle(gpu, port, name):
    """Step-by-step lockstep with the CPU oracle: tables and coefficients compared at EVERY step."""
    from oracle.pyoracle import ModelDef

    case = CASES[name]
    ctx = _ctx(gpu, case["model"])
    om = port.model(ModelDef(**case["model"]))
    rg, ro = ctx.run(**case["run"]), om.run(**case["run"])
    for s in range(1, min(case["steps"], 30) + 1):
        dg, do = rg.step(), ro.step()
        wg, cg = rg.state()
        wo, co = ro.state()
        assert np.array_equal(wg, wo), (name, s)
        assert cg.tobytes() == co.tobytes(), (name, s)
        _check_diag(dg, do, name, s)
    for a, b in zip(rg.csr(), ro.csr()):
        assert a.tobytes() == b.tobytes()


def test_apply_terms_and_grow_match_golden(gpu, golden_small):
    gs = golden_small
    ctx = _ctx(gpu, CASES["disordered_4x3_d7"]["model"])
    res = ctx.apply_terms(gs["apply_src"])
    off = 0
    for i, (keys, amps) in enumerate(res):
        n = int(gs["apply_counts"][i])
        rk, ra = gs["apply_keys"][off:off + n], gs["apply_amps"][off:off + n]
        # the reference emits in term order; the device emits in ascending key order: compare as sorted sets
        order = np.lexsort(rk.T[::-1])
        assert np.array_equal(keys, rk[order]) and amps.tobytes() == ra[order].tobytes()
        off += n
    tw, rp, col, val = ctx.grow(gs["grow_seeds"], 2)
    assert np.array_equal(tw, gs["grow_table"]) and np.array_equal(rp, gs["grow_row_ptr"])
    assert np.array_equal(col, gs["grow_col"]) and val.tobytes() == gs["grow_val"].tobytes()


def test_selection_ties_match_golden(gpu, golden_small):
    """4-way tie at the cutoff: the seeded Fisher-Yates draw of engine.hpp:137-142 (test_engine.cpp:126-160)."""
    gs = golden_small
    ctx = _ctx(gpu, dict(kind=1, extents=(3,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(0.5,), d_pho=2))
    seen = set()
    for seed in range(16):
        kept = ctx.truncate_select(gs["sel_words"], gs["sel_coeff"], 3, seed)
        assert np.array_equal(kept, gs["sel_kept_%d" % seed])
        seen.add(kept.tobytes())
    assert len(seen) > 1


def test_selection_large_groups_against_oracle(gpu, port):
    """Selection paths beyond the golden vectors, on a 1e5+-row table (engine.hpp:107-156): (a) the usual case --
    the group sharing the cutoff's first 22 bits is tiny and one CTA finishes the digits; (b) > 65536 weights share
    those bits but differ further down (full radix passes); (c) a massive exact tie cut by the seeded draw."""
    from oracle.pyoracle import ModelDef

    kw = dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16)
    ctx = _ctx(gpu, kw)
    om = port.model(ModelDef(**kw))
    seed = om.pack([8] + [0] * 16).reshape(1, -1)
    table = ctx.grow(seed, 14)[0]
    n = table.shape[0]
    assert n > 100000
    rng = np.random.default_rng(5)
    cases = {
        "spread": (rng.standard_normal(n) + 1j * rng.standard_normal(n)) * np.exp(-8 * rng.random(n)),
        "shared_prefix": np.sqrt(1.0 + np.arange(n) * 2.0 ** -40) + 0j,
        "massive_tie": np.full(n, 0.5 + 0.5j),
    }
    cases["massive_tie"][:: 97] = 2.0
    cases["massive_tie"][5:: 89] = 0.0
    for name, c in cases.items():
        c = np.ascontiguousarray(c.astype(np.complex128))
        for q_nom, sd in ((1000, 3), (n // 2, 11), (n - 3, 2), (n + 5, 0)):
            got = ctx.truncate_select(table, c, q_nom, sd)
            want = om.truncate_select(table, c, q_nom, sd)
            assert np.array_equal(got, want), (name, q_nom, got.shape, want.shape)


@pytest.mark.parametrize("name", ["disordered_4x3_d7", "cube_2x2x2_d16", "tb_chain_31", "cfg2_layout_L16_d16_small",
                                  "square_3x3_d5"])
def test_operators_against_oracle(gpu, port, name):
    """Each stand-alone operator (host buffers in/out) against the oracle on fresh inputs."""
    from oracle.pyoracle import ModelDef, csr_expectation, csr_matvec, expmv, state_norm

    case = CASES[name]
    ctx = _ctx(gpu, case["model"])
    om = port.model(ModelDef(**case["model"]))
    ro = om.run(**case["run"])
    for _ in range(6):
        ro.step()
    w, c = ro.state()
    rp, col, val = ro.csr()
    rng = np.random.RandomState(0)
    x = rng.uniform(-1, 1, len(c)) + 1j * rng.uniform(-1, 1, len(c))
    assert ctx.csr_matvec(rp, col, val, x).tobytes() == csr_matvec(port, rp, col, val, x).tobytes()
    assert _close(ctx.csr_expectation(rp, col, val, x), csr_expectation(port, rp, col, val, x), RTOL, 1e-12)
    a, b = ctx.expmv(rp, col, val, c), expmv(port, rp, col, val, c)
    assert a[0].tobytes() == b[0].tobytes() and a[1] == b[1] and _close(a[2], b[2], 1e-9)
    a, b = ctx.expmv(rp, col, val, x, dt=0.02, substeps=3), expmv(port, rp, col, val, x, dt=0.02, substeps=3)
    assert a[0].tobytes() == b[0].tobytes() and a[1] == b[1]
    assert _close(ctx.state_norm(x), state_norm(port, x))
    assert _close(ctx.exciton_density(w, c), om.exciton_density(w, c))
    assert _close(ctx.exciton_density(w, c).sum(), np.sum(np.abs(c) ** 2), 1e-13)  # test_observables.cpp:73-86
    ag, ao = ctx.dipole_amplitude(w, c), om.dipole_amplitude(w, c)
    assert _close([ag.real, ag.imag], [ao.real, ao.imag], RTOL, 1e-16)
    if case["model"]["kind"] == 1:
        assert _close(ctx.phonon_numbers(w, c), om.phonon_numbers(w, c), RTOL, 1e-18)
    for q in (1, 7, max(1, len(c) // 3), len(c), len(c) + 5):
        for seed in (0, 5):
            assert np.array_equal(ctx.truncate_select(w, c, q, seed), om.truncate_select(w, c, q, seed)), (q, seed)
    kept = om.truncate_select(w, c, max(1, len(c) // 4), 1)
    for order in (0, 1, 2, 3):
        gg, go = ctx.grow(kept, order), om.grow(kept, order)
        for u, v in zip(gg, go):
            assert u.tobytes() == v.tobytes(), (name, order)
    tw = om.grow(kept, 1)[0]
    (cg, dg), (co, do) = ctx.remap(w, c, tw), om.remap(w, c, tw)
    assert cg.tobytes() == co.tobytes() and _close(dg, do, 1e-9, 1e-30)
    idx = rng.randint(0, len(w), 50)
    got = ctx.apply_terms(w[idx])
    for i, (keys, amps) in zip(idx, got):
        rk, ra = om.apply_terms(w[i])
        order = np.lexsort(rk.T[::-1])
        assert np.array_equal(keys, rk[order]) and amps.tobytes() == ra[order].tobytes()


def test_edge_cases(gpu, port):
    from oracle.pyoracle import ModelDef

    kw = CASES["cfg1_holstein_L4_d8"]["model"]
    ctx = _ctx(gpu, kw)
    om = port.model(ModelDef(**kw))
    # m = 0 returns the seeds (test_subspace.cpp:91-97); single seed; vacuum key has no diagonal (App. A.5)
    seed = om.pack([2, 0, 0, 0, 0]).reshape(1, -1)
    for order in (0, 1):
        for u, v in zip(ctx.grow(seed, order), om.grow(seed, order)):
            assert u.tobytes() == v.tobytes()
    # full coverage: growing far enough saturates the 4 * 8^4 space; the next order adds nothing
    a, b = ctx.grow(seed, 40), ctx.grow(seed, 41)
    assert a[0].shape[0] == 4 * 8 ** 4 and a[0].tobytes() == b[0].tobytes() and a[3].tobytes() == b[3].tobytes()
    ref = om.grow(seed, 40)
    assert all(u.tobytes() == v.tobytes() for u, v in zip(a, ref))
    # errors carry the reference's text
    with pytest.raises(gpu.PacesError, match="empty seed set"):
        ctx.grow(np.zeros((0, 1), np.uint32), 1)
    with pytest.raises(gpu.PacesError, match="must be sorted"):
        ctx.grow(np.array([[5], [3]], np.uint32), 1)
    with pytest.raises(gpu.PacesError, match="no support"):
        ctx.truncate_select(seed, np.zeros(1, np.complex128), 3, 0)
    rp = np.array([0, 1], np.int64)
    with pytest.raises(gpu.PacesError, match="reduce dt"):  # test_propagator.cpp:157-169
        ctx.expmv(rp, np.array([0], np.int32), np.array([1e6]), np.array([1.0 + 0j]), dt=1.0, max_order=20)
    with pytest.raises(gpu.PacesError, match="non-finite"):
        ctx.expmv(rp, np.array([0], np.int32), np.array([1.0]), np.array([np.nan + 0j]))
    # H = 0 is the identity in <= 2 orders (test_propagator.cpp:31-41); diagonal phase (:43-54)
    c, order, _ = ctx.expmv(np.array([0, 0, 0], np.int64), np.zeros(0, np.int32), np.zeros(0), np.array([1.0, 2.0j]))
    assert order <= 2 and np.array_equal(c, np.array([1.0, 2.0j]))
    c, order, _ = ctx.expmv(rp, np.array([0], np.int32), np.array([0.7]), np.array([1.0 + 0j]), dt=0.3)
    assert abs(c[0] - np.exp(-0.21j)) < 1e-15


def test_memory_cap_and_failed_step_keeps_state(gpu, monkeypatch):
    kw = CASES["cfg1_holstein_L4_d8"]
    ctx = _ctx(gpu, kw["model"])
    monkeypatch.setenv("PACES_MAX_MEMORY_BYTES", "1000")
    with pytest.raises(gpu.PacesError, match="memory cap"):  # test_engine.cpp:358-375
        ctx.run(**kw["run"])
    monkeypatch.delenv("PACES_MAX_MEMORY_BYTES")
    run = ctx.run(**kw["run"])
    for _ in range(3):
        run.step()
    w0, c0 = run.state()
    monkeypatch.setenv("PACES_MAX_MEMORY_BYTES", "1000")
    with pytest.raises(gpu.PacesError, match="memory cap"):
        run.step()
    w1, c1 = run.state()  # engine.hpp:263-267: a failed step leaves the last good state intact
    assert w0.tobytes() == w1.tobytes() and c0.tobytes() == c1.tobytes() and run.info()[3] == 3
    monkeypatch.delenv("PACES_MAX_MEMORY_BYTES")
    run.step()
    assert run.info()[3] == 4


def test_bit_identical_reruns(gpu):
    """test_engine.cpp:315-342: same config + seed -> identical bits, diagnostics included."""
    case = CASES["ties_holstein_L5_d6"]
    out = []
    for _ in range(2):
        ctx = _ctx(gpu, case["model"])
        run = ctx.run(**case["run"])
        diags = [run.step() for _ in range(40)]
        w, c = run.state()
        out.append((diags, w.tobytes(), c.tobytes()))
    assert out[0] == out[1]


def test_large_step_properties(gpu, port):
    """BASELINE config 2 layout (1D L=16, d_pho=16, 68-bit keys) at a size the oracle still checks in
    seconds, plus size-independent properties of the step."""
    from oracle.pyoracle import ModelDef

    kw = dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16)
    run_kw = dict(init="localized", site=-1, m_init=8, m=2, q_nom=20000, dt=0.05, rtol=1e-15, t_max=1.0, seed=7)
    ctx = _ctx(gpu, kw)
    run = ctx.run(**run_kw)
    om = port.model(ModelDef(**kw))
    ro = om.run(**run_kw)
    for s in range(1, 9):
        d, do = run.step(), ro.step()
        assert d["q_true"] == do["q_true"] and d["taylor_order"] == do["taylor_order"]
        assert d["norm_post"] <= d["norm_pre"] * (1 + 1e-15)  # truncation never adds norm (test_engine.cpp:206-229)
        assert abs(d["delta_norm_expmv"]) <= 1e-12
    w, c = run.state()
    wo, co = ro.state()
    assert np.array_equal(w, wo) and c.tobytes() == co.tobytes()
    assert d["q_true"] >= 20000
    # table strictly ascending (canonical order), CSR symmetric with ascending columns
    assert np.all(np.lexsort(w.T[::-1]) == np.arange(len(w)))
    rp, col, val = run.csr()
    assert all(a.tobytes() == b.tobytes() for a, b in zip((rp, col, val), ro.csr()))
    import scipy.sparse as sp

    h = sp.csr_matrix((val, col, rp), shape=(len(w), len(w)))
    assert (h != h.T).nnz == 0  # Hermiticity, exact (test_subspace.cpp:160-166)
    # remap round trip: projecting onto the own table is the identity with zero discarded weight
    c2, disc = ctx.remap(w, c, w)
    assert c2.tobytes() == c.tobytes() and disc == 0.0
    # select with q_nom >= support keeps exactly the support
    kept = ctx.truncate_select(w, c, len(w), 0)
    assert np.array_equal(kept, w[np.abs(c) ** 2 > 0])


@pytest.mark.parametrize("name,model,run_kw,steps", [
    # BASELINE config 3: 2D 6x6 aggregate, one mode per site, optical start (150-bit keys, 5 words); the
    # autocorrelation <mu(t)mu(0)> is ObservablesRow.amp
    ("cfg3_2d_6x6", dict(kind=1, extents=(6, 6), eps=(0.0,), hop=(-0.55,), omega=(1.0,), g=(0.71,), d_pho=16),
     dict(init="optical", m_init=5, m=2, q_nom=20000, dt=0.05, rtol=1e-15, t_max=5.0, seed=7), 8),
    # BASELINE config 4: 3D 4x4x4 aggregate, localized start at the centre site (262-bit keys, 9 words)
    ("cfg4_3d_4x4x4", dict(kind=1, extents=(4, 4, 4), eps=(0.0,), hop=(0.55,), omega=(1.0,), g=(0.71,), d_pho=16),
     dict(init="localized", site=-1, m_init=6, m=2, q_nom=20000, dt=0.05, rtol=1e-15, t_max=5.0, seed=7), 8),
    # paper regime key width: 1D N=75, d_pho=16 -> 7 + 300 bits = 10 words
    ("wide_1d_75", dict(kind=1, extents=(75,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16),
     dict(init="localized", site=-1, m_init=6, m=2, q_nom=5000, dt=0.05, rtol=1e-15, t_max=5.0, seed=7), 6),
])
def test_baseline_configs_against_oracle(gpu, port, name, model, run_kw, steps):
    """BASELINE.json configs 3 and 4 (and a 10-word key) in lockstep with the oracle: tables, CSR and coefficients
    bit-exact at every step, observables (density, autocorrelation amplitude) within 1e-10."""
    from oracle.pyoracle import ModelDef

    ctx = _ctx(gpu, model)
    rg = ctx.run(**run_kw)
    ro = port.model(ModelDef(**model)).run(**run_kw)
    assert rg.info()[:2] == ro.info()[:2]
    for s in range(1, steps + 1):
        dg, do = rg.step(), ro.step()
        wg, cg = rg.state()
        wo, co = ro.state()
        assert np.array_equal(wg, wo), (name, s)
        assert cg.tobytes() == co.tobytes(), (name, s)
        _check_diag(dg, do, name, s)
        og, oo = rg.observe(), ro.observe()
        assert _close(og["density"], oo["density"], RTOL, 1e-18), (name, s)
        assert abs(og["amp"] - oo["amp"]) <= 1e-12, (name, s, og["amp"], oo["amp"])
    for a, b in zip(rg.csr(), ro.csr()):
        assert a.tobytes() == b.tobytes()
    assert dg["q_true"] > run_kw["q_nom"]


def test_scale_beyond_reduction_grid(gpu):
    """Regression (round 1): above ~3.9e7 rows the remap kernel's grid outgrew the reduction scratch and corrupted
    the state.  BASELINE config 2 at q_nom = 1.5e7 (q_true ~ 4.5e7) must keep evolving sanely once truncation binds:
    Taylor order in the low tens, norm conserved, q_true/q_nom near the measured kappa ~ 3.3-3.7."""
    model = dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16)
    ctx = _ctx(gpu, model)
    run = ctx.run(init="localized", site=-1, m_init=10, m=2, q_nom=15_000_000, dt=0.05, rtol=1e-15, t_max=50.0, seed=7)
    bound = 0
    for s in range(1, 14):
        d = run.step()
        assert 10 <= d["taylor_order"] <= 40, (s, d)
        assert abs(d["norm_post"] - 1.0) < 1e-9 and abs(d["delta_norm_expmv"]) < 1e-12, (s, d)
        if d["discarded_weight"] > 0 and d["q_true"] > 39_000_000:
            bound += 1
            assert 2.5 * 15_000_000 < d["q_true"] < 4.5 * 15_000_000, (s, d)
    assert bound >= 2
    ctx.close()


@pytest.mark.parametrize("name,model,run_kw,steps", [
    ("1d_L16", dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16),
     dict(init="localized", site=-1, m_init=8, m=2, q_nom=30000, dt=0.05, rtol=1e-15, t_max=5.0, seed=7), 25),
    ("2d_4x3_disordered_m3", dict(kind=1, extents=(4, 3), eps=tuple(0.05 * i - 0.2 for i in range(12)), hop=(0.55,),
                                 omega=tuple(1.0 + 0.01 * i for i in range(12)), g=(0.71,), d_pho=7),
     dict(init="optical", m_init=4, m=3, q_nom=3000, dt=0.05, rtol=1e-15, t_max=5.0, seed=3), 20),
    ("3d_4x4x4_m1", dict(kind=1, extents=(4, 4, 4), eps=(0.0,), hop=(0.55,), omega=(1.0,), g=(0.71,), d_pho=16),
     dict(init="localized", site=-1, m_init=5, m=1, q_nom=8000, dt=0.05, rtol=1e-15, t_max=5.0, seed=7), 15),
    ("tb_chain", dict(kind=0, extents=(61,), eps=(0.0,), hop=(1.0,)),
     dict(init="localized", site=-1, m_init=3, m=2, q_nom=9, dt=0.05, rtol=1e-15, t_max=5.0, seed=1), 30),
])
def test_incremental_adapt_equals_full_expansion(gpu, monkeypatch, name, model, run_kw, steps):
    """The incremental adapt phase (BFS over the previous H_eff in old index space, incremental.cuh) against the full
    expansion (PB200_NO_INCREMENTAL=1), step by step: tables, CSR and coefficients bit-identical, same diagnostics.
    The incremental run must really have taken the incremental path, including steps that needed key-based
    re-expansion of previous-frontier rows and keys from outside the previous table."""
    monkeypatch.delenv("PB200_NO_INCREMENTAL", raising=False)
    ri = _ctx(gpu, model).run(**run_kw)
    monkeypatch.setenv("PB200_NO_INCREMENTAL", "1")
    rf = _ctx(gpu, model).run(**run_kw)
    for s in range(1, steps + 1):
        monkeypatch.delenv("PB200_NO_INCREMENTAL", raising=False)
        di = ri.step()
        monkeypatch.setenv("PB200_NO_INCREMENTAL", "1")
        df = rf.step()
        assert di["q_true"] == df["q_true"] and di["taylor_order"] == df["taylor_order"], (name, s, di, df)
        for k in ("norm_pre", "norm_post", "energy", "discarded_weight"):
            assert _close(di[k], df[k], 1e-12, 1e-30), (name, s, k, di[k], df[k])
        wi, ci = ri.state()
        wf, cf = rf.state()
        assert np.array_equal(wi, wf), (name, s)
        assert ci.tobytes() == cf.tobytes(), (name, s)
        if s % 5 == 0 or s == steps:
            assert all(a.tobytes() == b.tobytes() for a, b in zip(ri.csr(), rf.csr())), (name, s)
    si, sf = ri.adapt_stats(), rf.adapt_stats()
    assert sf["incremental_steps"] == 0
    # step 1 only evolves; while the space is still exploding (more new keys than old rows) a step may fall back
    assert si["incremental_steps"] + si["fallbacks"] == steps - 1 and si["incremental_steps"] >= (steps - 1) // 2, si
    if name != "tb_chain":
        assert si["expanded_rows"] > 0 and si["side_keys"] > 0, si


@pytest.mark.gpu
@pytest.mark.parametrize("name,model,run_kw,steps,coded", [
    ("1d_L16_uniform", dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16),
     dict(init="localized", site=-1, m_init=8, m=2, q_nom=30000, dt=0.05, rtol=1e-15, t_max=5.0, seed=7), 20, True),
    ("2d_4x3_disordered", dict(kind=1, extents=(4, 3), eps=tuple(0.05 * i - 0.2 for i in range(12)), hop=(0.55,),
                              omega=tuple(1.0 + 0.01 * i for i in range(12)), g=(0.71,), d_pho=7),
     dict(init="optical", m_init=4, m=2, q_nom=3000, dt=0.05, rtol=1e-15, t_max=5.0, seed=3), 16, True),
    ("3d_4x4x4", dict(kind=1, extents=(4, 4, 4), eps=(0.0,), hop=(0.55,), omega=(1.0,), g=(0.71,), d_pho=16),
     dict(init="localized", site=-1, m_init=5, m=1, q_nom=8000, dt=0.05, rtol=1e-15, t_max=5.0, seed=7), 12, True),
    ("tb_chain", dict(kind=0, extents=(61,), eps=tuple(0.01 * i for i in range(61)), hop=(1.0,)),
     dict(init="localized", site=-1, m_init=3, m=2, q_nom=9, dt=0.05, rtol=1e-15, t_max=5.0, seed=1), 12, True),
    # 90 sites x 31 levels of a disordered coupling: more distinct matrix elements than the table holds -> no codes
    ("1d_L90_disordered_g", dict(kind=1, extents=(90,), eps=(0.0,), hop=(1.0,), omega=(1.0,),
                                g=tuple(0.5 + 0.001 * i for i in range(90)), d_pho=32),
     dict(init="localized", site=-1, m_init=3, m=1, q_nom=500, dt=0.05, rtol=1e-15, t_max=5.0, seed=2), 6, False),
])
def test_value_codes_equal_double_values(gpu, port, monkeypatch, name, model, run_kw, steps, coded):
    """Taylor tile kernels reading 2-byte value codes + the model's table of matrix elements (taylor.cuh, TaylorCodes;
    the codes travel with the entries through the incremental adapt phase) against the same kernels reading the 8-byte
    values (PB200_NO_VALUE_CODES=1) and against the oracle: coefficients bit-identical at every step.  Uniform models
    (diagonal tabulated), disordered omega / eps (diagonal kept per row), tight binding, and a model whose table
    would be too large (falls back to the values by itself)."""
    from oracle import pyoracle

    monkeypatch.delenv("PB200_NO_VALUE_CODES", raising=False)
    rc = _ctx(gpu, model).run(**run_kw)
    monkeypatch.setenv("PB200_NO_VALUE_CODES", "1")
    rv = _ctx(gpu, model).run(**run_kw)
    monkeypatch.delenv("PB200_NO_VALUE_CODES", raising=False)
    ro = port.model(pyoracle.ModelDef(**model)).run(**run_kw)
    for s in range(1, steps + 1):
        dc, dv, do = rc.step(), rv.step(), ro.step()
        assert dc["q_true"] == dv["q_true"] == do["q_true"], (name, s)
        assert dc["taylor_order"] == dv["taylor_order"] == do["taylor_order"], (name, s)
        (wc, cc), (wv, cv), (wo, co) = rc.state(), rv.state(), ro.state()
        assert np.array_equal(wc, wv) and np.array_equal(wc, wo), (name, s)
        assert cc.tobytes() == cv.tobytes() == co.tobytes(), (name, s)
    assert all(a.tobytes() == b.tobytes() for a, b in zip(rc.csr(), ro.csr())), name
    tc, tv = rc.times(), rv.times()
    assert tv["spmv_nnz_coded"] == 0
    if coded:
        assert tc["spmv_nnz_coded"] == tc["spmv_nnz"] > 0, (name, tc)
        assert rc.adapt_stats()["incremental_steps"] >= steps // 2
    else:
        assert tc["spmv_nnz_coded"] == 0, (name, tc)


@pytest.mark.gpu
@pytest.mark.parametrize("rtol,substeps,max_order", [(1e-15, 1, 200), (1e-6, 1, 200), (1e-3, 2, 200), (0.5, 1, 200),
                                                     (1e-15, 3, 200), (1e-15, 1, 9)])
def test_paired_taylor_orders_equal_single_orders(gpu, port, monkeypatch, rtol, substeps, max_order):
    """expmv with paired orders (an order whose predecessor did not meet the stop rule leaves c alone, the next one
    adds both terms in the reference's order; kernels.cuh TAYLOR_DEFER / TAYLOR_CATCHUP) against one order per launch
    (PB200_NO_TAYLOR_DEFER=1) and against the oracle: coefficients bit-identical, same order and norms, for stop
    orders of either parity, substeps, and a series that runs into max_order (same error, propagator.hpp:87-89)."""
    from oracle import pyoracle

    model = dict(kind=1, extents=(5,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=6)
    run_kw = dict(init="localized", site=-1, m_init=5, m=2, q_nom=700, dt=0.05, rtol=rtol, max_order=max_order,
                  substeps=substeps, t_max=5.0, seed=7)
    monkeypatch.delenv("PB200_NO_TAYLOR_DEFER", raising=False)
    rp = _ctx(gpu, model).run(**run_kw)
    monkeypatch.setenv("PB200_NO_TAYLOR_DEFER", "1")
    rs = _ctx(gpu, model).run(**run_kw)
    monkeypatch.delenv("PB200_NO_TAYLOR_DEFER", raising=False)
    ro = port.model(pyoracle.ModelDef(**model)).run(**run_kw)
    if max_order == 9:  # rtol 1e-15 needs ~11 orders: every implementation must refuse with the reference's text
        for r in (rp, rs):
            with pytest.raises(gpu.PacesError, match="reduce dt"):
                r.step()
        with pytest.raises(Exception, match="reduce dt"):
            ro.step()
        return
    orders = set()
    for s in range(1, 13):
        dp, ds, do = rp.step(), rs.step(), ro.step()
        orders.add(dp["taylor_order"])
        assert dp["taylor_order"] == ds["taylor_order"] == do["taylor_order"], (s, dp, ds, do)
        for k in ("norm_pre", "norm_post", "energy", "discarded_weight", "delta_norm_expmv"):
            assert _close(dp[k], ds[k], 1e-13, 1e-14), (s, k, dp[k], ds[k])  # reduction shapes differ (grid sizes)
            assert _close(dp[k], do[k], 1e-10, 1e-13), (s, k, dp[k], do[k])
        (wp, cp), (ws, cs), (wo, co) = rp.state(), rs.state(), ro.state()
        assert np.array_equal(wp, ws) and np.array_equal(wp, wo), s
        assert cp.tobytes() == cs.tobytes() == co.tobytes(), s
    tp, ts = rp.times(), rs.times()
    assert ts["taylor_deferred"] == 0 and tp["taylor_orders"] == ts["taylor_orders"]
    if min(orders) >= 4:
        assert tp["taylor_deferred"] >= (tp["taylor_orders"] - 3 * 12 * substeps) // 2, (tp, orders)


def test_weight_histogram_against_oracle(gpu, port):
    """SURVEY 8f rank 1 (observables.hpp:123-176, test_observables.cpp:170-220), entirely on the device (hand-written
    radix sort, prefix sums, grid reduction): support, marks, sampled ranks and weights exact; tail slope to 1e-10."""
    from oracle import pyoracle

    case = CASES["disordered_L5_d6_optical"]
    ctx = _ctx(gpu, case["model"])
    run = ctx.run(**case["run"])
    for _ in range(12):
        run.step()
    _, c = run.state()
    rng = np.random.default_rng(3)
    big = (rng.standard_normal(200001) + 1j * rng.standard_normal(200001)) * np.exp(-9 * rng.random(200001))
    big[::11] = 0
    ties = np.repeat(np.array([0.5, 0.25, 0.125, 0.0625], np.complex128), 700)  # exact ties across several tiles
    for vec, resident in ((c, True), (big, False), (ties, False), (np.array([0, 3 + 4j, 0]), False)):
        for bins in (0, 1, 2, 50):
            want = pyoracle.weight_histogram(port, vec, bins)
            gots = [ctx.weight_histogram(vec, bins)] + ([run.weight_histogram(bins)] if resident else [])
            for got in gots:
                for k in want:
                    if k == "tail_exponent":
                        assert _close(got[k], want[k], 1e-10, 1e-12), (k, bins, got[k], want[k])
                        continue
                    same = (got[k].tobytes() == want[k].tobytes()) if hasattr(want[k], "tobytes") else got[k] == want[k]
                    assert same, (k, bins, got[k], want[k])
    with pytest.raises(gpu.PacesError, match="empty state"):
        ctx.weight_histogram(np.zeros(4, np.complex128))


def test_checkpoint_resume_roundtrip(gpu, port):
    """download (canonical order = checkpoint order, io.hpp:77-99), reload into a fresh context
    with pb200_run_load_state and continue: identical to the uninterrupted run."""
    case = CASES["disordered_L5_d6_optical"]
    ctx = _ctx(gpu, case["model"])
    run = ctx.run(**case["run"])
    for _ in range(10):
        run.step()
    w, c = run.state()
    _, _, t, sd = run.info()
    cont = [run.step() for _ in range(10)]
    w_end, c_end = run.state()
    ctx2 = _ctx(gpu, case["model"])
    kw = {k: v for k, v in case["run"].items() if k not in ("init", "site")}
    run2 = ctx2.load_state(w, c, t=t, steps_done=sd, **kw)
    resumed = [run2.step() for _ in range(10)]
    w2, c2 = run2.state()
    assert resumed == cont
    assert w2.tobytes() == w_end.tobytes() and c2.tobytes() == c_end.tobytes()


def test_host_step_operator(gpu, port):
    """paces::step on host buffers (pb200_step) and its overlapped-transfer form (pb200_step_io) against the oracle."""
    from oracle.pyoracle import ModelDef

    case = CASES["cfg2_layout_L16_d16_small"]
    ctx = _ctx(gpu, case["model"])
    ro = port.model(ModelDef(**case["model"])).run(**case["run"])
    for _ in range(5):
        ro.step()
    kw = {k: v for k, v in case["run"].items() if k not in ("init", "site")}
    ow = np.zeros(200000 * ctx.words, np.uint32)
    oc = np.zeros(200000, np.complex128)
    for s in range(6, 12):
        w, c = ro.state()
        t = ro.info()[2]
        a = ctx.step(w, c, t, s, **kw)
        b = ctx.step(w, c, t, s, out_words=ow, out_coeff=oc, **kw)
        do = ro.step()
        wo, co = ro.state()
        for got in (a, b):
            assert np.array_equal(got[0], wo) and got[1].tobytes() == co.tobytes(), s
            _check_diag(got[2], do, "host_step", s)
    with pytest.raises(gpu.PacesError, match="must be sorted"):
        ctx.step(w[::-1].copy(), c, t, 12, out_words=ow, out_coeff=oc, **kw)
    with pytest.raises(gpu.PacesError, match="too small"):
        ctx.step(w, c, t, 12, out_words=ow[: 10 * ctx.words], out_coeff=oc[:10], **kw)
    # the context is still usable after the failures
    assert np.array_equal(ctx.step(w, c, t, 12, **kw)[0], ctx.step(w, c, t, 12, out_words=ow, out_coeff=oc, **kw)[0])


def test_host_step_reuses_resident_space_only_when_input_matches(gpu, port):
    """pb200_step_io keeps its last result resident.  When the caller hands that very state back (verified on the
    device, bit for bit) the step reuses the resident H_eff and takes the incremental adapt path; any difference in
    the coefficients or the keys must be honoured -- the step is redone from the caller's buffers.  Every result is
    compared with the oracle stepping from exactly the state that was passed in."""
    from oracle.pyoracle import ModelDef

    case = CASES["cfg2_layout_L16_d16_small"]
    ctx = _ctx(gpu, case["model"])
    om = port.model(ModelDef(**case["model"]))
    ro = om.run(**case["run"])
    for _ in range(5):
        ro.step()
    kw = {k: v for k, v in case["run"].items() if k not in ("init", "site")}
    cap = 400000
    bufs = [(np.zeros(cap * ctx.words, np.uint32), np.zeros(cap, np.complex128)) for _ in range(2)]
    w, c = ro.state()
    t = ro.info()[2]
    # chain: feed the result back in, six times
    inc0 = ctx.adapt_stats()["incremental_steps"]
    for k, s in enumerate(range(6, 12)):
        ow, oc, d = ctx.step(w, c, t, s, out_words=bufs[k & 1][0], out_coeff=bufs[k & 1][1], **kw)
        do = ro.step()
        wo, co = ro.state()
        assert np.array_equal(ow, wo) and oc.tobytes() == co.tobytes(), s
        _check_diag(d, do, "step_io chain", s)
        w, c, t = ow, oc, d["t"]
    assert ctx.adapt_stats()["incremental_steps"] - inc0 >= 4  # all but the first call reuse the resident space
    w, c = np.array(w, copy=True), np.array(c, copy=True)  # the results above live in the output buffers

    def oracle_step(words, coeff, tt, s):
        kept = om.truncate_select(words, coeff, kw["q_nom"], port.mix_seed(kw["seed"] + s))
        tw, rp, col, val = om.grow(kept, kw["m"])
        psi, disc = om.remap(words, coeff, tw)
        from oracle.pyoracle import expmv

        psi2, order, _ = expmv(port, rp, col, val, psi, dt=kw["dt"], rtol=kw["rtol"], max_order=200, substeps=1)
        return tw, psi2, order

    # (a) same shape, one coefficient changed: the resident copy must NOT be used
    c_mod = np.array(c, copy=True)
    c_mod[len(c_mod) // 3] *= 0.5
    ow, oc, d = ctx.step(w, c_mod, t, 12, out_words=bufs[0][0], out_coeff=bufs[0][1], **kw)
    tw, psi, order = oracle_step(w, c_mod, t, 12)
    assert np.array_equal(ow, tw) and oc.tobytes() == psi.tobytes() and d["taylor_order"] == order
    # (b) the unmodified state again right after: the resident state is now the result of (a), so this is a miss too
    ow, oc, d = ctx.step(w, c, t, 12, out_words=bufs[1][0], out_coeff=bufs[1][1], **kw)
    tw, psi, order = oracle_step(w, c, t, 12)
    assert np.array_equal(ow, tw) and oc.tobytes() == psi.tobytes() and d["taylor_order"] == order
    # (c) feed (b)'s result back (a hit), then the same call with ONE key replaced by another sorted, valid key
    w1, c1, t1 = np.array(ow, copy=True), np.array(oc, copy=True), d["t"]
    ow, oc, d = ctx.step(w1, c1, t1, 13, out_words=bufs[0][0], out_coeff=bufs[0][1], **kw)
    tw, psi, order = oracle_step(w1, c1, t1, 13)
    assert np.array_equal(ow, tw) and oc.tobytes() == psi.tobytes()
    w2, c2, t2 = np.array(ow, copy=True), np.array(oc, copy=True), d["t"]
    w_bad = np.array(w2, copy=True)
    L, d_pho = case["model"]["extents"][0], case["model"]["d_pho"]
    cand = ctx.pack([L - 1] + [d_pho - 1] * L)  # the largest key of the layout: the table stays sorted and unique
    assert tuple(cand) > tuple(w_bad[-1])
    w_bad[-1] = cand
    ow, oc, d = ctx.step(w_bad, c2, t2, 14, out_words=bufs[1][0], out_coeff=bufs[1][1], **kw)
    tw, psi, order = oracle_step(w_bad, c2, t2, 14)
    assert np.array_equal(ow, tw) and oc.tobytes() == psi.tobytes() and d["taylor_order"] == order


@pytest.mark.gpu
def test_large_neighbour_order_takes_the_full_path(gpu, port):
    """Round-1 advice: the incremental adapt path keeps BFS distances in bytes, so m >= 255 must take the full path
    (the reference puts no bound on m; a large m means growth to closure on a small model).  m = 300 and m = 255
    against the oracle, step by step."""
    from oracle import pyoracle

    model = dict(kind=1, extents=(3,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(0.7,), d_pho=3)
    for m in (255, 300):
        run_kw = dict(init="localized", site=-1, m_init=m, m=m, q_nom=40, dt=0.05, rtol=1e-15, t_max=1.0, seed=3)
        rg = _ctx(gpu, model).run(**run_kw)
        ro = port.model(pyoracle.ModelDef(**model)).run(**run_kw)
        for s in range(1, 7):
            dg, do = rg.step(), ro.step()
            (wg, cg), (wo, co) = rg.state(), ro.state()
            assert np.array_equal(wg, wo), (m, s)
            assert cg.tobytes() == co.tobytes(), (m, s)
            assert dg["q_true"] == do["q_true"] == 81, (m, s, dg, do)  # 3 sites x 3^3 phonon configurations: closure
        assert rg.adapt_stats()["incremental_steps"] == 0


@pytest.mark.gpu
def test_step_io_rejects_overlapping_buffers(gpu):
    """Round-1 advice: pb200_step_io reads its inputs while it writes its outputs; in-place calls are refused."""
    case = CASES["disordered_L5_d6_optical"]
    ctx = _ctx(gpu, case["model"])
    run = ctx.run(**case["run"])
    for _ in range(4):
        run.step()
    w, c = run.state()
    _, _, t, sd = run.info()
    kw = {k: v for k, v in case["run"].items() if k not in ("init", "site")}
    cap = 4 * len(c)
    bw = np.zeros(cap * ctx.words, np.uint32)
    bc = np.zeros(cap, np.complex128)
    bw[: w.size] = w.ravel()
    bc[: len(c)] = c
    with pytest.raises(Exception, match="must not overlap"):
        ctx.step(bw[: w.size], bc[: len(c)], t, sd + 1, out_words=bw, out_coeff=bc, **kw)
    ow, oc = np.zeros_like(bw), np.zeros_like(bc)
    dr = run.step()  # (the host-buffer step below replaces this context's resident state)
    wr, cr = run.state()
    w2, c2, d = ctx.step(bw[: w.size], bc[: len(c)], t, sd + 1, out_words=ow, out_coeff=oc, **kw)
    assert np.array_equal(w2, wr) and c2.tobytes() == cr.tobytes() and d["q_true"] == dr["q_true"]
