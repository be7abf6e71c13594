"""Pins the CPU restatement (oracle/paces_oracle.cpp): bit-for-bit against the committed golden fixtures
(generated from the unmodified reference by tests/golden/make_golden.py) and, where oracle/_ref exists,
against the reference itself on fresh inputs.  No GPU needed."""
import numpy as np
import pytest

from cases import CASES
from oracle import pyoracle
from oracle.pyoracle import ModelDef, csr_expectation, csr_matvec, expmv, fnv1a64, state_norm


def _snap(run, d):
    w, c = run.state()
    rp, col, val = run.csr()
    return dict(diag=d, nnz=int(rp[-1]), table=fnv1a64(w), coeff=fnv1a64(c), row_ptr=fnv1a64(rp), col=fnv1a64(col),
                val=fnv1a64(val))


@pytest.mark.parametrize("name", list(CASES))
def test_port_trajectory_matches_golden(port, golden, name):
    case, g = CASES[name], golden[name]
    m = port.model(ModelDef(**case["model"]))
    assert dict(sites=m.layout_sites, words=m.words, bits=m.total_bits, terms=m.n_terms) == g["layout"]
    run = m.run(**case["run"])
    rows, nnz, _, _ = run.info()
    w, c = run.state()
    assert (rows, nnz, fnv1a64(w), fnv1a64(c)) == (g["init"]["q_true"], g["init"]["nnz"], g["init"]["table"], g["init"]["coeff"])
    for s in range(1, case["steps"] + 1):
        d = run.step()
        if str(s) in g["snaps"]:
            assert _snap(run, d) == g["snaps"][str(s)], f"{name} step {s}"
    ob = run.observe()
    fo = g["final_observe"]
    assert [ob["amp"].real, ob["amp"].imag] == fo["amp"]
    assert [float(x) for x in ob["density"]] == fo["density"]
    for k in ("norm", "energy", "rmsd", "xbar"):
        assert ob[k] == fo[k], k


def test_port_apply_terms_and_grow_match_golden(port, golden_small):
    gs = golden_small
    m = port.model(ModelDef(**CASES["disordered_4x3_d7"]["model"]))
    off = 0
    for i, src in enumerate(gs["apply_src"]):
        keys, amps = m.apply_terms(src)
        n = int(gs["apply_counts"][i])
        assert np.array_equal(keys, gs["apply_keys"][off:off + n])
        assert amps.tobytes() == gs["apply_amps"][off:off + n].tobytes()
        off += n
    tw, rp, col, val = m.grow(gs["grow_seeds"], 2)
    assert np.array_equal(tw, gs["grow_table"]) and np.array_equal(rp, gs["grow_row_ptr"])
    assert np.array_equal(col, gs["grow_col"]) and val.tobytes() == gs["grow_val"].tobytes()


def test_port_selection_ties_match_golden(port, golden_small):
    gs = golden_small
    m = port.model(ModelDef(kind=1, extents=(3,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(0.5,), d_pho=2))
    seen = set()
    for seed in range(16):
        kept = m.truncate_select(gs["sel_words"], gs["sel_coeff"], 3, seed)
        assert np.array_equal(kept, gs["sel_kept_%d" % seed])
        seen.add(kept.tobytes())
    assert len(seen) > 1  # the seed really chooses among the four tied keys


def test_codec_known_answers(port):
    # basis_codec worked example (test_basis_codec.cpp:17-34): dims (8,8,2,2,2048,16) -> 0x6001,0x020F style
    # layouts are exercised through uint32 words here: straddling 7-bit sites and exhaustive round trips.
    m = port.model(ModelDef(kind=1, extents=(5,), d_pho=100))  # 3 + 5*7 = 38 bits, sites straddle word 0/1
    assert (m.words, m.total_bits) == (2, 38)
    rng = np.random.RandomState(1)
    for _ in range(2000):
        occ = np.concatenate([[rng.randint(5)], rng.randint(0, 100, 5)]).astype(np.uint32)
        w = m.pack(occ)
        assert np.array_equal(m.unpack(w), occ)
        assert w[1] & ((1 << (64 - 38)) - 1) == 0  # padding bits stay clean (test_basis_codec.cpp:113-124)
    # order compatibility: lexicographic order of words == lexicographic order of occupations (:97-111)
    occs = np.stack([np.concatenate([[rng.randint(5)], rng.randint(0, 100, 5)]) for _ in range(500)]).astype(np.uint32)
    words = np.stack([m.pack(o) for o in occs])
    assert np.array_equal(np.lexsort(words.T[::-1]), np.lexsort(occs.T[::-1]))
    with pytest.raises(Exception, match="out of range"):
        m.pack([5, 0, 0, 0, 0, 0])
    with pytest.raises(Exception, match="corrupt row"):
        m.unpack(np.array([0xFFFFFFFF, 0xFC000000], np.uint32))


def test_ladder_elements_exact(port):
    # test_lattice_models.cpp:71-85: shifted-oscillator ladder elements g*sqrt(n+1), cutoff drops raising (:119-141)
    m = port.model(ModelDef(kind=1, extents=(1,), eps=(0.0,), hop=(), omega=(1.0,), g=(2.5,), d_pho=6))
    for n in range(6):
        keys, amps = m.apply_terms(m.pack([0, n]))
        got = {int(m.unpack(k)[1]): a for k, a in zip(keys, amps)}
        want = {}
        if n + 1 < 6:
            want[n + 1] = 2.5 * np.sqrt(float(n + 1))
        if n >= 1:
            want[n - 1] = 2.5 * np.sqrt(float(n))
        if n > 0:
            want[n] = 1.0 * n
        assert got == want


def test_expmv_errors_and_identity(port):
    rp = np.array([0, 0, 0], np.int64)
    c, order, last = expmv(port, rp, np.zeros(0, np.int32), np.zeros(0), np.array([1.0, 2.0j]))
    assert order <= 2 and np.array_equal(c, np.array([1.0, 2.0j]))  # H = 0 (test_propagator.cpp:31-41)
    rp = np.array([0, 1], np.int64)
    with pytest.raises(Exception, match="reduce dt"):  # test_propagator.cpp:157-169
        expmv(port, rp, np.array([0], np.int32), np.array([1e6]), np.array([1.0 + 0j]), dt=1.0, max_order=20)
    with pytest.raises(Exception, match="non-finite"):
        expmv(port, rp, np.array([0], np.int32), np.array([1.0]), np.array([np.nan + 0j]))
    # diagonal phase (test_propagator.cpp:43-54)
    c, order, _ = expmv(port, rp, np.array([0], np.int32), np.array([0.7]), np.array([1.0 + 0j]), dt=0.3)
    assert abs(c[0] - np.exp(-0.21j)) < 1e-15


def test_memory_cap_message(port, monkeypatch):
    m = port.model(ModelDef(**CASES["cfg1_holstein_L4_d8"]["model"]))
    monkeypatch.setenv("PACES_MAX_MEMORY_BYTES", "1000")
    with pytest.raises(Exception, match="memory cap"):
        m.run(**CASES["cfg1_holstein_L4_d8"]["run"])


# ---------------------------------------------------------------------------------------------------------
# port vs the reference itself, fresh random inputs (only where oracle/_ref was built)
# ---------------------------------------------------------------------------------------------------------
def _random_state(m, run_kw, steps):
    run = m.run(**run_kw)
    for _ in range(steps):
        run.step()
    return run


@pytest.mark.parametrize("name", ["disordered_4x3_d7", "cube_2x2x2_d16", "tb_chain_31"])
def test_port_vs_reference_functions(port, ref, name):
    if ref is None:
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    case = CASES[name]
    mp, mr = port.model(ModelDef(**case["model"])), ref.model(ModelDef(**case["model"]))
    rr = _random_state(mr, case["run"], 6)
    w, c = rr.state()
    rp, col, val = rr.csr()
    rng = np.random.RandomState(0)
    x = rng.uniform(-1, 1, len(c)) + 1j * rng.uniform(-1, 1, len(c))
    assert csr_matvec(port, rp, col, val, x).tobytes() == csr_matvec(ref, rp, col, val, x).tobytes()
    assert csr_expectation(port, rp, col, val, x) == csr_expectation(ref, rp, col, val, x)
    a, b = expmv(port, rp, col, val, c), expmv(ref, rp, col, val, c)
    assert a[0].tobytes() == b[0].tobytes() and a[1:] == b[1:]
    assert state_norm(port, x) == state_norm(ref, x)
    assert mp.exciton_density(w, c).tobytes() == mr.exciton_density(w, c).tobytes()
    assert mp.dipole_amplitude(w, c) == mr.dipole_amplitude(w, c)
    if case["model"]["kind"] == 1:
        assert mp.phonon_numbers(w, c).tobytes() == mr.phonon_numbers(w, c).tobytes()
    for bins in (0, 1, 17):  # weight_histogram, observables.hpp:123-176 (test_observables.cpp:170-220)
        a, b = pyoracle.weight_histogram(port, c, bins), pyoracle.weight_histogram(ref, c, bins)
        assert all((a[k].tobytes() == b[k].tobytes()) if hasattr(a[k], "tobytes") else a[k] == b[k] for k in a)
    for q in (1, 7, len(c) // 3, len(c)):
        for seed in (0, 5):
            assert np.array_equal(mp.truncate_select(w, c, q, seed), mr.truncate_select(w, c, q, seed))
    kept = mr.truncate_select(w, c, max(1, len(c) // 4), 1)
    for order in (0, 1, 2):
        gp, gr = mp.grow(kept, order), mr.grow(kept, order)
        for u, v in zip(gp, gr):
            assert u.tobytes() == v.tobytes()
    tw = mr.grow(kept, 1)[0]
    (cp, dp), (cr, dr) = mp.remap(w, c, tw), mr.remap(w, c, tw)
    assert cp.tobytes() == cr.tobytes() and dp == dr
    for i in rng.randint(0, len(w), 50):
        kp, kr = mp.apply_terms(w[i]), mr.apply_terms(w[i])
        assert np.array_equal(kp[0], kr[0]) and kp[1].tobytes() == kr[1].tobytes()


def test_reference_run_loop_equals_stepwise_driver(ref):
    """ref_shim's po_run_step restates run()'s loop body; check it against the reference's own run()."""
    if ref is None:
        pytest.skip("oracle/_ref not built")
    case = CASES["ties_holstein_L5_d6"]
    m = ref.model(ModelDef(**case["model"]))
    diags, final, err = m.run_all(**case["run"])
    assert err == "" and len(diags) == case["steps"]
    run = m.run(**case["run"])
    for s in range(case["steps"]):
        assert run.step() == diags[s]
    assert run.state()[0].tobytes() == final.state()[0].tobytes()
    assert run.state()[1].tobytes() == final.state()[1].tobytes()
