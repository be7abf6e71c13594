"""GPU tests that mirror the reference's oracle-free / dense-oracle acceptance checks, run through
the C ABI on the B200: dense exponential fidelity on a fully covered space, symmetry and conservation laws.  The
dense oracle of the reference (oracle.hpp, Eigen) is restated with numpy/scipy on the CSR the library returns for
the full space -- that CSR is itself pinned bit for bit to the reference by test_gpu_parity.py."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import paper_2603_07341_b200 as pb

    return pb


def _ctx(gpu, **kw):
    return gpu.Context(gpu.ModelDef(**kw))


def _full_space(ctx, seed_occ):
    """grow_subspace far enough to cover the whole sector: table + dense H (test_propagator.cpp:23-27)."""
    import scipy.sparse as sp

    seed = ctx.pack(seed_occ).reshape(1, -1)
    tw, rp, col, val = ctx.grow(seed, 64)
    h = sp.csr_matrix((val, col, rp), shape=(len(tw), len(tw))).toarray()
    return tw, h


def test_run_matches_dense_exponential(gpu):
    """test_engine.cpp:162-186 / acceptance C1: with q_nom >= the full dimension the trajectory is exact dynamics;
    fidelity with exp(-iHt) psi0 from a dense eigendecomposition >= 1 - 1e-10, discarded weight exactly 0."""
    model = dict(kind=1, extents=(3,), eps=(0.1, -0.05, 0.2), hop=(0.55,), omega=(1.0,), g=(0.71,), d_pho=6)
    ctx = _ctx(gpu, **model)
    tw, h = _full_space(ctx, [1, 0, 0, 0])
    dim = 3 * 6 ** 3
    assert len(tw) == dim and np.array_equal(h, h.T)
    lam, v = np.linalg.eigh(h)
    run = ctx.run(init="localized", site=1, m_init=40, m=2, q_nom=dim, dt=0.05, rtol=1e-15, t_max=10.0, seed=1)
    w0, c0 = run.state()
    assert np.array_equal(w0, tw)  # m_init covers the sector: same canonical table
    for s in range(1, 101):
        d = run.step()
        assert d["discarded_weight"] == 0.0  # test_engine.cpp:188-204
        assert abs(d["delta_norm_expmv"]) <= 1e-12 and 3 <= d["taylor_order"] <= 40  # acceptance C2
    w, c = run.state()
    assert np.array_equal(w, tw)
    exact = v @ (np.exp(-1j * lam * 5.0) * (v.T @ c0))
    fidelity = abs(np.vdot(exact, c)) ** 2
    assert fidelity >= 1 - 1e-10, fidelity
    # energy conserved to 1e-10 relative (test_observables.cpp:109-121)
    e0 = np.real(np.vdot(c0, h @ c0))
    e1 = np.real(np.vdot(c, h @ c))
    assert abs(e1 - e0) <= 1e-10 * max(1.0, abs(e0))


def test_hop_sign_invariance_and_sector_conservation(gpu):
    """acceptance C4 / test_engine.cpp:258-298: J -> -J leaves the site populations of a bipartite lattice unchanged
    (<= 1e-10), and the one-exciton sector is conserved: sum of the density equals the squared norm (1e-13)."""
    dens = {}
    for j in (0.55, -0.55):
        ctx = _ctx(gpu, kind=1, extents=(5,), eps=(0.0,), hop=(j,), omega=(1.0,), g=(0.71,), d_pho=6)
        run = ctx.run(init="localized", site=-1, m_init=6, m=2, q_nom=400, dt=0.05, rtol=1e-15, t_max=3.0, seed=3)
        rows = []
        for s in range(40):
            run.step()
            o = run.observe()
            assert abs(o["density"].sum() - o["norm"] ** 2) <= 1e-13  # test_observables.cpp:73-86
            rows.append(o["density"].copy())
        dens[j] = np.array(rows)
    assert np.max(np.abs(dens[0.55] - dens[-0.55])) <= 1e-10


def test_dipole_amplitude_of_optical_state_and_monomer_phase(gpu):
    """test_observables.cpp:123-154: the optical state has autocorrelation amplitude 1 at t = 0; a single uncoupled
    site evolves with the pure phase exp(-i eps t) to 1e-12."""
    ctx = _ctx(gpu, kind=1, extents=(4,), eps=(0.0,), hop=(0.3,), omega=(1.0,), g=(0.5,), d_pho=4)
    run = ctx.run(init="optical", m_init=4, m=2, q_nom=200, dt=0.05, rtol=1e-15, t_max=1.0, seed=0)
    assert abs(run.observe()["amp"] - 1.0) <= 1e-14
    eps = 0.37
    mono = _ctx(gpu, kind=1, extents=(1,), eps=(eps,), hop=(0.0,), omega=(1.0,), g=(0.0,), d_pho=3)
    run = mono.run(init="optical", m_init=2, m=2, q_nom=10, dt=0.05, rtol=1e-15, t_max=2.0, seed=0)
    for s in range(1, 21):
        run.step()
        assert abs(run.observe()["amp"] - np.exp(-1j * eps * 0.05 * s)) <= 1e-12


def test_tight_binding_ballistic_spread(gpu):
    """test_engine.cpp:231-256 / acceptance C3 (shortened): free exciton on an open chain, rmsd against the dense
    propagator of the hopping matrix to 1e-8."""
    L, J = 41, 1.0
    ctx = _ctx(gpu, kind=0, extents=(L,), eps=(0.0,), hop=(J,))
    run = ctx.run(init="localized", site=-1, m_init=L, m=2, q_nom=L, dt=0.05, rtol=1e-15, t_max=4.0, seed=0)
    h = np.zeros((L, L))
    for a in range(L - 1):
        h[a, a + 1] = h[a + 1, a] = J
    lam, v = np.linalg.eigh(h)
    psi0 = np.zeros(L)
    psi0[L // 2] = 1.0
    x = np.arange(L)
    for s in range(1, 61):
        run.step()
        if s % 20 == 0:
            p = np.abs(v @ (np.exp(-1j * lam * 0.05 * s) * (v.T @ psi0))) ** 2
            rmsd = np.sqrt(np.sum(p * (x - L // 2) ** 2))
            o = run.observe()
            assert abs(o["rmsd"] - rmsd) <= 1e-8, (s, o["rmsd"], rmsd)
            assert np.max(np.abs(o["density"] - p)) <= 1e-10
