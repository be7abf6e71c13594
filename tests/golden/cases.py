"""Named model / run configurations shared by the golden generator and the parity tests.

Each case is (ModelDef kwargs, run kwargs, number of steps, steps at which a snapshot is hashed).
Sizes are chosen so the CPU checkers finish each case in about a second.
"""
import numpy as np

_rng = np.random.RandomState(20260307)


def _r(n, lo, hi):
    return tuple(float(x) for x in _rng.uniform(lo, hi, n))


CASES = {
    # BASELINE config 1 / SURVEY App. B: 1D Holstein L=4, d_pho=8, localized centre start
    "cfg1_holstein_L4_d8": dict(
        model=dict(kind=1, extents=(4,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=8),
        run=dict(init="localized", site=-1, m_init=6, m=2, q_nom=2000, dt=0.05, rtol=1e-15, t_max=5.0, seed=7),
        steps=100, snaps=(1, 2, 10, 25, 50, 100)),
    # symmetric chain: exact weight ties at the cutoff exercise the seeded Fisher-Yates path
    "ties_holstein_L5_d6": dict(
        model=dict(kind=1, extents=(5,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=6),
        run=dict(init="localized", site=-1, m_init=6, m=2, q_nom=300, dt=0.05, rtol=1e-15, t_max=5.0, seed=7),
        steps=100, snaps=(2, 20, 60, 100)),
    # fully disordered 1D chain, optical start (SURVEY App. C.1 model)
    "disordered_L5_d6_optical": dict(
        model=dict(kind=1, extents=(5,), eps=(0.13, -0.2, 0.05, 0.3, -0.11), hop=(0.55, 0.5, 0.6, 0.45),
                   omega=(1.0, 0.97, 1.03, 0.99, 1.01), g=(0.71, 0.65, 0.8, 0.75, 0.6), d_pho=6),
        run=dict(init="optical", m_init=4, m=2, q_nom=400, dt=0.05, rtol=1e-15, t_max=3.0, seed=11),
        steps=60, snaps=(1, 2, 30, 60)),
    # 2D 3x3 with straddling registers (d_pho=5 -> 3-bit sites, 4+27=31 bits) -- single word
    "square_3x3_d5": dict(
        model=dict(kind=1, extents=(3, 3), eps=(0.0,), hop=(-0.55,), omega=(1.0,), g=(0.71,), d_pho=5),
        run=dict(init="optical", m_init=4, m=2, q_nom=500, dt=0.05, rtol=1e-15, t_max=2.0, seed=3),
        steps=40, snaps=(1, 2, 20, 40)),
    # 3D 2x2x2, d_pho=16 -> 3+32=35 bits, two words, register straddles the word boundary
    "cube_2x2x2_d16": dict(
        model=dict(kind=1, extents=(2, 2, 2), eps=(0.0,), hop=(0.55,), omega=(1.0,), g=(0.71,), d_pho=16),
        run=dict(init="localized", site=-1, m_init=4, m=2, q_nom=600, dt=0.05, rtol=1e-15, t_max=2.0, seed=5),
        steps=40, snaps=(1, 2, 20, 40)),
    # disordered 2D 4x3, d_pho=7: 4 + 12*3 = 40 bits, two words
    "disordered_4x3_d7": dict(
        model=dict(kind=1, extents=(4, 3), eps=_r(12, -0.3, 0.3), hop=_r(17, 0.3, 0.8), omega=_r(12, 0.9, 1.1),
                   g=_r(12, 0.4, 0.9), d_pho=7),
        run=dict(init="localized", site=5, m_init=3, m=2, q_nom=700, dt=0.04, rtol=1e-15, t_max=1.2, seed=99),
        steps=30, snaps=(1, 2, 15, 30)),
    # wide key: 1D L=16, d_pho=16 (BASELINE config 2 layout, 68 bits, three words) at a small q_nom
    "cfg2_layout_L16_d16_small": dict(
        model=dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16),
        run=dict(init="localized", site=-1, m_init=4, m=2, q_nom=1500, dt=0.05, rtol=1e-15, t_max=1.0, seed=7),
        steps=20, snaps=(1, 2, 10, 20)),
    # tight binding chain (no phonon registers), ballistic spreading
    "tb_chain_31": dict(
        model=dict(kind=0, extents=(31,), eps=(0.0,), hop=(1.0,), omega=(), g=(), d_pho=1),
        run=dict(init="localized", site=-1, m_init=2, m=2, q_nom=40, dt=0.05, rtol=1e-15, t_max=2.0, seed=1),
        steps=40, snaps=(1, 2, 20, 40)),
    # substeps > 1 and m = 1
    "substeps_L4_d4_m1": dict(
        model=dict(kind=1, extents=(4,), eps=(0.2,), hop=(0.8,), omega=(1.0,), g=(1.3,), d_pho=4),
        run=dict(init="localized", site=0, m_init=3, m=1, q_nom=60, dt=0.1, rtol=1e-14, substeps=3, t_max=2.0, seed=2),
        steps=20, snaps=(1, 2, 10, 20)),
}
