"""Acceptance criteria and the CLI front-end through the drop-in shim, on the GPU box.  The binaries are built in the
build container against the UNMODIFIED reference headers (oracle/Makefile: accept, cli) and read nothing from
/root/reference at run time.
  oracle/_ref/acceptance_b200  acceptance_main.cpp criteria 3, 6, 10 + test_engine.cpp tie-break statistic (10^4 seeds)
                               + checkpoint round trip / resume, written with the reference's unqualified calls
  oracle/_ref/paces_b200       `dynamics` / `spectrum` (proj/tools/paces.cpp:84-130, test_cli.cpp:139-154)"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ACCEPT = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")
CLI = os.path.join(ROOT, "oracle", "_ref", "paces_b200")

SMALL_HOLSTEIN = """
[model]
kind = holstein
extents = 3
eps = 0.0
J = 1.0
omega0 = 1.0
g = 1.0
d_pho = 4

[run]
initial = localized
m_init = 6
m = 2
q_nom = 64
dt = 0.05
t_max = 0.5
seed = 7
"""

SPECTRUM = """
[model]
kind = holstein
extents = 2 2
eps = 0.0
J = -0.55
omega0 = 1.0
g = 0.71
d_pho = 6

[run]
initial = optical
m_init = 4
m = 2
q_nom = 300
dt = 0.05
t_max = 4.0
seed = 3

[spectrum]
tau = 17.33
"""


@pytest.mark.gpu
def test_reference_acceptance_criteria_through_the_shim():
    if not os.path.exists(ACCEPT):
        pytest.skip("oracle/_ref/acceptance_b200 was not built (needs the reference headers at build time)")
    r = subprocess.run([ACCEPT], capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "all passed" in r.stdout


def _cli(args, cwd):
    r = subprocess.run([CLI] + args, capture_output=True, text=True, timeout=600, cwd=cwd)
    assert r.returncode == 0, (args, r.stdout[-2000:], r.stderr[-2000:])
    return r.stdout


@pytest.mark.gpu
def test_cli_dynamics_is_reproducible_and_equals_the_reference(tmp_path):
    """test_cli.cpp:139-154: the three output files exist and two runs are byte-identical; beyond the reference's own
    test, the GPU run's checkpoint is byte-identical to the CPU reference's (--cpu) and its CSVs agree field by field
    to 1e-12."""
    if not os.path.exists(CLI):
        pytest.skip("oracle/_ref/paces_b200 was not built (needs the reference headers at build time)")
    (tmp_path / "run.conf").write_text(SMALL_HOLSTEIN)
    base = ["dynamics", "--config", str(tmp_path / "run.conf"), "--deterministic"]
    out = _cli(base + ["--out", str(tmp_path / "out1")], tmp_path)
    assert "dynamics: 10 steps" in out
    _cli(base + ["--out", str(tmp_path / "out2")], tmp_path)
    _cli(base + ["--cpu", "--out", str(tmp_path / "cpu")], tmp_path)
    for name in ("observables.csv", "diagnostics.csv", "checkpoint.bin"):
        a, b = (tmp_path / "out1" / name).read_bytes(), (tmp_path / "out2" / name).read_bytes()
        assert len(a) > 0 and a == b, name
    assert (tmp_path / "out1" / "checkpoint.bin").read_bytes() == (tmp_path / "cpu" / "checkpoint.bin").read_bytes()
    for name in ("observables.csv", "diagnostics.csv"):
        ga = (tmp_path / "out1" / name).read_text().splitlines()
        ca = (tmp_path / "cpu" / name).read_text().splitlines()
        assert len(ga) == len(ca) and ga[0] == ca[0], name
        for lg, lc in zip(ga, ca):
            if lg.startswith("#") or not lg[:1].lstrip("-").isdigit():
                assert lg == lc, (name, lg, lc)
                continue
            for xg, xc in zip(lg.split(","), lc.split(",")):
                assert abs(float(xg) - float(xc)) <= 1e-12 * max(1.0, abs(float(xc))), (name, lg, lc)
    # resume: the second half of the run from the first half's checkpoint ends in the same bytes
    (tmp_path / "half.conf").write_text(SMALL_HOLSTEIN.replace("t_max = 0.5", "t_max = 0.25"))
    _cli(["dynamics", "--config", str(tmp_path / "half.conf"), "--out", str(tmp_path / "half")], tmp_path)
    _cli(["dynamics", "--config", str(tmp_path / "run.conf"), "--resume", str(tmp_path / "half" / "checkpoint.bin"),
          "--out", str(tmp_path / "rest")], tmp_path)
    assert (tmp_path / "rest" / "checkpoint.bin").read_bytes() == (tmp_path / "out1" / "checkpoint.bin").read_bytes()


@pytest.mark.gpu
def test_cli_spectrum_equals_the_reference(tmp_path):
    if not os.path.exists(CLI):
        pytest.skip("oracle/_ref/paces_b200 was not built (needs the reference headers at build time)")
    (tmp_path / "spec.conf").write_text(SPECTRUM)
    _cli(["spectrum", "--config", str(tmp_path / "spec.conf"), "--out", str(tmp_path / "gpu")], tmp_path)
    _cli(["spectrum", "--config", str(tmp_path / "spec.conf"), "--cpu", "--out", str(tmp_path / "cpu")], tmp_path)
    g = [ln for ln in (tmp_path / "gpu" / "spectrum.csv").read_text().splitlines() if ln and ln[0] != "#"]
    c = [ln for ln in (tmp_path / "cpu" / "spectrum.csv").read_text().splitlines() if ln and ln[0] != "#"]
    assert len(g) == len(c) > 10 and g[0] == c[0]
    for lg, lc in zip(g[1:], c[1:]):
        for xg, xc in zip(lg.split(","), lc.split(",")):
            assert abs(float(xg) - float(xc)) <= 1e-10 * max(1.0, abs(float(xc))), (lg, lc)
