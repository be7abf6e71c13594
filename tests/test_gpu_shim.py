"""Drop-in proof on the GPU box: oracle/_ref/shim_parity (built in the build container from tests/cpp/shim_parity.cpp
against the UNMODIFIED reference headers) runs the reference's paces::run()/step()/free functions next to
paces::b200::* (include/paces_b200.hpp over libpaces_b200.so) and compares them.  The binary reads nothing from
/root/reference at run time."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_parity")


@pytest.mark.gpu
def test_cpp_shim_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/shim_parity was not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "all checks passed" in r.stdout


def test_shim_header_compiles_against_reference():
    """CPU-side: the shim header is source-compatible with the reference headers (syntax + types)."""
    ref = "/root/reference/proj/include"
    if not os.path.exists(os.path.join(ref, "paces", "engine.hpp")):
        pytest.skip("reference headers not present on this machine")
    src = '#include "paces/engine.hpp"\n#include "paces_b200.hpp"\nint main() { return 0; }\n'
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-fopenmp", "-I" + ref, "-I" + os.path.join(ROOT, "include"),
                        "-x", "c++", "-"], input=src, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
