import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


def _have_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _have_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def port():
    """The CPU restatement (oracle/libpaces_oracle.so); built on demand."""
    from oracle import pyoracle

    if not os.path.exists(pyoracle.PORT_LIB):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "port"])
    return pyoracle.load_port()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference behind ref_shim.cpp; None where it was never built."""
    from oracle import pyoracle

    if not os.path.exists(pyoracle.REF_LIB) and os.path.exists("/root/reference/proj/include/paces/engine.hpp"):
        subprocess.call(["make", "-C", os.path.join(ROOT, "oracle"), "ref"])
    if not os.path.exists(pyoracle.REF_LIB):
        return None
    return pyoracle.load_reference()


@pytest.fixture(scope="session")
def golden():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_small():
    import numpy as np

    return np.load(os.path.join(ROOT, "tests", "golden", "golden_small.npz"))
