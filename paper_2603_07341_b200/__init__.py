"""paces-b200: B200-native adapt-evolve-truncate timestep of paces (arXiv 2603.07341).

The product is ``libpaces_b200.so`` (hand-written sm_100a CUDA behind the C ABI of ``include/paces_b200.h``);
this package is its thin ctypes mirror of the reference's operator API.  There is no CPU fallback: creating a
:class:`Context` without a CUDA device raises.
"""
from .api import (Context, Diag, ModelDef, PacesError, PhaseTimes, Run, csr_expectation, csr_matvec, expmv,  # noqa: F401
                  lib_path, load_library, state_norm, EXPORTED_SYMBOLS)

__all__ = ["Context", "Diag", "ModelDef", "PacesError", "PhaseTimes", "Run", "csr_expectation", "csr_matvec", "expmv",
           "lib_path", "load_library", "state_norm", "EXPORTED_SYMBOLS"]
