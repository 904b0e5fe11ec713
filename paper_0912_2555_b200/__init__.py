"""B200-native MAP accepting-cycle detection (arXiv 0912.2555, DiVinE CUDA).

The hot path — CSR build, (max, vertex-id) propagation to fixpoint, witness
detection and demotion, the iteration loop — runs as hand-written sm_100a
kernels behind the C ABI in include/cycheck_b200.h. This package is the thin
host mirror of the reference interface (cycheck::build_snapshot, run_map, …).
"""
from .api import *  # noqa: F401,F403
from .api import __all__  # noqa: F401
from ._abi import EXPORTED_SYMBOLS, LIB_PATH, GenParams, preset, prepare  # noqa: F401

__version__ = "0.1.0"
