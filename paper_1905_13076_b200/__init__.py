"""B200-native PP-PC hot path (periodic Parareal with a multiharmonic coarse solver).

The compute path is libpppc_b200.so (CUDA sm_100a kernels behind the C ABI in
include/pppc_b200.h); this package is the thin host-side mirror of the
reference's propagator / PP-PC interface (see api.py).
"""
from .api import *  # noqa: F401,F403
from .api import ParasteadyError, PeriodicProblem, Propagator, TimeMesh  # noqa: F401
from ._abi import EXPORTED, LIB_PATH, lib  # noqa: F401
