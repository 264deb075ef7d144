"""The C-ABI boundary: the library loads, exports every symbol include/pppc_b200.h
declares, and fails loudly (no CPU fallback) when no B200 is present.  CPU only."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1905_13076_b200 as ps
from paper_1905_13076_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "pppc_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ps_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = C.CDLL(_abi.LIB_PATH)
    declared = declared_symbols()
    assert len(declared) >= 35
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(_abi.EXPORTED), set(declared) ^ set(_abi.EXPORTED)


def test_struct_layouts_match_header():
    assert C.sizeof(_abi.ps_problem_desc) == 144
    assert C.sizeof(_abi.ps_batch_status) == 72
    assert C.sizeof(_abi.ps_newton_settings) == 32
    # + final_defect, then the per-iteration COCG / fine / spectral arrays
    assert C.sizeof(_abi.ps_history) == 8 + 8 * 256 + 4 * 8 + 4 * 8 + 8 + 8 + 3 * 8 * 256
    assert C.sizeof(_abi.ps_krylov_settings) == 16


def test_default_settings_are_reference_defaults():
    s = _abi.ps_solver_settings()
    assert _abi.lib().ps_default_settings(C.byref(s)) == 0
    assert (s.newton.tol_abs, s.newton.tol_rel, s.newton.max_iter, s.newton.damping) == (1e-9, 1e-8, 30, 1.0)
    assert s.newton.line_search == 0


def test_last_engine_needs_a_context():
    e = C.c_int32(-1)
    assert _abi.lib().ps_last_engine(None, C.byref(e), None, None) == _abi.PS_ERR_BAD_ARG
    assert e.value == -1


def _has_gpu():
    name = C.create_string_buffer(64)
    return _abi.lib().ps_device_info(name, 64, None, None, None) == 0


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_device():
    p = ps.build_dae_pair()
    with pytest.raises(ps.ParasteadyError) as e:
        ps.Propagator(p, ps.TimeMesh(4, 1, p.period))
    assert e.value.code == _abi.PS_ERR_CUDA and "no CPU fallback" in str(e.value)
    with pytest.raises(ps.ParasteadyError):
        ps.forward_dft(np.ones((4, 1)))
