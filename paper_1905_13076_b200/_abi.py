"""ctypes declarations of include/pppc_b200.h (the C ABI of libpppc_b200.so).

Loading is lazy; a missing shared library raises immediately (there is no CPU
fallback for the device path).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PPPC_LIB: load another build of the library (kernel-variant experiments)
LIB_PATH = os.environ.get("PPPC_LIB") or os.path.join(_HERE, "libpppc_b200.so")

PS_OK = 0
PS_ERR_BAD_ARG = 1
PS_ERR_NEWTON_MAXITER = 2
PS_ERR_NEWTON_DIVERGED = 3
PS_ERR_SINGULAR = 4
PS_ERR_PCG_MAXITER = 5
PS_ERR_NONFINITE = 6
PS_ERR_ODD_BLOCKS = 7
PS_ERR_SINGULAR_BLOCK = 8
PS_ERR_CONJ_SYMMETRY = 9
PS_ERR_CUDA = 10
PS_ERR_NOT_LINEAR = 11
PS_ERR_NOT_SETUP = 12
PS_ERR_COCG_MAXITER = 13
PS_ERR_WATCHDOG = 14
PS_MAX_HISTORY = 256

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int32)


class ps_curve(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("nu", C.c_double),
                ("k1", C.c_double), ("k2", C.c_double), ("k3", C.c_double)]


class ps_problem_desc(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("nnz", C.c_int32),
        ("row_ptr", ip), ("col_idx", ip), ("mass", dp), ("stiffness", dp),
        ("n_elem", C.c_int32), ("nodes_per_elem", C.c_int32),
        ("elem_nodes", ip), ("elem_stiff", dp), ("elem_inv_area", dp), ("elem_curve", ip),
        ("n_curves", C.c_int32), ("pad_", C.c_int32), ("curves", C.POINTER(ps_curve)),
        ("period", C.c_double), ("n_terms", C.c_int32), ("pad2_", C.c_int32),
        ("patterns", dp), ("amplitude", dp), ("frequency_hz", dp), ("phase_rad", dp),
    ]


class ps_time_mesh(C.Structure):
    _fields_ = [("subintervals", C.c_int32), ("fine_steps", C.c_int32), ("period", C.c_double)]


class ps_newton_settings(C.Structure):
    _fields_ = [("tol_abs", C.c_double), ("tol_rel", C.c_double), ("max_iter", C.c_int32),
                ("line_search", C.c_int32), ("damping", C.c_double)]


class ps_krylov_settings(C.Structure):
    _fields_ = [("tol_rel", C.c_double), ("max_iter", C.c_int32), ("warm_start", C.c_int32)]


class ps_solver_settings(C.Structure):
    _fields_ = [("newton", ps_newton_settings), ("pcg", ps_krylov_settings),
                ("cocg", ps_krylov_settings), ("max_batch", C.c_int32), ("engine", C.c_int32)]


class ps_batch_status(C.Structure):
    _fields_ = [("code", C.c_int32), ("failed_index", C.c_int32), ("t_next", C.c_double),
                ("residual", C.c_double), ("newton_iterations", C.c_int64),
                ("pcg_iterations", C.c_int64), ("max_newton_iterations", C.c_int32),
                ("max_pcg_iterations", C.c_int32), ("lockstep_pcg_iterations", C.c_int64),
                ("algorithmic_bytes", C.c_double), ("kernel_ms", C.c_double)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class ps_engine_settings(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iterations", C.c_int32),
                ("use_conjugate_symmetry", C.c_int32), ("bin_mask", ip),
                ("shift_kind", C.c_int32), ("pad_", C.c_int32)]


class ps_history(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32),
                ("jumps", C.c_double * PS_MAX_HISTORY),
                ("fine_ms", C.c_double), ("coarse_ms", C.c_double), ("spectral_ms", C.c_double),
                ("total_ms", C.c_double), ("fine_pcg_iterations", C.c_int64),
                ("coarse_pcg_iterations", C.c_int64), ("cocg_iterations", C.c_int64),
                ("newton_iterations", C.c_int64), ("fine_bytes", C.c_double),
                ("final_defect", C.c_double),
                ("cocg_per_iteration", C.c_int64 * PS_MAX_HISTORY),
                ("fine_ms_per_iteration", C.c_double * PS_MAX_HISTORY),
                ("spectral_ms_per_iteration", C.c_double * PS_MAX_HISTORY)]


class ps_polar_cable_params(C.Structure):
    _fields_ = [("nr", C.c_int32), ("ntheta", C.c_int32), ("radius", C.c_double),
                ("r_conductor", C.c_double), ("r_insulator", C.c_double),
                ("sigma_conductor", C.c_double), ("sigma_insulator", C.c_double),
                ("sigma_sheath", C.c_double), ("brauer_k1", C.c_double), ("brauer_k2", C.c_double),
                ("brauer_k3", C.c_double), ("linear_sheath", C.c_int32),
                ("return_in_sheath", C.c_int32), ("current", C.c_double),
                ("frequency_hz", C.c_double), ("ripple_terms", C.c_int32), ("pad_", C.c_int32),
                ("ripple_fraction", C.c_double), ("ripple_frequency_hz", C.c_double)]


class ps_radial_cable_params(C.Structure):
    _fields_ = [("n_r", C.c_int32), ("source_region", C.c_int32), ("r1", C.c_double),
                ("r2", C.c_double), ("r3", C.c_double), ("sigma_wire", C.c_double),
                ("sigma_sleeve", C.c_double), ("sigma_shield", C.c_double),
                ("brauer_k1", C.c_double), ("brauer_k2", C.c_double), ("brauer_k3", C.c_double),
                ("linear_sleeve", C.c_int32), ("pad_", C.c_int32), ("current", C.c_double),
                ("frequency_hz", C.c_double)]


vp = C.c_void_p
_SIGNATURES = {
    "ps_create": (C.c_int, [C.POINTER(ps_problem_desc), C.POINTER(ps_time_mesh),
                            C.POINTER(ps_solver_settings), vp, C.POINTER(vp)]),
    "ps_destroy": (None, [vp]),
    "ps_last_error": (C.c_char_p, [vp]),
    "ps_last_engine": (C.c_int, [vp, ip, ip, ip]),
    "ps_global_error": (C.c_char_p, []),
    "ps_dim": (C.c_int, [vp]),
    "ps_is_linear": (C.c_int, [vp]),
    "ps_create_frozen": (C.c_int, [vp, dp, C.POINTER(vp)]),
    "ps_default_settings": (C.c_int, [C.POINTER(ps_solver_settings)]),
    "ps_device_info": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                 C.POINTER(C.c_int)]),
    "ps_newton_step": (C.c_int, [vp, C.c_int32, dp, dp, C.c_double, dp, ip, dp,
                                 C.POINTER(ps_batch_status)]),
    "ps_fine_propagate_batch": (C.c_int, [vp, C.c_int32, C.c_int32, dp, dp, C.POINTER(ps_batch_status)]),
    "ps_fine_propagate_batch_dev": (C.c_int, [vp, C.c_int32, C.c_int32, vp, vp, C.POINTER(ps_batch_status)]),
    "ps_coarse_propagate_batch": (C.c_int, [vp, C.c_int32, C.c_int32, dp, dp, C.POINTER(ps_batch_status)]),
    "ps_coarse_propagate_batch_dev": (C.c_int, [vp, C.c_int32, C.c_int32, vp, vp,
                                                C.POINTER(ps_batch_status)]),
    "ps_coarse_sweep": (C.c_int, [vp, dp, C.POINTER(ps_batch_status)]),
    "ps_assemble_operators": (C.c_int, [vp, C.c_int32, dp, dp, dp]),
    "ps_eval_excitation": (C.c_int, [vp, C.c_int32, dp, dp]),
    "ps_mh_setup": (C.c_int, [vp, C.c_int32, ip, C.c_int32]),
    "ps_assemble_rhs": (C.c_int, [vp, dp, dp, dp]),
    "ps_mh_solve": (C.c_int, [vp, dp, dp, C.POINTER(ps_batch_status)]),
    "ps_pppc_correct": (C.c_int, [vp, dp, dp, dp, dp, C.POINTER(ps_batch_status)]),
    "ps_forward_dft": (C.c_int, [C.c_int32, C.c_int32, dp, dp]),
    "ps_inverse_dft": (C.c_int, [C.c_int32, C.c_int32, dp, dp]),
    "ps_jump_norm": (C.c_int, [C.c_int32, C.c_int32, dp, dp, dp]),
    "ps_eval_reluctivity": (C.c_int, [C.POINTER(ps_curve), C.c_int32, dp, dp, dp]),
    "ps_pppc_solve": (C.c_int, [vp, C.POINTER(ps_engine_settings), dp, dp, dp, C.POINTER(ps_history)]),
    "ps_fine_periodicity_defect": (C.c_int, [vp, dp, dp]),
    "ps_classic_parareal": (C.c_int, [vp, C.POINTER(ps_engine_settings), dp, dp, dp, C.POINTER(ps_history)]),
    "ps_pp_ic_solve": (C.c_int, [vp, C.POINTER(ps_engine_settings), dp, dp, C.POINTER(ps_history)]),
    "ps_sequential_steady_state": (C.c_int, [vp, C.c_double, C.c_int32, dp, ip, ip, dp]),
    "ps_polar_cable_defaults": (C.c_int, [C.POINTER(ps_polar_cable_params)]),
    "ps_build_polar_cable": (C.c_int, [C.POINTER(ps_polar_cable_params), C.POINTER(vp)]),
    "ps_radial_cable_defaults": (C.c_int, [C.POINTER(ps_radial_cable_params)]),
    "ps_build_radial_cable": (C.c_int, [C.POINTER(ps_radial_cable_params), C.POINTER(vp)]),
    "ps_problem_get_desc": (C.POINTER(ps_problem_desc), [vp]),
    "ps_problem_coordinates": (dp, [vp]),
    "ps_problem_free": (None, [vp]),
    "ps_builder_error": (C.c_char_p, []),
    "ps_mm_read": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "ps_csr_shape": (C.c_int, [vp, ip, ip, C.POINTER(C.c_int64)]),
    "ps_csr_row_ptr": (ip, [vp]),
    "ps_csr_col_idx": (ip, [vp]),
    "ps_csr_values": (dp, [vp]),
    "ps_csr_free": (None, [vp]),
    "ps_mm_write": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, ip, ip, dp]),
    "ps_load_problem": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(vp)]),
    "ps_format_double": (C.c_int, [C.c_double, C.c_char_p, C.c_int32]),
    "ps_write_trajectory_csv": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, dp, C.POINTER(ps_time_mesh)]),
    "ps_write_history_csv": (C.c_int, [C.c_char_p, C.c_int32, dp, dp]),
    "ps_seeded_normal": (None, [C.c_uint64, C.c_int64, C.c_double, dp]),
    "ps_seeded_uniform": (None, [C.c_uint64, C.c_int64, C.c_double, C.c_double, dp]),
}

# Every symbol the header declares (checked by tests/test_abi.py).
EXPORTED = sorted(_SIGNATURES)

_lib = None


def lib() -> C.CDLL:
    """The loaded libpppc_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib

_SIGNATURES["ps_phase_probe"] = (C.c_int, [vp, C.c_int32, C.c_int32, dp, dp])
_SIGNATURES["ps_refill_probe"] = (C.c_int, [vp, C.c_int32, dp, dp, dp, C.c_double, dp, dp, dp])
_SIGNATURES["ps_mh_bins"] = (C.c_int, [vp, ip, C.c_int32])
_SIGNATURES["ps_mh_forward"] = (C.c_int, [vp, dp, dp])
_SIGNATURES["ps_mh_inverse"] = (C.c_int, [vp, dp, dp, dp, dp])
EXPORTED = sorted(_SIGNATURES)
