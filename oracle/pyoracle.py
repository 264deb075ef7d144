"""ctypes wrapper of liboracle_pppc.so — TEST INFRASTRUCTURE ONLY.

The oracle is the CPU restatement of the reference algorithm (oracle.cpp).  It
consumes a ps_problem_desc: either its own (build_polar_cable / seeded_normal
below come from oracle/polar_mesh.cpp, so the reference arm of bench.py never
loads the product library) or the product builder's, which tests/test_builders.py
proves bit-identical.  Only the ctypes declarations and plain settings
dataclasses are shared with the product package; nothing here loads
libpppc_b200.so."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1905_13076_b200 import _abi
from paper_1905_13076_b200.api import (EngineSettings, KrylovSettings, NewtonSettings, ParasteadyError,
                                       TimeMesh, solver_settings)

HERE = os.path.dirname(os.path.abspath(__file__))
# PPPC_ORACLE_LIB: the same source built for the host (bench.py oracle_native)
LIB = os.environ.get("PPPC_ORACLE_LIB") or os.path.join(HERE, "liboracle_pppc.so")
DIRECT, ITERATIVE = 0, 1

dp, ip, vp = _abi.dp, _abi.ip, C.c_void_p


class or_stats(C.Structure):
    _fields_ = [("newton_iterations", C.c_int64), ("pcg_iterations", C.c_int64),
                ("max_newton_iterations", C.c_int32), ("max_pcg_iterations", C.c_int32),
                ("failed_index", C.c_int32), ("code", C.c_int32)]


_SIG = {
    "or_last_error": (C.c_char_p, []),
    "or_create": (C.c_int, [C.POINTER(_abi.ps_problem_desc), dp, C.POINTER(vp)]),
    "or_free": (None, [vp]),
    "or_dim": (C.c_int, [vp]),
    "or_nnz": (C.c_int, [vp]),
    "or_is_linear": (C.c_int, [vp]),
    "or_frozen": (C.c_int, [vp, dp, C.POINTER(vp)]),
    "or_nu": (None, [C.POINTER(_abi.ps_curve), C.c_int32, dp, dp, dp]),
    "or_excitation": (C.c_int, [vp, C.c_double, dp]),
    "or_stiffness_at": (C.c_int, [vp, dp, dp]),
    "or_newton_matrix_at": (C.c_int, [vp, dp, dp]),
    "or_newton_step": (C.c_int, [vp, C.POINTER(_abi.ps_solver_settings), C.c_int32, dp, C.c_double,
                                 C.c_double, dp, ip, dp, C.POINTER(C.c_int64)]),
    "or_fine_propagate_batch": (C.c_int, [vp, C.POINTER(_abi.ps_time_mesh), C.POINTER(_abi.ps_solver_settings),
                                          C.c_int32, C.c_int32, C.c_int32, dp, dp, C.c_int32,
                                          C.POINTER(or_stats)]),
    "or_coarse_propagate_batch": (C.c_int, [vp, C.POINTER(_abi.ps_time_mesh),
                                            C.POINTER(_abi.ps_solver_settings), C.c_int32, C.c_int32,
                                            C.c_int32, dp, dp, C.c_int32, C.POINTER(or_stats)]),
    "or_coarse_sweep": (C.c_int, [vp, C.POINTER(_abi.ps_time_mesh), C.POINTER(_abi.ps_solver_settings),
                                  C.c_int32, dp]),
    "or_forward_dft": (C.c_int, [C.c_int32, C.c_int32, dp, dp]),
    "or_inverse_dft": (C.c_int, [C.c_int32, C.c_int32, dp, dp]),
    "or_assemble_rhs": (C.c_int, [vp, C.POINTER(_abi.ps_time_mesh), dp, dp, dp]),
    "or_mh_solve": (C.c_int, [vp, C.POINTER(_abi.ps_time_mesh), C.POINTER(_abi.ps_solver_settings), C.c_int32,
                              C.c_int32, ip, C.c_int32, dp, dp, C.c_int32, C.POINTER(C.c_int64)]),
    "or_solve_cyclic_direct": (C.c_int, [vp, C.POINTER(_abi.ps_time_mesh), dp, dp]),
    "or_last_direct_timing": (C.c_int, [dp, dp, dp]),
    "or_jump_norm": (C.c_double, [C.c_int32, C.c_int32, dp, dp]),
    "or_pppc_solve": (C.c_int, [vp, C.POINTER(_abi.ps_time_mesh), C.POINTER(_abi.ps_solver_settings),
                                C.POINTER(_abi.ps_engine_settings), C.c_int32, dp, dp, dp,
                                C.POINTER(_abi.ps_history), C.c_int32]),
    "or_classic_parareal": (C.c_int, [vp, C.POINTER(_abi.ps_time_mesh), C.POINTER(_abi.ps_solver_settings),
                                      C.POINTER(_abi.ps_engine_settings), C.c_int32, dp, dp, dp,
                                      C.POINTER(_abi.ps_history), C.c_int32]),
    "or_pp_ic_solve": (C.c_int, [vp, C.POINTER(_abi.ps_time_mesh), C.POINTER(_abi.ps_solver_settings),
                                 C.POINTER(_abi.ps_engine_settings), C.c_int32, dp, dp,
                                 C.POINTER(_abi.ps_history), C.c_int32]),
    "or_fine_periodicity_defect": (C.c_int, [vp, C.POINTER(_abi.ps_time_mesh),
                                             C.POINTER(_abi.ps_solver_settings), C.c_int32, dp, dp, C.c_int32]),
    "or_polar_cable_defaults": (C.c_int, [C.POINTER(_abi.ps_polar_cable_params)]),
    "or_build_polar_cable": (C.c_int, [C.POINTER(_abi.ps_polar_cable_params), C.POINTER(vp)]),
    "or_mesh_error": (C.c_char_p, []),
    "or_mesh_desc": (C.POINTER(_abi.ps_problem_desc), [vp]),
    "or_mesh_coordinates": (dp, [vp]),
    "or_mesh_free": (None, [vp]),
    "or_seeded_normal": (None, [C.c_uint64, C.c_int64, C.c_double, dp]),
    "or_seeded_uniform": (None, [C.c_uint64, C.c_int64, C.c_double, C.c_double, dp]),
    "or_sequential_steady_state": (C.c_int, [vp, C.POINTER(_abi.ps_time_mesh),
                                             C.POINTER(_abi.ps_solver_settings), C.c_int32, C.c_double,
                                             C.c_int32, dp, ip, ip, dp]),
}
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} missing: run __graft_entry__.build()")
        h = C.CDLL(LIB)
        for name, (res, args) in _SIG.items():
            fn = getattr(h, name)
            fn.restype, fn.argtypes = res, args
        _lib = h
    return _lib


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return None if a is None else a.ctypes.data_as(dp)


def _check(rc):
    if rc != 0:
        raise ParasteadyError(rc, lib().or_last_error().decode())


def workers_default():
    return max(1, os.cpu_count() or 1)


class OracleProblem:
    """A problem built by the oracle's own builder (oracle/polar_mesh.cpp): the
    same accessors Oracle needs (desc, coordinates) plus numpy views."""

    def __init__(self, handle):
        self._h = handle
        self.desc = lib().or_mesh_desc(handle).contents
        self.dim, self.nnz = int(self.desc.dim), int(self.desc.nnz)
        self.period = float(self.desc.period)
        self.coordinates = np.ctypeslib.as_array(lib().or_mesh_coordinates(handle), shape=(self.dim, 2)).copy()

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().or_mesh_free(self._h)
                self._h = None
        except Exception:
            pass

    def array(self, name):
        d = self.desc
        n = {"row_ptr": self.dim + 1, "col_idx": self.nnz, "mass": self.nnz, "stiffness": self.nnz,
             "elem_nodes": d.n_elem * d.nodes_per_elem, "elem_stiff": d.n_elem * d.nodes_per_elem ** 2,
             "elem_inv_area": d.n_elem, "elem_curve": d.n_elem, "patterns": d.n_terms * self.dim,
             "amplitude": d.n_terms, "frequency_hz": d.n_terms, "phase_rad": d.n_terms}[name]
        ptr = getattr(d, name)
        if not ptr:
            return None
        return np.ctypeslib.as_array(ptr, shape=(n,)).copy()


def build_polar_cable(**params) -> OracleProblem:
    """The canonical polar P1 cable from the oracle's own builder."""
    p = _abi.ps_polar_cable_params()
    lib().or_polar_cable_defaults(C.byref(p))
    for k, v in params.items():
        if not hasattr(p, k):
            raise ParasteadyError(_abi.PS_ERR_BAD_ARG, f"problem: unknown polar cable parameter {k!r}")
        setattr(p, k, v)
    h = vp()
    if lib().or_build_polar_cable(C.byref(p), C.byref(h)) != 0:
        raise ParasteadyError(_abi.PS_ERR_BAD_ARG, lib().or_mesh_error().decode())
    return OracleProblem(h)


def seeded_normal(seed: int, count: int, sigma: float) -> np.ndarray:
    out = np.empty(count)
    lib().or_seeded_normal(seed, count, sigma, _p(out))
    return out


def seeded_uniform(seed: int, count: int, lo: float, hi: float) -> np.ndarray:
    out = np.empty(count)
    lib().or_seeded_uniform(seed, count, lo, hi, _p(out))
    return out


class Oracle:
    """CPU restatement of parasteady over one PeriodicProblem."""

    def __init__(self, problem, _handle=None):
        self.problem = problem
        if _handle is not None:
            self._h = _handle
        else:
            h = vp()
            coords = None if problem.coordinates is None else _f(problem.coordinates)
            self._coords = coords
            _check(lib().or_create(C.byref(problem.desc), _p(coords), C.byref(h)))
            self._h = h
        self.dim = lib().or_dim(self._h)
        self.nnz = lib().or_nnz(self._h)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().or_free(self._h)
                self._h = None
        except Exception:
            pass

    def is_linear(self):
        return bool(lib().or_is_linear(self._h))

    def frozen(self, reference=None) -> "Oracle":
        h = vp()
        ref = None if reference is None else _f(reference)
        _check(lib().or_frozen(self._h, _p(ref), C.byref(h)))
        return Oracle(self.problem, _handle=h)

    @staticmethod
    def _s(newton=None, pcg=None, cocg=None):
        return solver_settings(newton or NewtonSettings(), pcg or KrylovSettings(), cocg or KrylovSettings())

    def excitation(self, t):
        f = np.empty(self.dim)
        _check(lib().or_excitation(self._h, float(t), _p(f)))
        return f

    def stiffness_at(self, u):
        K = np.empty(self.nnz)
        _check(lib().or_stiffness_at(self._h, _p(_f(u)), _p(K)))
        return K

    def newton_matrix_at(self, u):
        J = np.empty(self.nnz)
        _check(lib().or_newton_matrix_at(self._h, _p(_f(u)), _p(J)))
        return J

    def newton_step(self, u_prev, t_next, dt, newton=None, pcg=None, mode=ITERATIVE):
        s = self._s(newton, pcg)
        out = np.empty(self.dim)
        its = C.c_int32(0)
        trace = np.zeros(s.newton.max_iter)
        pcg_its = C.c_int64(0)
        _check(lib().or_newton_step(self._h, C.byref(s), mode, _p(_f(u_prev)), float(t_next), float(dt), _p(out),
                                    C.byref(its), _p(trace), C.byref(pcg_its)))
        return out, its.value, list(trace[:its.value]), pcg_its.value

    def _batch(self, fn, mesh, n_first, U, newton, pcg, mode, workers):
        U = _f(U).reshape(-1, self.dim)
        out = np.empty_like(U)
        s = self._s(newton, pcg)
        m = mesh.c()
        st = or_stats()
        _check(fn(self._h, C.byref(m), C.byref(s), mode, n_first, U.shape[0], _p(U), _p(out),
                  workers or workers_default(), C.byref(st)))
        self.last_stats = st
        return out

    def fine_propagate_batch(self, mesh, n_first, U, newton=None, pcg=None, mode=ITERATIVE, workers=None):
        return self._batch(lib().or_fine_propagate_batch, mesh, n_first, U, newton, pcg, mode, workers)

    def coarse_propagate_batch(self, mesh, n_first, U, newton=None, pcg=None, mode=ITERATIVE, workers=None):
        return self._batch(lib().or_coarse_propagate_batch, mesh, n_first, U, newton, pcg, mode, workers)

    def coarse_sweep(self, mesh, newton=None, pcg=None, mode=ITERATIVE):
        out = np.empty((mesh.subintervals, self.dim))
        s = self._s(newton, pcg)
        m = mesh.c()
        _check(lib().or_coarse_sweep(self._h, C.byref(m), C.byref(s), mode, _p(out)))
        return out

    def assemble_rhs(self, mesh, F, G):
        out = np.empty((mesh.subintervals, self.dim))
        m = mesh.c()
        _check(lib().or_assemble_rhs(self._h, C.byref(m), _p(_f(F)), _p(_f(G)), _p(out)))
        return out

    def mh_solve(self, mesh, rhs, use_conjugate_symmetry=True, bin_mask=None, shift_kind=0, mode=ITERATIVE,
                 cocg=None, workers=None):
        out = np.empty((mesh.subintervals, self.dim))
        s = self._s(cocg=cocg)
        m = mesh.c()
        mask = None if bin_mask is None else np.ascontiguousarray(bin_mask, dtype=np.int32)
        its = C.c_int64(0)
        _check(lib().or_mh_solve(self._h, C.byref(m), C.byref(s), mode, int(bool(use_conjugate_symmetry)),
                                 None if mask is None else mask.ctypes.data_as(ip), shift_kind, _p(_f(rhs)),
                                 _p(out), workers or workers_default(), C.byref(its)))
        self.last_cocg_iterations = its.value
        if mode == DIRECT:
            f, sv, w = C.c_double(0), C.c_double(0), C.c_double(0)
            lib().or_last_direct_timing(C.byref(f), C.byref(sv), C.byref(w))
            self.last_direct_timing = dict(factor_s=f.value, solve_s=sv.value, wall_s=w.value)
        return out

    def solve_cyclic_direct(self, mesh, rhs):
        out = np.empty((mesh.subintervals, self.dim))
        m = mesh.c()
        _check(lib().or_solve_cyclic_direct(self._h, C.byref(m), _p(_f(rhs)), _p(out)))
        return out

    def solve_pp_pc(self, settings: EngineSettings, mode=ITERATIVE, keep_iterates=False, workers=None):
        mesh = settings.mesh
        s = self._s(settings.newton, settings.pcg, settings.cocg)
        m = mesh.c()
        e = _abi.ps_engine_settings()
        e.tol, e.max_iterations = settings.tol, settings.max_iterations
        e.use_conjugate_symmetry = int(bool(settings.use_conjugate_symmetry))
        mask = None if settings.bin_mask is None else np.ascontiguousarray(settings.bin_mask, dtype=np.int32)
        e.bin_mask = None if mask is None else mask.ctypes.data_as(ip)
        e.shift_kind = settings.shift_kind
        ref = None if settings.frozen_reference is None else _f(settings.frozen_reference)
        U = np.empty((mesh.subintervals, self.dim))
        its = np.empty((settings.max_iterations, mesh.subintervals, self.dim)) if keep_iterates else None
        h = _abi.ps_history()
        _check(lib().or_pppc_solve(self._h, C.byref(m), C.byref(s), C.byref(e), mode, _p(ref), _p(U), _p(its),
                                   C.byref(h), workers or workers_default()))
        hist = dict(iterations=h.iterations, converged=bool(h.converged),
                    jumps=[h.jumps[k] for k in range(min(h.iterations, _abi.PS_MAX_HISTORY))],
                    fine_pcg_iterations=h.fine_pcg_iterations, coarse_pcg_iterations=h.coarse_pcg_iterations,
                    cocg_iterations=h.cocg_iterations, newton_iterations=h.newton_iterations,
                    cocg_per_iteration=[h.cocg_per_iteration[k]
                                        for k in range(min(h.iterations, _abi.PS_MAX_HISTORY))])
        return U, hist, (its[:h.iterations] if its is not None else None)

    def _parareal(self, settings, u0, mode, keep_iterates, workers):
        mesh = settings.mesh
        s = self._s(settings.newton, settings.pcg, settings.cocg)
        m = mesh.c()
        e = _abi.ps_engine_settings()
        e.tol, e.max_iterations = settings.tol, settings.max_iterations
        n1 = mesh.subintervals + 1
        its = np.empty((settings.max_iterations, n1, self.dim)) if keep_iterates else None
        h = _abi.ps_history()
        if u0 is None:
            U = np.empty((mesh.subintervals, self.dim))
            _check(lib().or_pp_ic_solve(self._h, C.byref(m), C.byref(s), C.byref(e), mode, _p(U), _p(its),
                                        C.byref(h), workers or workers_default()))
        else:
            U = np.empty((n1, self.dim))
            _check(lib().or_classic_parareal(self._h, C.byref(m), C.byref(s), C.byref(e), mode, _p(_f(u0)), _p(U),
                                             _p(its), C.byref(h), workers or workers_default()))
        hist = dict(iterations=h.iterations, converged=bool(h.converged),
                    jumps=[h.jumps[k] for k in range(min(h.iterations, _abi.PS_MAX_HISTORY))],
                    final_defect=h.final_defect, fine_pcg_iterations=h.fine_pcg_iterations,
                    coarse_pcg_iterations=h.coarse_pcg_iterations, newton_iterations=h.newton_iterations)
        return U, hist, (its[:h.iterations] if its is not None else None)

    def classic_parareal(self, settings: EngineSettings, u0, mode=ITERATIVE, keep_iterates=False, workers=None):
        """proj/src/engine.cpp:76-129: states [N+1][d]."""
        return self._parareal(settings, u0, mode, keep_iterates, workers)

    def solve_pp_ic(self, settings: EngineSettings, mode=ITERATIVE, keep_iterates=False, workers=None):
        """proj/src/engine.cpp:131-185: trajectory [N][d] (T_0..T_{N-1})."""
        return self._parareal(settings, None, mode, keep_iterates, workers)

    def fine_periodicity_defect(self, mesh, U, newton=None, pcg=None, mode=ITERATIVE, workers=None):
        s = self._s(newton, pcg)
        m = mesh.c()
        out = C.c_double(0.0)
        _check(lib().or_fine_periodicity_defect(self._h, C.byref(m), C.byref(s), mode, _p(_f(U)), C.byref(out),
                                                workers or workers_default()))
        return out.value

    def sequential_steady_state(self, mesh, tol, max_periods, newton=None, pcg=None, mode=ITERATIVE):
        s = self._s(newton, pcg)
        m = mesh.c()
        U = np.empty((mesh.subintervals, self.dim))
        per, conv = C.c_int32(0), C.c_int32(0)
        defects = np.zeros(max_periods)
        _check(lib().or_sequential_steady_state(self._h, C.byref(m), C.byref(s), mode, float(tol), max_periods,
                                                _p(U), C.byref(per), C.byref(conv), _p(defects)))
        return U, per.value, bool(conv.value), list(defects[:per.value])


def nu(kind, b2, nu_const=0.0, k1=0.0, k2=0.0, k3=0.0):
    c = _abi.ps_curve(0 if kind == "constant" else 1, 0, nu_const, k1, k2, k3)
    x = _f(np.atleast_1d(b2))
    a, b = np.empty_like(x), np.empty_like(x)
    lib().or_nu(C.byref(c), x.shape[0], _p(x), _p(a), _p(b))
    return a, b


def forward_dft(U):
    U = _f(U)
    if U.ndim == 1:
        U = U.reshape(-1, 1)
    n, d = U.shape
    spec = np.empty((n, d, 2))
    _check(lib().or_forward_dft(n, d, _p(U), _p(spec)))
    return spec[..., 0] + 1j * spec[..., 1]


def inverse_dft(S):
    S = np.asarray(S, dtype=np.complex128)
    if S.ndim == 1:
        S = S.reshape(-1, 1)
    n, d = S.shape
    buf = np.ascontiguousarray(np.stack([S.real, S.imag], axis=-1))
    out = np.empty((n, d))
    _check(lib().or_inverse_dft(n, d, _p(buf), _p(out)))
    return out


def jump_norm(cur, prev):
    a, b = _f(cur), _f(prev)
    if a.ndim == 1:
        a, b = a.reshape(1, -1), b.reshape(1, -1)
    if a.size == 0 or a.shape != b.shape:
        raise ParasteadyError(1, "engine: jump_norm needs two state lists of equal length")
    return lib().or_jump_norm(a.shape[0], a.shape[1], _p(a), _p(b))
