"""Host-side mirror of the reference's propagator / PP-PC interface over the C ABI.

Names and argument meaning follow parasteady (proj/include/parasteady/*.hpp):
TimeMesh, NewtonSettings, EngineSettings, PeriodicProblem (+ builders),
Propagator.{fine,coarse}_propagate, newton_step, frozen_coarse_linearization,
MultiharmonicCyclicSolver, assemble_rhs, jump_norm, forward_dft / inverse_dft,
solve_pp_pc and fine_periodicity_defect.  Errors raise ParasteadyError carrying
the reference's message text.  Every compute call runs on the B200 through
libpppc_b200.so; there is no CPU code path here.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _abi
from ._abi import lib

K_PI = 3.14159265358979323846
K_VACUUM_RELUCTIVITY = 1.0 / (4.0e-7 * K_PI)


class ParasteadyError(RuntimeError):
    """Raised with the reference's error message (proj/src/*.cpp runtime_error texts)."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def _dp(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(_abi.dp)


def _ip(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(_abi.ip)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _raise(code: int, ctx=None):
    if code == _abi.PS_OK:
        return
    L = lib()
    msg = L.ps_last_error(ctx) if ctx else L.ps_global_error()
    raise ParasteadyError(code, (msg or b"").decode() or f"pppc error {code}")


# ------------------------------------------------------------------ settings
@dataclass
class TimeMesh:
    """proj/include/parasteady/types.hpp:21-40."""
    subintervals: int
    fine_steps: int
    period: float

    def __post_init__(self):
        if self.subintervals < 2:
            raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "mesh: need at least 2 subintervals")
        if self.fine_steps < 1:
            raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "mesh: need at least 1 fine step per subinterval")
        if not self.period > 0.0:
            raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "mesh: period must be positive")

    def coarse_dt(self) -> float:
        return self.period / self.subintervals

    def fine_dt(self) -> float:
        return self.coarse_dt() / self.fine_steps

    def boundary(self, n: int) -> float:
        if n == self.subintervals:
            return self.period
        return float(n) * self.period / self.subintervals

    def c(self) -> _abi.ps_time_mesh:
        return _abi.ps_time_mesh(self.subintervals, self.fine_steps, self.period)


@dataclass
class NewtonSettings:
    """proj/include/parasteady/propagators.hpp:19-24 (same defaults)."""
    tol_abs: float = 1e-9
    tol_rel: float = 1e-8
    max_iter: int = 30
    damping: float = 1.0
    line_search: int = 0   # extension: step halvings (0 = reference update)


@dataclass
class KrylovSettings:
    tol_rel: float = 1e-12
    max_iter: int = 20000
    # COCG only: start a context's multiharmonic solve from its previous solution
    warm_start: bool = False


def solver_settings(newton: Optional[NewtonSettings] = None, pcg: Optional[KrylovSettings] = None,
                    cocg: Optional[KrylovSettings] = None, max_batch: int = 0,
                    engine: int = 0) -> _abi.ps_solver_settings:
    newton = newton or NewtonSettings()
    pcg = pcg or KrylovSettings()
    cocg = cocg or KrylovSettings()
    s = _abi.ps_solver_settings()
    s.newton.tol_abs, s.newton.tol_rel = newton.tol_abs, newton.tol_rel
    s.newton.max_iter, s.newton.damping = newton.max_iter, newton.damping
    s.newton.line_search = newton.line_search
    s.pcg.tol_rel, s.pcg.max_iter = pcg.tol_rel, pcg.max_iter
    s.cocg.tol_rel, s.cocg.max_iter = cocg.tol_rel, cocg.max_iter
    s.cocg.warm_start = 1 if cocg.warm_start else 0
    s.max_batch = max_batch
    s.engine = engine
    return s


@dataclass
class EngineSettings:
    """proj/include/parasteady/engine.hpp:56-72 (PP-PC multiharmonic subset)."""
    mesh: TimeMesh
    tol: float = 1e-6
    max_iterations: int = 50
    newton: NewtonSettings = field(default_factory=NewtonSettings)
    pcg: KrylovSettings = field(default_factory=KrylovSettings)
    cocg: KrylovSettings = field(default_factory=KrylovSettings)
    use_conjugate_symmetry: bool = True
    frozen_reference: Optional[np.ndarray] = None
    bin_mask: Optional[Sequence[int]] = None
    shift_kind: int = 0


# ------------------------------------------------------------------ problems
class PeriodicProblem:
    """M u' + K(u) u = f(t), u(0) = u(T) as the structured ps_problem_desc.

    Built either by the C++ builders (polar P1 cable, the reference's radial
    cable) or from explicit matrices for linear problems
    (proj/include/parasteady/problem.hpp:74-104)."""

    def __init__(self):
        self._handle = None
        self._keep = []
        self._desc = None
        self.coordinates = None

    # -- construction
    @classmethod
    def _from_builder(cls, handle) -> "PeriodicProblem":
        p = cls()
        p._handle = handle
        p._desc = lib().ps_problem_get_desc(handle).contents
        coords = lib().ps_problem_coordinates(handle)
        if coords:
            p.coordinates = np.ctypeslib.as_array(coords, shape=(p.dim, 2)).copy()
        return p

    @classmethod
    def linear(cls, mass, stiffness, terms: Sequence[dict], period: float) -> "PeriodicProblem":
        """Linear problem from dense or scipy.sparse M, K and excitation terms
        [{"pattern": array, "amplitude": a, "frequency": f, "phase": p}, ...]."""
        M = mass.toarray() if hasattr(mass, "toarray") else np.asarray(mass, dtype=np.float64)
        K = stiffness.toarray() if hasattr(stiffness, "toarray") else np.asarray(stiffness, dtype=np.float64)
        d = M.shape[0]
        if M.shape != (d, d) or K.shape != (d, d):
            raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "problem: matrix dimensions do not match the excitation")
        for name, A in (("mass", M), ("stiffness", K)):
            scale = max(1.0, float(np.max(np.abs(A))) if A.size else 1.0)
            if float(np.max(np.abs(A - A.T))) / scale > 1e-12:
                raise ParasteadyError(_abi.PS_ERR_BAD_ARG, f"problem: {name} matrix is not symmetric")
        mask = (M != 0) | (K != 0) | np.eye(d, dtype=bool)
        row_ptr = np.zeros(d + 1, dtype=np.int32)
        cols = []
        for i in range(d):
            c = np.nonzero(mask[i])[0]
            cols.append(c)
            row_ptr[i + 1] = row_ptr[i] + len(c)
        col_idx = np.ascontiguousarray(np.concatenate(cols).astype(np.int32))
        rows = np.repeat(np.arange(d), np.diff(row_ptr))
        p = cls()
        arrays = dict(row_ptr=row_ptr, col_idx=col_idx, mass=_f64(M[rows, col_idx]),
                      stiffness=_f64(K[rows, col_idx]))
        p._set_arrays(d, arrays, terms, period)
        return p

    def _set_arrays(self, d, arrays, terms, period):
        n_terms = len(terms)
        pat = _f64(np.concatenate([np.asarray(t["pattern"], dtype=np.float64).reshape(d) for t in terms])
                   if n_terms else np.zeros(1))
        amp = _f64([t.get("amplitude", 0.0) for t in terms] or [0.0])
        freq = _f64([t.get("frequency", 0.0) for t in terms] or [0.0])
        phase = _f64([t.get("phase", 0.0) for t in terms] or [0.0])
        self._keep = [arrays, pat, amp, freq, phase]
        desc = _abi.ps_problem_desc()
        desc.dim = d
        desc.nnz = int(arrays["row_ptr"][-1])
        desc.row_ptr = _ip(arrays["row_ptr"])
        desc.col_idx = _ip(arrays["col_idx"])
        desc.mass = _dp(arrays["mass"])
        desc.stiffness = _dp(arrays["stiffness"])
        desc.period = float(period)
        desc.n_terms = n_terms
        desc.patterns = _dp(pat)
        desc.amplitude = _dp(amp)
        desc.frequency_hz = _dp(freq)
        desc.phase_rad = _dp(phase)
        self._desc = desc

    def __del__(self):
        if getattr(self, "_handle", None) is not None:
            try:
                lib().ps_problem_free(self._handle)
            except Exception:
                pass
            self._handle = None

    # -- accessors (numpy views onto the description)
    @property
    def desc(self) -> _abi.ps_problem_desc:
        return self._desc

    @property
    def dim(self) -> int:
        return int(self._desc.dim)

    @property
    def nnz(self) -> int:
        return int(self._desc.nnz)

    @property
    def period(self) -> float:
        return float(self._desc.period)

    def is_linear(self) -> bool:
        return bool(self._desc.stiffness)

    def _arr(self, ptr, n, dtype=np.float64):
        return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)

    @property
    def row_ptr(self):
        return self._arr(self._desc.row_ptr, self.dim + 1, np.int32)

    @property
    def col_idx(self):
        return self._arr(self._desc.col_idx, self.nnz, np.int32)

    @property
    def mass_values(self):
        return self._arr(self._desc.mass, self.nnz)

    @property
    def stiffness_values(self):
        return self._arr(self._desc.stiffness, self.nnz) if self.is_linear() else None

    def csr(self, values) -> "scipy.sparse.csr_matrix":  # noqa: F821
        import scipy.sparse as sp
        return sp.csr_matrix((values, self.col_idx, self.row_ptr), shape=(self.dim, self.dim))

    def excitation_terms(self):
        d, n = self.dim, self._desc.n_terms
        pat = self._arr(self._desc.patterns, n * d).reshape(n, d) if n else np.zeros((0, d))
        return [dict(pattern=pat[k], amplitude=self._desc.amplitude[k], frequency=self._desc.frequency_hz[k],
                     phase=self._desc.phase_rad[k]) for k in range(n)]


def _polar_params(**kw) -> _abi.ps_polar_cable_params:
    p = _abi.ps_polar_cable_params()
    lib().ps_polar_cable_defaults(C.byref(p))
    for k, v in kw.items():
        if not hasattr(p, k):
            raise ParasteadyError(_abi.PS_ERR_BAD_ARG, f"problem: unknown polar cable parameter {k!r}")
        setattr(p, k, v)
    return p


def build_polar_cable(**params) -> PeriodicProblem:
    """2-D structured polar P1 coax cable of BASELINE.json."""
    h = C.c_void_p()
    rc = lib().ps_build_polar_cable(C.byref(_polar_params(**params)), C.byref(h))
    if rc != _abi.PS_OK:
        raise ParasteadyError(rc, lib().ps_builder_error().decode())
    return PeriodicProblem._from_builder(h)


def build_coax_cable(**params) -> PeriodicProblem:
    """The reference's 1-D radial cable (proj/src/problem.cpp:242-361)."""
    p = _abi.ps_radial_cable_params()
    lib().ps_radial_cable_defaults(C.byref(p))
    for k, v in params.items():
        if not hasattr(p, k):
            raise ParasteadyError(_abi.PS_ERR_BAD_ARG, f"problem: unknown cable parameter {k!r}")
        setattr(p, k, v)
    h = C.c_void_p()
    rc = lib().ps_build_radial_cable(C.byref(p), C.byref(h))
    if rc != _abi.PS_OK:
        raise ParasteadyError(rc, lib().ps_builder_error().decode())
    return PeriodicProblem._from_builder(h)


def build_scalar_test(m: float, k: float, amplitude: float, frequency_hz: float) -> PeriodicProblem:
    """proj/src/problem.cpp:150-169."""
    if m < 0.0:
        raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "problem: scalar mass must be non-negative")
    if m == 0.0 and k <= 0.0:
        raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "problem: degenerate scalar system")
    if not frequency_hz > 0.0:
        raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "problem: frequency must be positive")
    terms = [dict(pattern=[1.0], amplitude=amplitude, frequency=frequency_hz)] if amplitude != 0.0 else []
    return PeriodicProblem.linear([[m]], [[k]], terms, 1.0 / frequency_hz)


def build_dae_pair() -> PeriodicProblem:
    """proj/src/problem.cpp:171-188."""
    return PeriodicProblem.linear([[1.0, 0.0], [0.0, 0.0]], [[2.0, -1.0], [-1.0, 2.0]],
                                  [dict(pattern=[1.0, 0.0], amplitude=1.0, frequency=50.0)], 1.0 / 50.0)


# --------------------------------------------------------------------- files
def _builder_fail(rc):
    raise ParasteadyError(rc, lib().ps_builder_error().decode())


def read_matrix_market(path: str):
    """proj/src/matrix_market.cpp:30-81 -> scipy.sparse.csr_matrix."""
    import scipy.sparse as sp
    h = C.c_void_p()
    rc = lib().ps_mm_read(str(path).encode(), C.byref(h))
    if rc != _abi.PS_OK:
        _builder_fail(rc)
    try:
        r, c, n = C.c_int32(0), C.c_int32(0), C.c_int64(0)
        lib().ps_csr_shape(h, C.byref(r), C.byref(c), C.byref(n))
        rp = np.ctypeslib.as_array(lib().ps_csr_row_ptr(h), shape=(r.value + 1,)).copy()
        ci = np.ctypeslib.as_array(lib().ps_csr_col_idx(h), shape=(max(1, n.value),))[:n.value].copy()
        va = np.ctypeslib.as_array(lib().ps_csr_values(h), shape=(max(1, n.value),))[:n.value].copy()
        return sp.csr_matrix((va, ci, rp), shape=(r.value, c.value))
    finally:
        lib().ps_csr_free(h)


def write_matrix_market(path: str, matrix) -> None:
    """proj/src/matrix_market.cpp:83-93 (general storage, shortest round-trip values)."""
    import scipy.sparse as sp
    m = sp.csr_matrix(matrix)
    m.sort_indices()
    rp = np.ascontiguousarray(m.indptr, dtype=np.int32)
    ci = np.ascontiguousarray(m.indices, dtype=np.int32)
    va = _f64(m.data)
    rc = lib().ps_mm_write(str(path).encode(), m.shape[0], m.shape[1], _ip(rp), _ip(ci), _dp(va))
    if rc != _abi.PS_OK:
        _builder_fail(rc)


def load_problem(mass_path: str, stiffness_path: str, excitation_path: str) -> PeriodicProblem:
    """proj/src/problem.cpp:363-421: the "files" problem class on the device path."""
    h = C.c_void_p()
    rc = lib().ps_load_problem(str(mass_path).encode(), str(stiffness_path).encode(), str(excitation_path).encode(),
                               C.byref(h))
    if rc != _abi.PS_OK:
        _builder_fail(rc)
    return PeriodicProblem._from_builder(h)


def format_double(value: float) -> str:
    """proj/src/io.cpp:151-155 (shortest round-trip decimal)."""
    buf = C.create_string_buffer(64)
    _raise(lib().ps_format_double(float(value), buf, 64))
    return buf.value.decode()


def write_trajectory_csv(path: str, states, mesh: TimeMesh) -> None:
    """proj/src/io.cpp:157-170."""
    S = _f64(states)
    if S.ndim == 1:
        S = S.reshape(-1, 1)
    rc = lib().ps_write_trajectory_csv(str(path).encode(), S.shape[0], S.shape[1], _dp(S), C.byref(mesh.c()))
    if rc != _abi.PS_OK:
        _builder_fail(rc)


def write_history_csv(path: str, jumps, seconds=None) -> None:
    """proj/src/io.cpp:172-178."""
    j = _f64(jumps).reshape(-1)
    s = None if seconds is None else _f64(seconds).reshape(-1)
    rc = lib().ps_write_history_csv(str(path).encode(), j.shape[0], _dp(j), _dp(s))
    if rc != _abi.PS_OK:
        _builder_fail(rc)


def seeded_normal(seed: int, count: int, sigma: float) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    lib().ps_seeded_normal(seed, count, sigma, _dp(out))
    return out


def seeded_uniform(seed: int, count: int, lo: float, hi: float) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    lib().ps_seeded_uniform(seed, count, lo, hi, _dp(out))
    return out


# ---------------------------------------------------------------- propagator
@dataclass
class StepResult:
    """proj/include/parasteady/propagators.hpp:26-31."""
    state: np.ndarray
    iterations: int
    residual_norms: list


class Propagator:
    """Implicit-Euler fine/coarse propagator over a two-level time mesh
    (proj/include/parasteady/propagators.hpp:53-76) running on one B200.

    One context = one CUDA stream; batched calls propagate many subintervals
    in a single persistent kernel launch."""

    def __init__(self, problem: PeriodicProblem, mesh: TimeMesh, newton: Optional[NewtonSettings] = None,
                 pcg: Optional[KrylovSettings] = None, cocg: Optional[KrylovSettings] = None,
                 max_batch: int = 0, stream: Optional[int] = None, _ctx=None, engine: int = 0):
        self.problem = problem
        self.mesh = mesh
        self.newton = newton or NewtonSettings()
        self.pcg = pcg or KrylovSettings()
        self.cocg = cocg or KrylovSettings()
        self.last_status = _abi.ps_batch_status()
        if _ctx is not None:
            self._ctx = _ctx
            return
        # engine: 0 by size, 1 lane engine, 2 block engine, 3 cluster engine (ps_solver_settings.engine)
        self._settings = solver_settings(self.newton, self.pcg, self.cocg, max_batch, engine)
        ctx = C.c_void_p()
        m = mesh.c()
        rc = lib().ps_create(C.byref(problem.desc), C.byref(m), C.byref(self._settings),
                             C.c_void_p(stream) if stream else None, C.byref(ctx))
        _raise(rc)
        self._ctx = ctx

    def close(self):
        if getattr(self, "_ctx", None):
            lib().ps_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def dim(self) -> int:
        return self.problem.dim

    def last_engine(self) -> dict:
        """ps_last_engine: which engine ran the last propagation (lane / block /
        cluster) and the cluster geometry."""
        e, c, n = C.c_int32(0), C.c_int32(0), C.c_int32(0)
        _raise(lib().ps_last_engine(self._ctx, C.byref(e), C.byref(c), C.byref(n)))
        return {"engine": {0: "none", 1: "lane", 2: "block", 3: "cluster"}[e.value],
                "cluster_ctas": c.value, "coresident_clusters": n.value}

    def _check(self, rc):
        _raise(rc, self._ctx)

    def _states(self, U, count=None) -> np.ndarray:
        U = _f64(U)
        if U.ndim == 1:
            U = U.reshape(1, -1)
        if U.shape[1] != self.dim or (count is not None and U.shape[0] != count):
            raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "problem: state dimension mismatch")
        return U

    # -- batched propagation (the hot path)
    def fine_propagate_batch(self, n_first: int, U_start) -> np.ndarray:
        U = self._states(U_start)
        out = np.empty_like(U)
        st = _abi.ps_batch_status()
        rc = lib().ps_fine_propagate_batch(self._ctx, n_first, U.shape[0], _dp(U), _dp(out), C.byref(st))
        self.last_status = st
        self._check(rc)
        return out

    def coarse_propagate_batch(self, n_first: int, U_start) -> np.ndarray:
        U = self._states(U_start)
        out = np.empty_like(U)
        st = _abi.ps_batch_status()
        rc = lib().ps_coarse_propagate_batch(self._ctx, n_first, U.shape[0], _dp(U), _dp(out), C.byref(st))
        self.last_status = st
        self._check(rc)
        return out

    def fine_propagate(self, n: int, u_start) -> np.ndarray:
        return self.fine_propagate_batch(n, u_start)[0]

    def coarse_propagate(self, n: int, u_start) -> np.ndarray:
        return self.coarse_propagate_batch(n, u_start)[0]

    def fine_propagate_batch_dev(self, n_first: int, count: int, src_ptr: int, dst_ptr: int):
        st = _abi.ps_batch_status()
        rc = lib().ps_fine_propagate_batch_dev(self._ctx, n_first, count, C.c_void_p(src_ptr),
                                               C.c_void_p(dst_ptr), C.byref(st))
        self.last_status = st
        self._check(rc)
        return st

    def newton_step_batch(self, U_prev, t_next, dt: float):
        U = self._states(U_prev)
        t = _f64(np.broadcast_to(np.asarray(t_next, dtype=np.float64), (U.shape[0],)))
        out = np.empty_like(U)
        its = np.zeros(U.shape[0], dtype=np.int32)
        trace = np.zeros((U.shape[0], self.newton.max_iter), dtype=np.float64)
        st = _abi.ps_batch_status()
        rc = lib().ps_newton_step(self._ctx, U.shape[0], _dp(U), _dp(t), float(dt), _dp(out), _ip(its),
                                  _dp(trace), C.byref(st))
        self.last_status = st
        self._check(rc)
        return [StepResult(out[n], int(its[n]), list(trace[n, :its[n]])) for n in range(U.shape[0])]

    def coarse_sweep(self) -> np.ndarray:
        out = np.empty((self.mesh.subintervals, self.dim), dtype=np.float64)
        st = _abi.ps_batch_status()
        rc = lib().ps_coarse_sweep(self._ctx, _dp(out), C.byref(st))
        self.last_status = st
        self._check(rc)
        return out

    # -- operators
    def assemble(self, U):
        """K(u) and J(u) values on the CSR pattern for each state (device refill path)."""
        U = self._states(U)
        K = np.empty((U.shape[0], self.problem.nnz))
        J = np.empty_like(K)
        self._check(lib().ps_assemble_operators(self._ctx, U.shape[0], _dp(U), _dp(K), _dp(J)))
        return K, J

    def excitation(self, t) -> np.ndarray:
        t = _f64(np.atleast_1d(t))
        out = np.empty((t.shape[0], self.dim))
        self._check(lib().ps_eval_excitation(self._ctx, t.shape[0], _dp(t), _dp(out)))
        return out

    def frozen(self, reference=None) -> "Propagator":
        """frozen_coarse_linearization (proj/src/engine.cpp:66-74) on the device."""
        ref = None if reference is None else _f64(reference)
        if ref is not None and ref.shape != (self.dim,):
            raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "engine: frozen reference state dimension mismatch")
        ctx = C.c_void_p()
        self._check(lib().ps_create_frozen(self._ctx, _dp(ref), C.byref(ctx)))
        return Propagator(self.problem, self.mesh, self.newton, self.pcg, self.cocg, _ctx=ctx)

    # -- spectral (linear contexts)
    def mh_setup(self, use_conjugate_symmetry=True, bin_mask=None, shift_kind=0):
        mask = _checked_mask(bin_mask, self.mesh.subintervals, use_conjugate_symmetry)
        self._mask = mask
        self._check(lib().ps_mh_setup(self._ctx, int(bool(use_conjugate_symmetry)), _ip(mask), int(shift_kind)))

    def assemble_rhs(self, F, G) -> np.ndarray:
        F = self._states(F, self.mesh.subintervals)
        G = self._states(G, self.mesh.subintervals)
        out = np.empty_like(F)
        self._check(lib().ps_assemble_rhs(self._ctx, _dp(F), _dp(G), _dp(out)))
        return out

    def mh_solve(self, rhs) -> np.ndarray:
        R = self._states(rhs, self.mesh.subintervals)
        out = np.empty_like(R)
        st = _abi.ps_batch_status()
        rc = lib().ps_mh_solve(self._ctx, _dp(R), _dp(out), C.byref(st))
        self.last_status = st
        self._check(rc)
        return out

    # -- kernel probes (tests of the hot-path kernels themselves)
    def refill_probe(self, U, U_prev, t_next, dt: float):
        """One fused refill inside the persistent kernel: (A = M/dt + J(U) [n][nnz],
        R = M (U - U_prev)/dt + K(U) U - f(t_next) [n][d], Dinv [n][d])."""
        U = self._states(U)
        Up = self._states(U_prev, U.shape[0])
        t = _f64(np.broadcast_to(np.asarray(t_next, dtype=np.float64), (U.shape[0],)))
        A = np.empty((U.shape[0], self.problem.nnz))
        R = np.empty_like(U)
        D = np.empty_like(U)
        self._check(lib().ps_refill_probe(self._ctx, U.shape[0], _dp(U), _dp(Up), _dp(t), float(dt), _dp(A), _dp(R),
                                          _dp(D)))
        return A, R, D

    def mh_bins(self):
        buf = np.zeros(self.mesh.subintervals + 1, dtype=np.int32)
        n = lib().ps_mh_bins(self._ctx, _ip(buf), buf.shape[0])
        if n < 0:
            self._check(-n)
        return buf[:n].copy()

    def mh_forward(self, rhs) -> np.ndarray:
        """dft_forward_kernel on the solved bins: [H][d] complex."""
        R = self._states(rhs, self.mesh.subintervals)
        H = len(self.mh_bins())
        out = np.empty((H, self.dim, 2))
        self._check(lib().ps_mh_forward(self._ctx, _dp(R), _dp(out)))
        return out[..., 0] + 1j * out[..., 1]

    def mh_inverse(self, spectrum, U_old=None):
        """idft_jump_kernel + jump_finalize_kernel: (U [N][d], jump)."""
        S = np.asarray(spectrum, dtype=np.complex128)
        buf = np.ascontiguousarray(np.stack([S.real, S.imag], axis=-1))
        old = None if U_old is None else self._states(U_old, self.mesh.subintervals)
        U = np.empty((self.mesh.subintervals, self.dim))
        jump = C.c_double(0.0)
        self._check(lib().ps_mh_inverse(self._ctx, _dp(buf), _dp(old), _dp(U), C.byref(jump)))
        return U, jump.value

    def pppc_correct(self, F, G, U):
        F = self._states(F, self.mesh.subintervals)
        G = self._states(G, self.mesh.subintervals)
        Uo = self._states(U, self.mesh.subintervals).copy()
        jump = C.c_double(0.0)
        st = _abi.ps_batch_status()
        rc = lib().ps_pppc_correct(self._ctx, _dp(F), _dp(G), _dp(Uo), C.byref(jump), C.byref(st))
        self.last_status = st
        self._check(rc)
        return Uo, jump.value


def newton_step(problem: PeriodicProblem, u_prev, t_next: float, dt: float,
                settings: Optional[NewtonSettings] = None, mesh: Optional[TimeMesh] = None) -> StepResult:
    """proj/src/propagators.cpp:27-58 on the device (batch of one)."""
    if not dt > 0.0:
        raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "propagator: step size must be positive")
    settings = settings or NewtonSettings()
    if settings.max_iter < 1:
        raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "propagator: Newton needs at least one iteration")
    mesh = mesh or TimeMesh(2, 1, problem.period)
    prop = Propagator(problem, mesh, settings, max_batch=1)
    try:
        return prop.newton_step_batch(np.asarray(u_prev, dtype=np.float64).reshape(1, -1), [t_next], dt)[0]
    finally:
        prop.close()


def coarse_step(problem, u_prev, t_next, dt, settings=None) -> np.ndarray:
    return newton_step(problem, u_prev, t_next, dt, settings).state


# ------------------------------------------------------------------ spectral
@dataclass
class Harmonic:
    index: int
    omega: float


def frequency_set(n_blocks: int, period: float):
    """proj/src/spectral.cpp:94-103 (host logic)."""
    if n_blocks < 2 or n_blocks % 2 != 0:
        raise ParasteadyError(_abi.PS_ERR_ODD_BLOCKS,
                              f"spectral: frequency_set requires an even number of blocks >= 2, got {n_blocks}")
    if not period > 0.0:
        raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "spectral: period must be positive")
    out = []
    for b in range(n_blocks):
        idx = b if b <= n_blocks // 2 else b - n_blocks
        out.append(Harmonic(idx, 2.0 * K_PI * idx / period))
    return out


def forward_dft(states) -> np.ndarray:
    """Unitary DFT across the trajectory index on the device; returns complex [N][d]."""
    U = _f64(states)
    if U.ndim == 1:
        U = U.reshape(-1, 1)
    n, d = U.shape
    spec = np.empty((n, d, 2), dtype=np.float64)
    _raise(lib().ps_forward_dft(n, d, _dp(U), _dp(spec)))
    return spec[..., 0] + 1j * spec[..., 1]


def inverse_dft(spectrum) -> np.ndarray:
    S = np.asarray(spectrum, dtype=np.complex128)
    if S.ndim == 1:
        S = S.reshape(-1, 1)
    n, d = S.shape
    buf = np.ascontiguousarray(np.stack([S.real, S.imag], axis=-1))
    out = np.empty((n, d), dtype=np.float64)
    _raise(lib().ps_inverse_dft(n, d, _dp(buf), _dp(out)))
    return out


def jump_norm(current, previous) -> float:
    """proj/src/engine.cpp:54-64 on the device."""
    a, b = _f64(current), _f64(previous)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    if b.ndim == 1:
        b = b.reshape(1, -1)
    if a.size == 0 or a.shape != b.shape:
        raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "engine: jump_norm needs two state lists of equal length")
    out = C.c_double(0.0)
    _raise(lib().ps_jump_norm(a.shape[0], a.shape[1], _dp(a), _dp(b), C.byref(out)))
    return out.value


def reluctivity(kind: str, b2, nu: float = 0.0, k1: float = 0.0, k2: float = 0.0, k3: float = 0.0):
    """ReluctivityCurve::nu / nu_prime on the device (proj/src/problem.cpp:84-98)."""
    c = _abi.ps_curve(0 if kind == "constant" else 1, 0, nu, k1, k2, k3)
    x = _f64(np.atleast_1d(b2))
    n_out, p_out = np.empty_like(x), np.empty_like(x)
    _raise(lib().ps_eval_reluctivity(C.byref(c), x.shape[0], _dp(x), _dp(n_out), _dp(p_out)))
    return n_out, p_out


class MultiharmonicCyclicSolver:
    """proj/include/parasteady/spectral.hpp:94-111 over a linear (frozen) propagator."""

    def __init__(self, linear: Propagator, use_conjugate_symmetry: bool = True, bin_mask=None, shift_kind=0):
        self.linear = linear
        linear.mh_setup(use_conjugate_symmetry, bin_mask, shift_kind)

    def solve(self, rhs) -> np.ndarray:
        return self.linear.mh_solve(rhs)


def assemble_rhs(fine, coarse, linear: Propagator) -> np.ndarray:
    return linear.assemble_rhs(fine, coarse)


# -------------------------------------------------------------------- engine
def _checked_mask(bin_mask, n_blocks: int, use_conjugate_symmetry: bool):
    """The C ABI reads bins 0..N/2 (conjugate symmetry) or 0..N-1 of the mask."""
    if bin_mask is None:
        return None
    mask = np.ascontiguousarray(bin_mask, dtype=np.int32).reshape(-1)
    need = n_blocks // 2 + 1 if use_conjugate_symmetry else n_blocks
    if mask.shape[0] != need:
        raise ParasteadyError(_abi.PS_ERR_BAD_ARG, f"spectral: bin mask needs {need} entries, got {mask.shape[0]}")
    return mask


def _checked_reference(ref, dim: int):
    """frozen_coarse_linearization (proj/src/engine.cpp:66-74): empty = zero state."""
    if ref is None:
        return None
    ref = _f64(ref).reshape(-1)
    if ref.shape[0] == 0:
        return None
    if ref.shape[0] != dim:
        raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "engine: frozen reference state dimension mismatch")
    return ref


@dataclass
class PeriodicSolveResult:
    trajectory: np.ndarray          # [N][d] states at T_0..T_{N-1}
    history: dict
    iterates: Optional[np.ndarray] = None


def solve_pp_pc(problem: PeriodicProblem, settings: EngineSettings, keep_iterates: bool = False,
                stream: Optional[int] = None) -> PeriodicSolveResult:
    """PP-PC with the multiharmonic coarse solver (proj/src/engine.cpp:187-270),
    driven by the C++ host driver ps_pppc_solve."""
    mesh = settings.mesh
    prop = Propagator(problem, mesh, settings.newton, settings.pcg, settings.cocg, stream=stream)
    try:
        e = _abi.ps_engine_settings()
        e.tol = settings.tol
        e.max_iterations = settings.max_iterations
        e.use_conjugate_symmetry = int(bool(settings.use_conjugate_symmetry))
        mask = _checked_mask(settings.bin_mask, mesh.subintervals, settings.use_conjugate_symmetry)
        e.bin_mask = _ip(mask)
        e.shift_kind = settings.shift_kind
        ref = _checked_reference(settings.frozen_reference, problem.dim)
        U = np.empty((mesh.subintervals, problem.dim))
        its = (np.empty((settings.max_iterations, mesh.subintervals, problem.dim)) if keep_iterates else None)
        h = _abi.ps_history()
        rc = lib().ps_pppc_solve(prop._ctx, C.byref(e), _dp(ref), _dp(U), _dp(its), C.byref(h))
        _raise(rc, prop._ctx)
        hist = dict(iterations=h.iterations, converged=bool(h.converged),
                    jumps=[h.jumps[k] for k in range(min(h.iterations, _abi.PS_MAX_HISTORY))],
                    fine_ms=h.fine_ms, coarse_ms=h.coarse_ms, spectral_ms=h.spectral_ms, total_ms=h.total_ms,
                    fine_pcg_iterations=h.fine_pcg_iterations, coarse_pcg_iterations=h.coarse_pcg_iterations,
                    cocg_iterations=h.cocg_iterations, newton_iterations=h.newton_iterations,
                    fine_bytes=h.fine_bytes,
                    cocg_per_iteration=[h.cocg_per_iteration[k] for k in range(min(h.iterations, _abi.PS_MAX_HISTORY))],
                    fine_ms_per_iteration=[h.fine_ms_per_iteration[k]
                                           for k in range(min(h.iterations, _abi.PS_MAX_HISTORY))],
                    spectral_ms_per_iteration=[h.spectral_ms_per_iteration[k]
                                               for k in range(min(h.iterations, _abi.PS_MAX_HISTORY))])
        return PeriodicSolveResult(U, hist, its[:h.iterations] if its is not None else None)
    finally:
        prop.close()


@dataclass
class InitialValueSolveResult:
    states: np.ndarray              # [N+1][d] states at T_0..T_N
    history: dict
    iterates: Optional[np.ndarray] = None


def _parareal_family(problem: PeriodicProblem, settings: EngineSettings, u0, keep_iterates: bool,
                     stream: Optional[int]):
    mesh = settings.mesh
    if u0 is not None:
        u0 = _f64(u0).reshape(-1)
        if u0.shape[0] != problem.dim:
            raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "engine: initial state dimension mismatch")
    prop = Propagator(problem, mesh, settings.newton, settings.pcg, settings.cocg, stream=stream)
    try:
        e = _abi.ps_engine_settings()
        e.tol = settings.tol
        e.max_iterations = settings.max_iterations
        n1 = mesh.subintervals + 1
        its = np.empty((settings.max_iterations, n1, problem.dim)) if keep_iterates else None
        h = _abi.ps_history()
        if u0 is None:
            U = np.empty((mesh.subintervals, problem.dim))
            rc = lib().ps_pp_ic_solve(prop._ctx, C.byref(e), _dp(U), _dp(its), C.byref(h))
        else:
            U = np.empty((n1, problem.dim))
            rc = lib().ps_classic_parareal(prop._ctx, C.byref(e), _dp(u0), _dp(U), _dp(its), C.byref(h))
        _raise(rc, prop._ctx)
        hist = dict(iterations=h.iterations, converged=bool(h.converged),
                    jumps=[h.jumps[k] for k in range(min(h.iterations, _abi.PS_MAX_HISTORY))],
                    final_defect=h.final_defect, fine_ms=h.fine_ms, coarse_ms=h.coarse_ms, total_ms=h.total_ms,
                    fine_pcg_iterations=h.fine_pcg_iterations, coarse_pcg_iterations=h.coarse_pcg_iterations,
                    newton_iterations=h.newton_iterations, fine_bytes=h.fine_bytes)
        return U, hist, (its[:h.iterations] if its is not None else None)
    finally:
        prop.close()


def classic_parareal(problem: PeriodicProblem, u0, settings: EngineSettings, keep_iterates: bool = False,
                     stream: Optional[int] = None) -> InitialValueSolveResult:
    """Initial-value Parareal (proj/src/engine.cpp:76-129), driven by ps_classic_parareal."""
    return InitialValueSolveResult(*_parareal_family(problem, settings, u0, keep_iterates, stream))


def solve_pp_ic(problem: PeriodicProblem, settings: EngineSettings, keep_iterates: bool = False,
                stream: Optional[int] = None) -> PeriodicSolveResult:
    """PP-IC (proj/src/engine.cpp:131-185), driven by ps_pp_ic_solve."""
    return PeriodicSolveResult(*_parareal_family(problem, settings, None, keep_iterates, stream))


@dataclass
class SteadyStateResult:
    trajectory: np.ndarray          # [N][d] last period's states T_0..T_{N-1}
    periods: int
    converged: bool
    period_defects: list


def sequential_steady_state(problem: PeriodicProblem, mesh: TimeMesh, tol: float, max_periods: int,
                            newton: Optional[NewtonSettings] = None,
                            pcg: Optional[KrylovSettings] = None) -> SteadyStateResult:
    """Brute-force periodic steady state (proj/src/propagators.cpp:117-149) on the device."""
    prop = Propagator(problem, mesh, newton, pcg)
    try:
        U = np.empty((mesh.subintervals, problem.dim))
        per, conv = C.c_int32(0), C.c_int32(0)
        defects = np.zeros(max(1, int(max_periods)))
        prop._check(lib().ps_sequential_steady_state(prop._ctx, float(tol), int(max_periods), _dp(U), C.byref(per),
                                                     C.byref(conv), _dp(defects)))
        return SteadyStateResult(U, per.value, bool(conv.value), list(defects[:per.value]))
    finally:
        prop.close()


def fine_periodicity_defect(problem: PeriodicProblem, trajectory, mesh: TimeMesh,
                            newton: Optional[NewtonSettings] = None) -> float:
    """proj/src/engine.cpp:272-290."""
    T = _f64(trajectory)
    if T.shape[0] != mesh.subintervals:
        raise ParasteadyError(_abi.PS_ERR_BAD_ARG, "engine: trajectory length does not match the mesh")
    prop = Propagator(problem, mesh, newton)
    try:
        out = C.c_double(0.0)
        prop._check(lib().ps_fine_periodicity_defect(prop._ctx, _dp(T), C.byref(out)))
        return out.value
    finally:
        prop.close()


def device_info() -> dict:
    name = C.create_string_buffer(256)
    sm, ma, mi = C.c_int(0), C.c_int(0), C.c_int(0)
    _raise(lib().ps_device_info(name, 256, C.byref(sm), C.byref(ma), C.byref(mi)))
    return dict(name=name.value.decode(), sm_count=sm.value, cc=(ma.value, mi.value))


__all__ = [n for n in dir() if not n.startswith("_") and n not in ("C", "math", "np", "dataclass", "field",
                                                                   "Optional", "Sequence", "annotations")]
