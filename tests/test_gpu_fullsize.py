"""Full-size checks at BASELINE.json's own sizes, through properties that do not
need the oracle to finish the whole workload.

* configs[1] (nr=200 x ntheta=256, d = 50,945, N = 100 systems): one batched
  implicit-Euler step from the seeded N(0, 1e-3) starts.  Every system's
  result satisfies the reference's Newton stopping rule
  (proj/src/propagators.cpp:33,55) when its residual
  R = M (u - u_prev)/dt + K(u) u - f(t) is re-evaluated independently, with
  K(u) from the oracle and the products in SciPy.  Two systems are also
  compared with the oracle's own Newton step (1e-9 relative L2, same Newton
  iteration count).
* configs[2] (nr=500 x ntheta=512, d = 255,489, 256 samples, all bins
  0..128): the multiharmonic solve returns the periodic solution of the
  cyclic system Q U_n - C U_{n-1} = rhs_n (proj/src/spectral.cpp:118-150,
  257-279).  The time-domain residual is checked for every n.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_1905_13076_b200 as ps
from oracle import pyoracle as po
from helpers import NEWTON_BASELINE, rel_l2

pytestmark = pytest.mark.gpu

SEED = 19051307


def _csr(prob, values):
    d = prob.dim
    return sp.csr_matrix((values, prob.col_idx, prob.row_ptr), shape=(d, d))


def test_config2_full_size_newton_step_meets_stopping_rule():
    prob = ps.build_polar_cable(nr=200, ntheta=256)
    d = prob.dim
    assert d == 50945 and prob.nnz == 356097
    N = 100
    mesh = ps.TimeMesh(N, 20, prob.period)
    dt = mesh.fine_dt()
    prop = ps.Propagator(prob, mesh, NEWTON_BASELINE, ps.KrylovSettings(tol_rel=1e-12, max_iter=50000))
    U0 = np.stack([ps.seeded_normal(SEED + n, d, 1e-3) for n in range(1, N + 1)])
    t_next = np.array([mesh.boundary(n - 1) + dt for n in range(1, N + 1)])
    res = prop.newton_step_batch(U0, t_next, dt)
    orc = po.Oracle(prob)
    M = _csr(prob, prob.mass_values)
    for n in range(N):
        u = res[n].state
        assert np.all(np.isfinite(u)), n
        K = _csr(prob, orc.stiffness_at(u))
        f = orc.excitation(t_next[n])
        R = M @ (u - U0[n]) / dt + K @ u - f
        tol = NEWTON_BASELINE.tol_abs + NEWTON_BASELINE.tol_rel * np.linalg.norm(f)
        assert np.linalg.norm(R) <= tol * (1.0 + 1e-6), (n, np.linalg.norm(R), tol)
        assert res[n].iterations >= 1
    for n in (0, N - 1):
        u_o, its_o, _, _ = orc.newton_step(U0[n], t_next[n], dt, newton=NEWTON_BASELINE,
                                           pcg=ps.KrylovSettings(tol_rel=1e-12, max_iter=50000), mode=po.ITERATIVE)
        assert rel_l2(res[n].state, u_o) <= 1e-9, n
        assert res[n].iterations == its_o, n


def test_config3_full_size_multiharmonic_solves_the_cyclic_system():
    nr, nt, N = 500, 512, 256
    prob = ps.build_polar_cable(nr=nr, ntheta=nt)
    d = prob.dim
    assert d == 255489
    mesh = ps.TimeMesh(N, 1, prob.period)
    u_ref = ps.seeded_normal(SEED, d, 1e-3)
    lin = ps.Propagator(prob, mesh, max_batch=N).frozen(u_ref)
    lin.mh_setup(True)  # reference bin set 0..N/2, discrete implicit-Euler symbol
    g = ps.seeded_uniform(SEED + 1, d, 0.5, 1.5)
    eps = ps.seeded_normal(SEED + 2, N * d, 1e-4).reshape(N, d)
    rhs = np.sin(2 * np.pi * np.arange(N) / N)[:, None] * g[None, :] + eps
    U = lin.mh_solve(rhs)
    st = lin.last_status
    assert st.pcg_iterations > 0
    Kbar = _csr(prob, po.Oracle(prob).frozen(u_ref).stiffness_at(np.zeros(d)))
    dT = mesh.coarse_dt()
    C = _csr(prob, prob.mass_values) / dT
    Q = C + Kbar
    QU = (Q @ U.T).T
    CU = (C @ U.T).T
    res = QU - np.roll(CU, 1, axis=0) - rhs
    rel = np.linalg.norm(res) / np.linalg.norm(rhs)
    # fp64 floor of forming the residual: eps * || |Q| |U_n| + |C| |U_{n-1}| ||
    # (K-bar entries reach nu_vacuum ~ 8e5 on this mesh, so cancellation, not
    # the 1e-12 COCG tolerance, sets the level)
    absU = np.abs(U).T
    floor = np.finfo(np.float64).eps * np.linalg.norm(
        (abs(Q) @ absU).T + np.roll((abs(C) @ absU).T, 1, axis=0)) / np.linalg.norm(rhs)
    assert rel <= 1e-11 + 16.0 * floor, (rel, floor)
