"""Pins the CPU oracle to the reference's own known-answer tests.

Every expected value below is restated from the reference's test suite
(proj/tests/*.cpp, file:line cited per test) or from its acceptance criteria
(proj/tests/acceptance_main.cpp / SPEC.md:469-477).  The vectors are also kept
in tests/golden/reference_kats.json.  SciPy/NumPy serve as an independent
third implementation on small cases.  CPU only.
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse.linalg as spla

import paper_1905_13076_b200 as ps
from oracle import pyoracle as po
from helpers import NEWTON_BASELINE, random_linear_problem, rel_l2

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_kats.json")))


def test_time_mesh_snapping():
    """proj/tests/test_propagators.cpp:18-30."""
    m = ps.TimeMesh(3, 4, 0.02)
    assert m.coarse_dt() == 0.02 / 3
    assert m.fine_dt() == 0.02 / 3 / 4
    assert m.boundary(0) == 0.0 and m.boundary(1) == 0.02 / 3 and m.boundary(3) == 0.02
    for bad in ((1, 1, 1.0), (2, 0, 1.0), (2, 1, 0.0)):
        with pytest.raises(ps.ParasteadyError):
            ps.TimeMesh(*bad)


def test_brauer_golden():
    """proj/tests/test_problem.cpp:87-119."""
    g = GOLDEN["brauer"]
    nu, nup = po.nu("brauer", [0.0], k1=g["k1"], k2=g["k2"], k3=g["k3"])
    assert abs(nu[0] - g["nu0"]) <= g["nu0"] * 1e-14
    nu, nup = po.nu("brauer", [1e4, 1e300], k1=g["k1"], k2=g["k2"], k3=g["k3"])
    assert (nu == ps.api.K_VACUUM_RELUCTIVITY).all() and (nup == 0.0).all()
    nu, nup = po.nu("brauer", [2.0], k1=g["k1"], k2=g["k2"], k3=g["k3"])
    assert nu[0] < ps.api.K_VACUUM_RELUCTIVITY and nup[0] > 0.0
    rng = np.random.default_rng(7)
    a = np.sort(rng.uniform(0, 30, size=(200, 2)), axis=1)
    na, pa = po.nu("brauer", a[:, 0], k1=g["k1"], k2=g["k2"], k3=g["k3"])
    nb, _ = po.nu("brauer", a[:, 1], k1=g["k1"], k2=g["k2"], k3=g["k3"])
    assert (na <= nb).all() and (pa >= 0).all()


def test_dft_golden():
    """proj/tests/test_spectral.cpp:66-101."""
    g = GOLDEN["dft4"]
    hat = po.forward_dft(np.array(g["input"], dtype=float).reshape(4, 1))[:, 0]
    expect = np.array(g["re"]) + 1j * np.array(g["im"])
    assert np.max(np.abs(hat - expect)) <= 1e-14
    v = np.random.default_rng(31).uniform(-1, 1, 3)
    hat = po.forward_dft(np.tile(v, (8, 1)))
    assert np.linalg.norm(hat[0] - np.sqrt(8.0) * v) <= 1e-14
    assert np.max(np.abs(hat[1:])) <= 1e-14 * np.linalg.norm(v)
    n = 8
    hat = po.forward_dft(np.cos(2 * np.pi * np.arange(n) / n).reshape(n, 1))[:, 0]
    assert abs(hat[1] - np.sqrt(n) / 2) <= 1e-13 and abs(hat[7] - np.sqrt(n) / 2) <= 1e-13
    for b in (0, 2, 3, 4, 5, 6):
        assert abs(hat[b]) <= 1e-13


def test_dft_roundtrip_parseval_acceptance3():
    """Acceptance [3] (proj/tests/acceptance_main.cpp:138-163); NumPy as third implementation."""
    rng = np.random.default_rng(107)
    for _ in range(50):
        n = 2 * (1 + int(rng.integers(0, 16)))
        d = 1 + int(rng.integers(0, 8))
        U = rng.uniform(-1, 1, size=(n, d))
        hat = po.forward_dft(U)
        assert np.max(np.abs(hat - np.fft.fft(U, axis=0) / np.sqrt(n))) <= 1e-13
        back = po.inverse_dft(hat)
        assert np.max(np.abs(back - U)) <= 1e-12 * max(1.0, np.max(np.linalg.norm(U, axis=1)))
        assert abs(np.sum(np.abs(hat) ** 2) - np.sum(U ** 2)) <= 1e-10 * np.sum(U ** 2)
    spec = np.zeros((4, 1), dtype=complex)
    spec[1, 0] = 1j
    with pytest.raises(ps.ParasteadyError, match="conjugate symmetry"):
        po.inverse_dft(spec)


def test_jump_norm_golden():
    """proj/tests/test_engine.cpp:24-44."""
    for case in GOLDEN["jump_norm"]:
        assert abs(po.jump_norm(case["current"], case["previous"]) - case["expected"]) <= 1e-14
    with pytest.raises(ps.ParasteadyError):
        po.jump_norm(np.zeros((0, 2)), np.zeros((0, 2)))


def test_cyclic_system_and_rhs_rotation():
    """proj/tests/test_spectral.cpp:130-171: C = 200, Q = 202 for the DAE pair at N = 4."""
    p = ps.build_dae_pair()
    mesh = ps.TimeMesh(4, 1, p.period)
    orc = po.Oracle(p)
    rng = np.random.default_rng(41)
    F, G = rng.uniform(-1, 1, (4, 2)), rng.uniform(-1, 1, (4, 2))
    rhs = orc.assemble_rhs(mesh, F, G)
    M, K = p.csr(p.mass_values).toarray(), p.csr(p.stiffness_values).toarray()
    Q = M / mesh.coarse_dt() + K
    assert abs(Q[0, 0] - 202.0) <= 202 * 1e-15 and Q[0, 1] == -1.0 and Q[1, 1] == 2.0
    for row in range(4):
        sub = 4 if row == 0 else row
        expect = Q @ (F[sub - 1] - G[sub - 1]) + orc.excitation(mesh.boundary(sub))
        assert np.linalg.norm(rhs[row] - expect) <= 1e-12 * max(1.0, np.linalg.norm(expect))


def test_multiharmonic_vs_direct_acceptance1():
    """Acceptance [1]: 20 random instances, d <= 20, even N <= 32, 1e-10 (both oracle modes)."""
    rng = np.random.default_rng(101)
    worst = 0.0
    for _ in range(20):
        d = 2 + int(rng.integers(0, 19))
        n = 2 * (1 + int(rng.integers(0, 16)))
        p = random_linear_problem(d, 0.02, rng)
        mesh = ps.TimeMesh(n, 1, 0.02)
        rhs = rng.uniform(-1, 1, size=(n, d))
        orc = po.Oracle(p)
        direct = orc.solve_cyclic_direct(mesh, rhs)
        for mode in (po.DIRECT, po.ITERATIVE):
            mh = orc.mh_solve(mesh, rhs, mode=mode)
            worst = max(worst, np.linalg.norm(mh - direct) / np.linalg.norm(direct))
    assert worst <= 1e-10


def test_multiharmonic_full_bins_equals_mirror():
    """proj/tests/test_spectral.cpp:308-311."""
    rng = np.random.default_rng(67)
    p = random_linear_problem(3, 0.02, rng)
    mesh = ps.TimeMesh(8, 1, 0.02)
    rhs = rng.uniform(-1, 1, size=(8, 3))
    orc = po.Oracle(p)
    a = orc.mh_solve(mesh, rhs, use_conjugate_symmetry=True, mode=po.DIRECT)
    b = orc.mh_solve(mesh, rhs, use_conjugate_symmetry=False, mode=po.DIRECT)
    assert np.max(np.abs(a - b)) <= 1e-12 * max(1.0, np.max(np.linalg.norm(a, axis=1)))


def test_newton_step_vs_scipy():
    """Independent check of one implicit-Euler Newton step on the radial cable with SciPy."""
    cable = ps.build_coax_cable(n_r=51)
    orc = po.Oracle(cable)
    u, its, trace, _ = orc.newton_step(np.zeros(50), 0.005, 1e-3, mode=po.DIRECT)
    assert its >= 2 and all(b < a for a, b in zip(trace, trace[1:]))  # test_propagators.cpp:71-82
    # scipy Newton with the oracle's K/J assembly
    Mm = cable.csr(cable.mass_values)
    f = orc.excitation(0.005)
    x = np.zeros(50)
    for _ in range(its):
        K = cable.csr(orc.stiffness_at(x))
        J = cable.csr(orc.newton_matrix_at(x))
        R = Mm @ (x / 1e-3) + K @ x - f
        x = x + spla.spsolve((Mm / 1e-3 + J).tocsc(), -R)
    assert rel_l2(u, x) <= 1e-12
    u2, its2, _, _ = orc.newton_step(np.zeros(50), 0.005, 1e-3, mode=po.ITERATIVE)
    assert its2 == its and rel_l2(u2, u) <= 1e-10


def test_linear_newton_one_iteration():
    """proj/tests/test_propagators.cpp:52-61."""
    rng = np.random.default_rng(17)
    p = random_linear_problem(5, 0.02, rng)
    orc = po.Oracle(p)
    u_prev = rng.uniform(-1, 1, 5)
    for mode in (po.DIRECT, po.ITERATIVE):
        u, its, trace, _ = orc.newton_step(u_prev, 0.007, 1e-3, mode=mode)
        assert its == 1 and trace[-1] <= 1e-9 + 1e-8 * np.linalg.norm(orc.excitation(0.007))


def test_frozen_linearization_equals_stiffness():
    """proj/tests/test_engine.cpp:46-82."""
    cable = ps.build_coax_cable(n_r=21)
    orc = po.Oracle(cable)
    z = orc.frozen()
    ref = np.linspace(0.0, 2e-3, 20)
    r = orc.frozen(ref)
    K0 = orc.stiffness_at(np.zeros(20))
    Kr = orc.stiffness_at(ref)
    # the frozen problem is linear: its stiffness (state independent) equals K(ref)
    assert z.is_linear() and r.is_linear()
    assert np.array_equal(z.stiffness_at(np.ones(20)), K0)
    assert np.array_equal(r.stiffness_at(np.zeros(20)), Kr)
    assert np.max(np.abs(K0 - Kr)) > 0.0


def test_fine_composes_steps_bitwise():
    """proj/tests/test_propagators.cpp:127-145."""
    cable = ps.build_coax_cable(n_r=21)
    mesh = ps.TimeMesh(4, 3, cable.period)
    orc = po.Oracle(cable)
    u = np.zeros(20)
    for j in range(1, 4):
        t = mesh.boundary(2) if j == 3 else mesh.boundary(1) + j * mesh.fine_dt()
        u, _, _, _ = orc.newton_step(u, t, mesh.fine_dt(), mode=po.DIRECT)
    via = orc.fine_propagate_batch(mesh, 2, np.zeros((1, 20)), mode=po.DIRECT)[0]
    assert np.array_equal(u, via)


def test_sequential_steady_state_scalar():
    """proj/tests/test_propagators.cpp:163-194."""
    p = ps.build_scalar_test(1e-3, 1.0, 1.0, 50.0)
    orc = po.Oracle(p)
    mesh = ps.TimeMesh(20, 25, p.period)
    U, periods, conv, defects = orc.sequential_steady_state(mesh, 1e-8, 50, mode=po.DIRECT)
    assert conv and 2 <= periods <= 10 and defects[-1] < defects[0]
    analytic = 1.0 / np.hypot(1.0, 1e-3 * 2 * np.pi * 50)
    assert abs(np.max(np.abs(U)) - analytic) <= 0.05 * analytic
    p = ps.build_scalar_test(0.0, 4.0, 2.0, 50.0)
    orc = po.Oracle(p)
    mesh = ps.TimeMesh(10, 2, p.period)
    U, periods, conv, _ = orc.sequential_steady_state(mesh, 1e-12, 5, mode=po.DIRECT)
    assert conv and periods == 1 and U[0, 0] == 0.0
    for n in range(1, 10):
        expect = orc.excitation(mesh.boundary(n))[0] / 4.0
        assert abs(U[n, 0] - expect) <= 1e-14 * max(1.0, abs(expect))


def test_pppc_dae_three_ways_and_sequential():
    """proj/tests/test_engine.cpp:229-251 and acceptance [5]."""
    p = ps.build_dae_pair()
    mesh = ps.TimeMesh(8, 5, p.period)
    orc = po.Oracle(p)
    es = ps.EngineSettings(mesh, tol=1e-10)
    Ud, hd, _ = orc.solve_pp_pc(es, mode=po.DIRECT)
    Ui, hi, _ = orc.solve_pp_pc(es, mode=po.ITERATIVE)
    assert hd["converged"] and hi["converged"] and hd["iterations"] == hi["iterations"]
    assert np.max(np.abs(Ud - Ui)) <= 1e-8 * max(1.0, np.max(np.linalg.norm(Ud, axis=1)))
    assert orc.fine_periodicity_defect(mesh, Ud, mode=po.DIRECT) <= 1e-7
    # acceptance [5]: N = 8, s = 50, PP-PC tol 1e-8 vs sequential tol 1e-9 within 1e-7
    mesh = ps.TimeMesh(8, 50, p.period)
    U, h, _ = orc.solve_pp_pc(ps.EngineSettings(mesh, tol=1e-8), mode=po.DIRECT)
    S, periods, conv, _ = orc.sequential_steady_state(mesh, 1e-9, 5000, mode=po.DIRECT)
    assert h["converged"] and conv
    assert np.max(np.linalg.norm(U - S, axis=1)) / max(1.0, np.max(np.linalg.norm(S, axis=1))) <= 1e-7


def test_amplitude_first_order_acceptance6():
    """Acceptance [6] (proj/tests/acceptance_main.cpp:215-241)."""
    m, k, a, f = 1e-2, 1.0, 1.0, 50.0
    p = ps.build_scalar_test(m, k, a, f)
    analytic = a / np.hypot(k, m * 2 * np.pi * f)
    orc = po.Oracle(p)
    errs = []
    for n in (40, 80, 160):
        mesh = ps.TimeMesh(n, 1, p.period)
        zeros = np.zeros((n, 1))
        U = orc.solve_cyclic_direct(mesh, orc.assemble_rhs(mesh, zeros, zeros))
        hat = po.forward_dft(U)
        errs.append(abs(2 * abs(hat[1, 0]) / np.sqrt(n) - analytic))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(np.abs(rates - 1.0) <= 0.3), rates


def test_pppc_nonlinear_radial_cable():
    """proj/tests/test_engine.cpp:288-315 (n_r = 41, N = 4, s = 10, tol 1e-8)."""
    cable = ps.build_coax_cable(n_r=41)
    mesh = ps.TimeMesh(4, 10, cable.period)
    orc = po.Oracle(cable)
    es = ps.EngineSettings(mesh, tol=1e-8, max_iterations=10)
    U, h, _ = orc.solve_pp_pc(es, mode=po.DIRECT)
    assert h["converged"] and h["iterations"] <= 10
    assert orc.fine_periodicity_defect(mesh, U, mode=po.DIRECT) <= 1e-5
    j = h["jumps"]
    assert all(j[k] < j[k - 1] for k in range(2, len(j)))
    es2 = ps.EngineSettings(mesh, tol=1e-8, max_iterations=10, frozen_reference=U[0])
    U2, h2, _ = orc.solve_pp_pc(es2, mode=po.DIRECT)
    assert h2["converged"]
    assert np.max(np.linalg.norm(U - U2, axis=1)) <= 1e-6 * max(1.0, np.max(np.linalg.norm(U, axis=1)))


def test_line_search_extension_rescues_deep_saturation():
    """at BASELINE's I0 = 2000 A the reference's plain Newton 2-cycles
    from a random N(0,1e-3) start; the opt-in backtracking converges."""
    prob = ps.build_polar_cable(nr=12, ntheta=16)
    mesh = ps.TimeMesh(100, 20, prob.period)
    orc = po.Oracle(prob)
    u0 = ps.seeded_normal(19051308, prob.dim, 1e-3).reshape(1, -1)
    plain = ps.NewtonSettings(tol_abs=1e-9, tol_rel=1e-10, max_iter=50)
    with pytest.raises(ps.ParasteadyError, match="Newton did not converge"):
        orc.fine_propagate_batch(mesh, 1, u0, newton=plain, mode=po.DIRECT)
    F = orc.fine_propagate_batch(mesh, 1, u0, newton=NEWTON_BASELINE, mode=po.DIRECT)
    Fi = orc.fine_propagate_batch(mesh, 1, u0, newton=NEWTON_BASELINE, mode=po.ITERATIVE)
    assert rel_l2(Fi, F) <= 1e-9


# ------------------------------------------- §8(f) rank 1: Parareal and PP-IC
def _sequential_fine(orc, mesh, u0, mode=po.DIRECT):
    u = [np.asarray(u0, dtype=np.float64)]
    for n in range(1, mesh.subintervals + 1):
        u.append(orc.fine_propagate_batch(mesh, n, u[-1].reshape(1, -1), mode=mode)[0])
    return np.stack(u)


def test_classic_parareal_zero_excitation_fixed_point():
    """proj/tests/test_engine.cpp:126-133."""
    p = ps.build_scalar_test(1.0, 1.0, 0.0, 50.0)
    U, h, _ = po.Oracle(p).classic_parareal(ps.EngineSettings(ps.TimeMesh(6, 4, p.period)), np.zeros(1))
    assert h["converged"] and h["iterations"] == 1
    assert np.all(U == 0.0)


def test_classic_parareal_s1_one_iteration():
    """proj/tests/test_engine.cpp:134-140."""
    p = ps.build_dae_pair()
    U, h, _ = po.Oracle(p).classic_parareal(ps.EngineSettings(ps.TimeMesh(6, 1, p.period)), np.zeros(2))
    assert h["converged"] and h["iterations"] == 1


@pytest.mark.parametrize("mode", [po.DIRECT, po.ITERATIVE])
def test_classic_parareal_exact_termination(mode):
    """proj/tests/test_engine.cpp:141-165: with an unreachable tolerance the
    iteration stops on exact cancellation within N + 1 iterations, on the
    sequential fine solution bit for bit."""
    p = ps.build_dae_pair()
    mesh = ps.TimeMesh(6, 4, p.period)
    es = ps.EngineSettings(mesh, tol=1e-300, max_iterations=mesh.subintervals + 2)
    u0 = np.array([0.3, -0.2])
    orc = po.Oracle(p)
    U, h, _ = orc.classic_parareal(es, u0, mode=mode)
    assert h["converged"] and h["iterations"] <= mesh.subintervals + 1
    assert h["jumps"][-1] == 0.0
    assert np.array_equal(U, _sequential_fine(orc, mesh, u0, mode))


def test_classic_parareal_exactness_acceptance4():
    """Acceptance [4] (proj/tests/acceptance_main.cpp:165-191)."""
    p = ps.build_scalar_test(1.0, 1.0, 1.0, 50.0)
    mesh = ps.TimeMesh(10, 20, p.period)
    orc = po.Oracle(p)
    U, h, _ = orc.classic_parareal(ps.EngineSettings(mesh, tol=1e-300, max_iterations=10), np.zeros(1))
    F = _sequential_fine(orc, mesh, np.zeros(1))
    rel = np.max(np.linalg.norm(U - F, axis=1)) / max(1.0, np.max(np.linalg.norm(F, axis=1)))
    assert rel <= 1e-12


def test_pp_ic_needs_more_iterations_than_pp_pc_acceptance7():
    """Acceptance [7] (proj/tests/acceptance_main.cpp:243-275): linear radial
    cable, N = 20, s = 100, tol 1e-6: PP-PC within 5 iterations, PP-IC strictly
    more, both on the same periodic orbit."""
    cable = ps.build_coax_cable(linear_sleeve=True)
    mesh = ps.TimeMesh(20, 100, cable.period)
    orc = po.Oracle(cable)
    U_pc, h_pc, _ = orc.solve_pp_pc(ps.EngineSettings(mesh, tol=1e-6), mode=po.DIRECT)
    U_ic, h_ic, _ = orc.solve_pp_ic(ps.EngineSettings(mesh, tol=1e-6, max_iterations=500), mode=po.DIRECT)
    assert h_pc["converged"] and h_pc["iterations"] <= 5
    assert h_ic["converged"] and h_ic["iterations"] > h_pc["iterations"]
    assert h_ic["final_defect"] <= 1e-6
    scale = max(1.0, np.max(np.linalg.norm(U_pc, axis=1)))
    assert np.max(np.linalg.norm(U_ic - U_pc, axis=1)) / scale <= 1e-4


def test_parareal_settings_validation():
    """proj/tests/test_engine.cpp:104-123."""
    p = ps.build_dae_pair()
    orc = po.Oracle(p)
    with pytest.raises(ps.ParasteadyError, match="tolerance"):
        orc.solve_pp_ic(ps.EngineSettings(ps.TimeMesh(4, 2, p.period), tol=0.0))
    with pytest.raises(ps.ParasteadyError, match="iteration"):
        orc.classic_parareal(ps.EngineSettings(ps.TimeMesh(4, 2, p.period), max_iterations=0), np.zeros(2))
