"""Parity at the BASELINE.json configs themselves.

configs[0] (nr=40 x ntheta=64, N=20 x 50 steps, I0 = 2000 A): with the
reference's frozen-at-zero coarse operator (proj/src/engine.cpp:66-74) PP-PC does
not converge at the stated current; the device must reproduce the oracle's
iterates and its failure exactly.  The most saturated convergent current
(tools/current_bisect.py, profiles/r02_config0_current_bisect.jsonl) is the
full-PP-PC parity case: every iterate within 1e-9 and the same iteration count.

configs[1] (nr=200 x ntheta=256, d = 50,945, 20 implicit-Euler steps from
N(0, 1e-3) starts): 16 subintervals over ALL 20 steps against the oracle running
the identical Newton + Jacobi-PCG algorithm on the host cores.
"""
import os

import numpy as np
import pytest

import paper_1905_13076_b200 as ps
from oracle import pyoracle as po
from helpers import NEWTON_BASELINE, rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-9
SEED = 19051307
# tools/current_bisect.py bisect 20 2000 --steps 9 (oracle, direct LDL^T, 40 iterations;
# profiles/r02_config0_current_bisect.jsonl): 74.2 A converges in 35 iterations, 78.1 A
# not within 40, 143.8 A and above diverge
CONFIG0_CONVERGENT_CURRENT = float(os.environ.get("PPPC_CONFIG0_CURRENT", "74.2"))


def _config0(current):
    prob = ps.build_polar_cable(nr=40, ntheta=64, current=current)
    mesh = ps.TimeMesh(20, 50, prob.period)
    return prob, mesh


def _settings(mesh, iters, ref=None):
    return ps.EngineSettings(mesh, tol=1e-6, max_iterations=iters, newton=NEWTON_BASELINE,
                             pcg=ps.KrylovSettings(1e-12, 50000), cocg=ps.KrylovSettings(1e-12, 50000),
                             frozen_reference=ref)


def test_config0_2000A_frozen_zero_fails_like_the_oracle():
    """At 2000 A the frozen-at-zero coarse model (nu_steel = nu(0) = 400, ~90x
    too permeable in the saturated sheath) throws the first correction far off
    the orbit and Newton then fails in iteration 2 — identically on both sides."""
    prob, mesh = _config0(2000.0)
    orc = po.Oracle(po.build_polar_cable(nr=40, ntheta=64, current=2000.0))
    es1 = _settings(mesh, 1)
    r1 = ps.solve_pp_pc(prob, es1, keep_iterates=True)
    U1, h1, its1 = orc.solve_pp_pc(es1, mode=po.ITERATIVE, keep_iterates=True)
    assert rel_l2(r1.iterates[0], its1[0]) <= TOL
    assert abs(r1.history["jumps"][0] - h1["jumps"][0]) <= 1e-9 * h1["jumps"][0]
    assert h1["jumps"][0] > 1.0                       # the first correction already jumps O(1)
    es = _settings(mesh, 6)
    with pytest.raises(ps.ParasteadyError, match="Newton did not converge") as dev:
        ps.solve_pp_pc(prob, es)
    with pytest.raises(ps.ParasteadyError, match="Newton did not converge") as ref:
        orc.solve_pp_pc(es, mode=po.ITERATIVE)
    t_dev = str(dev.value).split("at t = ")[1].split(" ")[0]
    t_ref = str(ref.value).split("at t = ")[1].split(" ")[0]
    assert float(t_dev) == float(t_ref)


def test_config0_2000A_quarter_reference_iterates_match():
    """Frozen at the T/4 (peak current) state of one sequential period instead:
    PP-PC stagnates near jump 0.05 without converging; the first three iterates
    agree with the oracle to 1e-9."""
    prob, mesh = _config0(2000.0)
    orc = po.Oracle(po.build_polar_cable(nr=40, ntheta=64, current=2000.0))
    S, _, _, _ = orc.sequential_steady_state(mesh, 1e-300, 1, newton=NEWTON_BASELINE, mode=po.ITERATIVE)
    ref = S[5]
    es = _settings(mesh, 3, ref)
    res = ps.solve_pp_pc(prob, es, keep_iterates=True)
    U_o, h_o, its_o = orc.solve_pp_pc(es, mode=po.ITERATIVE, keep_iterates=True)
    assert not res.history["converged"] and not h_o["converged"]
    assert res.history["iterations"] == h_o["iterations"] == 3
    for k in range(3):
        assert rel_l2(res.iterates[k], its_o[k]) <= TOL, k
        assert abs(res.history["jumps"][k] - h_o["jumps"][k]) <= 1e-8 * h_o["jumps"][k], k
    assert min(h_o["jumps"]) > 1e-2


@pytest.mark.slow
def test_config0_most_saturated_convergent_current():
    """The configs[0] parity case: the most saturated current at which PP-PC with
    the reference's frozen-at-zero coarse operator still converges."""
    prob, mesh = _config0(CONFIG0_CONVERGENT_CURRENT)
    orc = po.Oracle(po.build_polar_cable(nr=40, ntheta=64, current=CONFIG0_CONVERGENT_CURRENT))
    es = _settings(mesh, 60)
    res = ps.solve_pp_pc(prob, es, keep_iterates=True)
    U_o, h_o, its_o = orc.solve_pp_pc(es, mode=po.ITERATIVE, keep_iterates=True)
    assert res.history["converged"] and h_o["converged"]
    assert res.history["iterations"] == h_o["iterations"]
    for k in range(h_o["iterations"]):
        assert rel_l2(res.iterates[k], its_o[k]) <= TOL, k
    assert rel_l2(res.trajectory, U_o) <= TOL
    assert ps.fine_periodicity_defect(prob, res.trajectory, mesh, newton=NEWTON_BASELINE) <= 1e-4


@pytest.mark.slow
def test_config1_full_length_16_subintervals():
    """configs[1] over all 20 fine steps for 16 subintervals: same Newton
    iteration totals and every end state within 1e-9 of the oracle (identical
    Newton + Jacobi-PCG algorithm, host cores)."""
    prob = ps.build_polar_cable(nr=200, ntheta=256)
    mesh = ps.TimeMesh(100, 20, prob.period)
    pcg = ps.KrylovSettings(1e-12, 50000)
    count = 16
    U = np.stack([ps.seeded_normal(SEED + n, prob.dim, 1e-3) for n in range(1, count + 1)])
    prop = ps.Propagator(prob, mesh, NEWTON_BASELINE, pcg, max_batch=count)
    F = prop.fine_propagate_batch(1, U)
    st = prop.last_status
    orc = po.Oracle(po.build_polar_cable(nr=200, ntheta=256))
    F_o = orc.fine_propagate_batch(mesh, 1, U, newton=NEWTON_BASELINE, pcg=pcg, mode=po.ITERATIVE,
                                   workers=os.cpu_count())
    so = orc.last_stats
    assert st.newton_iterations == so.newton_iterations
    # PCG counts are not pinned exactly: near the 1e-12 stop the device's tree sums and
    # the oracle's sequential sums cross it a few iterations apart (cluster engine:
    # 1886 against 1882 in the longest solve)
    assert abs(st.max_pcg_iterations - so.max_pcg_iterations) <= max(2, so.max_pcg_iterations // 200)
    assert abs(st.pcg_iterations - so.pcg_iterations) <= so.pcg_iterations // 200
    for n in range(count):
        assert rel_l2(F[n], F_o[n]) <= TOL, n
