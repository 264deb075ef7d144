"""Shared test fixtures: seeded problems and comparison helpers."""
import numpy as np

import paper_1905_13076_b200 as ps

# BASELINE Newton / solver settings: Newton 1e-10 relative (BASELINE
# configs[1]) with the reference's 1e-9 absolute floor, opt-in backtracking.
NEWTON_BASELINE = ps.NewtonSettings(tol_abs=1e-9, tol_rel=1e-10, max_iter=50, line_search=30)


def rel_l2(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


def random_linear_problem(d, period, rng):
    """Seeded analogue of proj/tests/support.hpp:45-61: singular PSD mass, SPD
    stiffness, two excitation harmonics."""
    rank = max(1, d // 2)
    B = rng.uniform(-1, 1, size=(rank, d))
    M = B.T @ B / d
    A = rng.uniform(-1, 1, size=(d, d))
    K = A @ A.T / d + 0.5 * np.eye(d)
    terms = []
    for h in (1, 2):
        terms.append(dict(pattern=rng.uniform(-1, 1, size=d), amplitude=1.0 + 0.5 * h,
                          frequency=h / period, phase=0.4 * h))
    return ps.PeriodicProblem.linear(M, K, terms, period)


def small_polar(**kw):
    args = dict(nr=10, ntheta=16)
    args.update(kw)
    return ps.build_polar_cable(**args)
