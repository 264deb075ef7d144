"""Problem builders (host C++): canonical polar P1 mesh counts and invariants,
and the reference's radial cable restated from proj/src/problem.cpp:242-361.  CPU only."""
import numpy as np
import pytest

import paper_1905_13076_b200 as ps
from oracle import pyoracle as po


@pytest.mark.parametrize("nr,nt", [(2, 4), (3, 5), (5, 8), (40, 64), (200, 256)])
def test_polar_counts(nr, nt):
    """d = 1 + (nr-1) nt, nnz = 1 + nt (7 nr - 9)."""
    p = ps.build_polar_cable(nr=nr, ntheta=nt)
    assert p.dim == 1 + (nr - 1) * nt
    assert p.nnz == 1 + nt * (7 * nr - 9)
    assert p.desc.n_elem == nt * (2 * nr - 1)
    rp = p.row_ptr
    assert rp[1] - rp[0] == nt + 1                     # the hub row
    assert np.max(np.diff(rp)[1:]) <= 7


def test_polar_invariants():
    p = ps.build_polar_cable()
    M = p.csr(p.mass_values)
    assert abs(M - M.T).max() == 0.0
    assert np.min(np.linalg.eigvalsh(M.toarray())) >= -1e-12 * abs(M).max()
    K0 = p.csr(po.Oracle(p).stiffness_at(np.zeros(p.dim))).toarray()
    assert np.max(np.abs(K0 - K0.T)) <= 1e-12 * np.max(np.abs(K0))
    assert np.min(np.linalg.eigvalsh(K0)) > 0.0
    pat = p.excitation_terms()[0]["pattern"]
    # the conductor carries exactly +1 and the sheath returns exactly -1 over the
    # free DOFs (proj/tests/test_problem.cpp:128-135 invariant)
    r = np.hypot(*p.coordinates.T)
    assert abs(pat[r < 2e-3 + 1e-9].sum() - 1.0) <= 1e-13
    assert abs(pat[r > 4e-3 - 1e-9].sum() + 1.0) <= 1e-13
    assert abs(pat.sum()) <= 1e-13
    # J - K is PSD (element weights 2 B^2 nu' >= 0), proj/tests/test_problem.cpp:165-172
    u = np.linspace(0, 5e-3, p.dim)
    orc = po.Oracle(p)
    D = p.csr(orc.newton_matrix_at(u) - orc.stiffness_at(u)).toarray()
    ev = np.linalg.eigvalsh(0.5 * (D + D.T))
    assert ev.min() >= -1e-10 * max(1.0, ev.max())


def _reference_radial_K(params, u, jacobian=False):
    """Direct restatement of CableGrid::weighted_stiffness / element_b_squared and the
    K/J closures (proj/src/problem.cpp:204-237, 344-359) as a dense matrix."""
    n_r, r3 = params["n_r"], params.get("r3", 5e-3)
    r1, r2 = params.get("r1", 2e-3), params.get("r2", 3.5e-3)
    k1, k2, k3 = 49.4, 1.46, 520.6
    vac = 1.0 / (4.0e-7 * 3.14159265358979323846)
    n_el = n_r - 1
    dim = n_r - 1
    h = r3 / n_el
    radii = np.array([r3 * i / n_el for i in range(n_r)])
    K = np.zeros((dim, dim))
    for e in range(n_el):
        ua = u[e] if e < dim else 0.0
        ub = u[e + 1] if e + 1 < dim else 0.0
        b2 = ((ub - ua) / h) ** 2
        mid = 0.5 * (radii[e] + radii[e + 1])
        if r1 <= mid < r2:
            expo = min(k2 * b2, 700.0)
            nu = min(k1 * np.exp(expo) + k3, vac)
            nup = 0.0 if k1 * np.exp(expo) + k3 >= vac else k1 * k2 * np.exp(expo)
        else:
            nu, nup = vac, 0.0
        w = nu + 2.0 * b2 * nup if jacobian else nu
        c = w * 2.0 * 3.14159265358979323846 * mid / h
        a, b = e, e + 1
        if a < dim:
            K[a, a] += c
        if a < dim and b < dim:
            K[a, b] -= c
            K[b, a] -= c
        if b < dim:
            K[b, b] += c
    return K


def test_radial_cable_matches_reference_formulas():
    """The generic element form reproduces the reference's 1-D closures."""
    params = dict(n_r=51)
    p = ps.build_coax_cable(**params)
    assert p.dim == 50 and not p.is_linear()                    # test_problem.cpp:121-126
    pat = p.excitation_terms()[0]["pattern"]
    assert abs(pat.sum() - 1.0) <= 1e-12 and pat.min() >= 0.0   # :128-135
    M = p.csr(p.mass_values).toarray()
    assert np.max(np.abs(M - M.T)) == 0.0 and np.max(np.abs(M[49])) == 0.0   # :137-146
    orc = po.Oracle(p)
    for u in (np.zeros(50), np.linspace(0.0, 5e-3, 50), np.random.default_rng(3).uniform(-1e-3, 1e-3, 50)):
        K = p.csr(orc.stiffness_at(u)).toarray()
        J = p.csr(orc.newton_matrix_at(u)).toarray()
        Kr, Jr = _reference_radial_K(params, u), _reference_radial_K(params, u, True)
        assert np.max(np.abs(K - Kr)) <= 1e-12 * np.max(np.abs(Kr))
        assert np.max(np.abs(J - Jr)) <= 1e-12 * np.max(np.abs(Jr))


def test_radial_linear_sleeve_is_linear():
    p = ps.build_coax_cable(n_r=51, linear_sleeve=1)
    assert p.is_linear()
    K = p.csr(p.stiffness_values).toarray()
    Kr = _reference_radial_K(dict(n_r=51), np.zeros(50))
    assert np.max(np.abs(K - Kr)) <= 1e-12 * np.max(np.abs(Kr))


@pytest.mark.parametrize("kw", [dict(n_r=2), dict(r2=2e-3), dict(source_region=3), dict(sigma_sleeve=-1.0)])
def test_radial_rejects_bad_parameters(kw):
    """proj/tests/test_problem.cpp:180-193."""
    with pytest.raises(ps.ParasteadyError):
        ps.build_coax_cable(**kw)


def test_seeded_generators_are_deterministic():
    a = ps.seeded_normal(19051307, 1001, 1e-3)
    b = ps.seeded_normal(19051307, 1001, 1e-3)
    assert np.array_equal(a, b) and abs(a.std() - 1e-3) < 1e-4
    u = ps.seeded_uniform(1, 1000, 0.5, 1.5)
    assert u.min() >= 0.5 and u.max() < 1.5


def test_excitation_frequency_validation_matches_reference():
    """proj/tests/test_problem.cpp:67-78: a non-integer multiple of 1/T is rejected."""
    bad = ps.PeriodicProblem.linear([[1.0]], [[1.0]], [dict(pattern=[1.0], amplitude=1.0, frequency=75.0)], 0.02)
    with pytest.raises(ps.ParasteadyError, match="integer multiple"):
        po.Oracle(bad)


@pytest.mark.parametrize("kw", [dict(nr=2, ntheta=4), dict(nr=10, ntheta=16), dict(),
                                dict(nr=12, ntheta=16, ripple_terms=5), dict(nr=40, ntheta=64, linear_sheath=1),
                                dict(nr=200, ntheta=256), dict(nr=33, ntheta=7, return_in_sheath=0, current=20.0),
                                dict(nr=10, ntheta=40, r_conductor=1e-5, r_insulator=2e-5)])
def test_oracle_builder_is_bit_identical(kw):
    """The oracle's own polar builder (oracle/polar_mesh.cpp) and the product
    builder (csrc/builders.cpp) are written independently; every array of the
    problem description they hand to the two sides must agree bit for bit, so
    feeding the oracle either problem is the same check."""
    a = ps.build_polar_cable(**kw)
    b = po.build_polar_cable(**kw)
    assert (a.dim, a.nnz, a.period) == (b.dim, b.nnz, b.period)
    da, db = a.desc, b.desc
    for f in ("n_elem", "nodes_per_elem", "n_curves", "n_terms"):
        assert getattr(da, f) == getattr(db, f), f
    for k in range(da.n_curves):
        ca, cb = da.curves[k], db.curves[k]
        assert (ca.kind, ca.nu, ca.k1, ca.k2, ca.k3) == (cb.kind, cb.nu, cb.k1, cb.k2, cb.k3)
    n = dict(row_ptr=a.dim + 1, col_idx=a.nnz, mass=a.nnz, stiffness=a.nnz,
             elem_nodes=da.n_elem * 3, elem_stiff=da.n_elem * 9, elem_inv_area=da.n_elem,
             elem_curve=da.n_elem, patterns=da.n_terms * a.dim, amplitude=da.n_terms,
             frequency_hz=da.n_terms, phase_rad=da.n_terms)
    for name, cnt in n.items():
        pa, pb = getattr(da, name), getattr(db, name)
        assert bool(pa) == bool(pb), name
        if not pa:
            continue
        xa = np.ctypeslib.as_array(pa, shape=(cnt,))
        xb = np.ctypeslib.as_array(pb, shape=(cnt,))
        assert xa.tobytes() == xb.tobytes(), name
    assert a.coordinates.tobytes() == b.coordinates.tobytes()


def test_oracle_generators_are_bit_identical():
    for seed, n in ((19051307, 1), (19051308, 50945), (5, 7)):
        assert ps.seeded_normal(seed, n, 1e-3).tobytes() == po.seeded_normal(seed, n, 1e-3).tobytes()
        assert ps.seeded_uniform(seed, n, 0.5, 1.5).tobytes() == po.seeded_uniform(seed, n, 0.5, 1.5).tobytes()
