"""Direct output tests of the hot-path kernels themselves, through the C ABI probes
(the refill and the spectral tile kernels were only checked
through whole solves or through side kernels).

* ps_refill_probe runs ONE fused refill inside the persistent propagation kernel
  (refill_row_ell, refill_row on long rows, refill_long_rows, refill_finish);
* ps_mh_forward / ps_mh_inverse run dft_forward_kernel and idft_jump_kernel +
  jump_finalize_kernel on a context's solved bins.

Each is compared with the CPU oracle's restatement of the reference:
proj/src/propagators.cpp:13-17 (step residual), proj/src/problem.cpp:344-359
(K and J closures), proj/src/spectral.cpp:32-84,257-279 (DFT, mirror, realify),
proj/src/engine.cpp:54-64 (jump_norm).
"""
import numpy as np
import pytest

import paper_1905_13076_b200 as ps
from oracle import pyoracle as po
from helpers import random_linear_problem, rel_l2, small_polar

pytestmark = pytest.mark.gpu


def _problems():
    return {
        "polar": small_polar(),
        "polar_c0": ps.build_polar_cable(nr=40, ntheta=64),
        # conductor and insulator inside the first band: every element is Brauer
        # steel, so the hub row (ntheta + 1 slots) carries per-system values
        "polar_steel_hub": ps.build_polar_cable(nr=10, ntheta=40, r_conductor=1e-5, r_insulator=2e-5),
        "radial": ps.build_coax_cable(n_r=51),
    }


@pytest.mark.parametrize("name", ["polar", "polar_c0", "polar_steel_hub", "radial"])
def test_refill_probe_matches_oracle(name):
    prob = _problems()[name]
    mesh = ps.TimeMesh(4, 3, prob.period)
    count = 5
    prop = ps.Propagator(prob, mesh, max_batch=count)
    orc = po.Oracle(prob)
    # states from tiny to deeply saturating (B up to several tesla in the steel)
    U = np.stack([ps.seeded_normal(41 + k, prob.dim, 10.0 ** (-6 + k)) for k in range(count)])
    Up = np.stack([ps.seeded_normal(71 + k, prob.dim, 10.0 ** (-6 + k)) for k in range(count)])
    t = np.array([0.0013, 0.005, 0.0071, 0.0199, 0.02])
    dt = mesh.fine_dt()
    A, R, D = prop.refill_probe(U, Up, t, dt)
    M = prob.csr(prob.mass_values)
    for n in range(count):
        J = orc.newton_matrix_at(U[n])
        A_o = prob.mass_values / dt + J
        assert rel_l2(A[n], A_o) <= 1e-14, n
        Kd = prob.csr(orc.stiffness_at(U[n]))
        mass_term = M @ (U[n] - Up[n]) / dt
        ku = Kd @ U[n]
        f = orc.excitation(t[n])
        R_o = mass_term + ku - f
        scale = np.linalg.norm(mass_term) + np.linalg.norm(ku) + np.linalg.norm(f)
        assert np.linalg.norm(R[n] - R_o) <= 1e-13 * scale, n
        diag = prob.csr(A_o).diagonal()
        assert rel_l2(D[n], 1.0 / diag) <= 1e-15, n


def test_refill_probe_is_batch_split_invariant():
    """A system's refill does not depend on the other systems of the batch."""
    prob = small_polar()
    mesh = ps.TimeMesh(4, 3, prob.period)
    prop = ps.Propagator(prob, mesh, max_batch=6)
    U = np.stack([ps.seeded_normal(5 + k, prob.dim, 1e-3) for k in range(6)])
    Up = 0.5 * U
    A6, R6, D6 = prop.refill_probe(U, Up, 0.004, 1e-5)
    A2, R2, D2 = prop.refill_probe(U[3:5], Up[3:5], 0.004, 1e-5)
    assert np.array_equal(A6[3:5], A2) and np.array_equal(R6[3:5], R2) and np.array_equal(D6[3:5], D2)


def _frozen_polar(nr=10, ntheta=16, n_blocks=16):
    prob = ps.build_polar_cable(nr=nr, ntheta=ntheta)
    mesh = ps.TimeMesh(n_blocks, 2, prob.period)
    return prob, mesh, ps.Propagator(prob, mesh).frozen()


def _odd_mask(n_blocks, conj=True, top=None):
    n = n_blocks // 2 + 1 if conj else n_blocks
    top = n_blocks // 2 if top is None else top
    mask = np.zeros(n, dtype=np.int32)
    for b in range(n):
        h = b if b <= n_blocks // 2 else n_blocks - b
        mask[b] = 1 if (h % 2 == 1 and h <= top) else 0
    return mask


@pytest.mark.parametrize("n_blocks,conj,mask", [(16, True, None), (16, True, "odd"), (16, False, None),
                                                (32, False, "odd"), (256, True, "odd63")])
def test_dft_forward_kernel_matches_oracle(n_blocks, conj, mask):
    prob, mesh, lin = _frozen_polar(n_blocks=n_blocks)
    m = None if mask is None else _odd_mask(n_blocks, conj, 63 if mask == "odd63" else None)
    lin.mh_setup(conj, m)
    bins = lin.mh_bins()
    expect = [b for b in range(n_blocks // 2 + 1 if conj else n_blocks) if m is None or m[b]]
    assert list(bins) == expect
    rng = np.random.default_rng(n_blocks)
    rhs = rng.normal(0.0, 1.0, size=(n_blocks, prob.dim))
    hat = lin.mh_forward(rhs)
    ref = po.forward_dft(rhs)[bins]
    assert np.max(np.abs(hat - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("n_blocks,conj,mask", [(16, True, None), (16, True, "odd"), (16, False, None),
                                                (256, True, "odd63")])
def test_idft_jump_kernel_matches_oracle(n_blocks, conj, mask):
    prob, mesh, lin = _frozen_polar(n_blocks=n_blocks)
    m = None if mask is None else _odd_mask(n_blocks, conj, 63 if mask == "odd63" else None)
    lin.mh_setup(conj, m)
    bins = lin.mh_bins()
    rng = np.random.default_rng(3 + n_blocks)
    U_true = rng.normal(0.0, 1e-3, size=(n_blocks, prob.dim))
    full = po.forward_dft(U_true)
    # the reference's mirror: every unsolved bin is zero, bin N - b = conj(bin b)
    kept = np.zeros_like(full)
    for b in bins:
        kept[b] = full[b]
        if conj and 0 < b < n_blocks // 2:
            kept[n_blocks - b] = np.conj(full[b])
    U_ref = po.inverse_dft(kept)
    U_old = U_true + rng.normal(0.0, 1e-5, size=U_true.shape)
    U, jump = lin.mh_inverse(full[bins], U_old)
    assert np.max(np.abs(U - U_ref)) <= 1e-13 * np.max(np.abs(U_ref))
    assert abs(jump - po.jump_norm(U_ref, U_old)) <= 1e-12 * po.jump_norm(U_ref, U_old)
    _, jump0 = lin.mh_inverse(full[bins], None)
    assert jump0 == 0.0


def test_idft_kernel_realify_check():
    """proj/src/spectral.cpp:72-84: without the conjugate mirror an asymmetric
    spectrum leaves an imaginary residue and is rejected."""
    prob, mesh, lin = _frozen_polar(n_blocks=8)
    lin.mh_setup(False)
    spec = np.zeros((8, prob.dim), dtype=complex)
    spec[1, 0] = 1j
    with pytest.raises(ps.ParasteadyError, match="conjugate symmetry violated"):
        lin.mh_inverse(spec)


# --------------------------------------- SURVEY App. A.3/A.4 variants of the MH solve
@pytest.mark.parametrize("n_blocks,nr,ntheta,top", [(16, 10, 16, None), (32, 10, 16, None), (256, 60, 96, 63)])
def test_masked_jomega_mh_solve_matches_oracle(n_blocks, nr, ntheta, top):
    """BASELINE configs[2]'s variant (odd bins 1..63 of N = 256, K + j omega M) at
    N = 16, 32 and mid size: the device COCG against the oracle's COCG (same
    algorithm) and direct complex LDL^T."""
    prob = ps.build_polar_cable(nr=nr, ntheta=ntheta)
    mesh = ps.TimeMesh(n_blocks, 2, prob.period)
    ref = ps.seeded_normal(19051309, prob.dim, 1e-3)
    lin = ps.Propagator(prob, mesh).frozen(ref)
    mask = _odd_mask(n_blocks, True, top)
    lin.mh_setup(True, mask, shift_kind=1)
    g = ps.seeded_uniform(19051310, prob.dim, 0.5, 1.5)
    n = np.arange(n_blocks).reshape(-1, 1)
    rhs = g * np.sin(2 * np.pi * n / n_blocks) + ps.seeded_normal(19051311, n_blocks * prob.dim, 1e-4).reshape(
        n_blocks, prob.dim)
    U = lin.mh_solve(rhs)
    orc = po.Oracle(prob).frozen(ref)
    U_o = orc.mh_solve(mesh, rhs, bin_mask=mask, shift_kind=1, mode=po.ITERATIVE)
    assert rel_l2(U, U_o) <= 1e-9
    U_d = orc.mh_solve(mesh, rhs, bin_mask=mask, shift_kind=1, mode=po.DIRECT)
    assert rel_l2(U, U_d) <= 1e-9


def test_mh_probe_on_linear_reference_problem():
    """The probes on a plain linear problem (the reference's random periodic
    problem, proj/tests/support.hpp:45-61) and the forward/inverse round trip."""
    rng = np.random.default_rng(11)
    p = random_linear_problem(7, 0.02, rng)
    mesh = ps.TimeMesh(12, 1, 0.02)
    lin = ps.Propagator(p, mesh)
    lin.mh_setup(True)
    X = rng.uniform(-1, 1, size=(12, 7))
    U, _ = lin.mh_inverse(lin.mh_forward(X))
    assert np.max(np.abs(U - X)) <= 1e-13
