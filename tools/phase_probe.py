#!/usr/bin/env python3
"""Time the PCG phases of the config-2 batch as standalone kernels (diagnostic).

  python tools/phase_probe.py [--reps 20] [--mode 0 1 2]
Runs one short nonlinear propagation to populate the buffers, then times each
phase probe; under ncu, profile `-k regex:phase_probe`."""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1905_13076_b200 as ps  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--mode", type=int, nargs="*", default=[1, 2, 3])
ap.add_argument("--nr", type=int, default=200)
ap.add_argument("--ntheta", type=int, default=256)
ap.add_argument("--N", type=int, default=100)
a = ap.parse_args()
prob = ps.build_polar_cable(nr=a.nr, ntheta=a.ntheta)
mesh = ps.TimeMesh(a.N, 1, prob.period)
newton = ps.NewtonSettings(tol_abs=1e-6, tol_rel=1e-10, max_iter=50, line_search=30)
prop = ps.Propagator(prob, mesh, newton, ps.KrylovSettings(tol_rel=1e-3))
U = np.stack([ps.seeded_normal(19051307 + n, prob.dim, 1e-3) for n in range(1, a.N + 1)])
prop.fine_propagate_batch(1, U)
peak = 6534.5
for mode in a.mode:
    ms, by = C.c_double(0), C.c_double(0)
    prop._check(ps.lib().ps_phase_probe(prop._ctx, mode, a.reps, C.byref(ms), C.byref(by)))
    gbs = by.value / (ms.value / 1e3) / 1e9
    print(f"mode {mode}: {ms.value * 1e3:.1f} us  bytes {by.value / 1e6:.1f} MB  {gbs:.0f} GB/s  "
          f"({gbs / peak:.2f} of {peak})", flush=True)
