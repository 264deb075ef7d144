#!/usr/bin/env python3
"""Diagnostic: time the config-2 fine batch (mesh N=100, s=20) in waves of W
systems (context max_batch = W), first `--steps` fine steps only via a mesh
with the same dt.  Prints ms per system-step per wave size."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_13076_b200 as ps  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--waves", type=int, nargs="*", default=[100, 50, 32, 25, 16])
ap.add_argument("--systems", type=int, default=100)
ap.add_argument("--fine-steps", type=int, default=2)
a = ap.parse_args()
prob = ps.build_polar_cable(nr=200, ntheta=256)
# same dt as config 2 (T / (100 * 20)) with fewer steps per subinterval
mesh = ps.TimeMesh(100 * 20 // a.fine_steps, a.fine_steps, prob.period)
newton = ps.NewtonSettings(tol_abs=1e-6, tol_rel=1e-10, max_iter=50, line_search=30)
pcg = ps.KrylovSettings(tol_rel=1e-12, max_iter=50000)
U = np.stack([ps.seeded_normal(19051307 + n, prob.dim, 1e-3) for n in range(1, a.systems + 1)])
dev = torch.device("cuda", 0)
Ud = torch.from_numpy(U).to(dev)
Od = torch.empty_like(Ud)
ref = None
for W in a.waves:
    prop = ps.Propagator(prob, mesh, newton, pcg, max_batch=W)
    prop.fine_propagate_batch_dev(1, W, Ud.data_ptr(), Od.data_ptr())  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    kms, pit = 0.0, 0
    for w0 in range(0, a.systems, W):
        cnt = min(W, a.systems - w0)
        st = prop.fine_propagate_batch_dev(1 + w0, cnt, Ud[w0].data_ptr(), Od[w0].data_ptr())
        kms += st.kernel_ms
        pit += st.lockstep_pcg_iterations
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    out = Od.cpu().numpy()
    if ref is None:
        ref = out.copy()
    diff = np.abs(out - ref).max()
    print(f"wave {W:4d}: {el * 1e3:9.1f} ms total, kernel {kms:9.1f} ms, "
          f"{el * 1e3 / (a.systems * a.fine_steps):7.2f} ms/system-step, lockstep intervals {pit}, "
          f"max|diff| vs first {diff:.2e}", flush=True)
    prop.close()
