#!/usr/bin/env python3
"""BASELINE configs[4] sizing sweep (measurement, bounded): the saturation-stress
cable (Brauer k2 = 4.0, I0 = 8000 A) on the nr = 2000 x ntheta = 2048 mesh
(d = 4,093,953), N in {16, 64, 256} subintervals batched on one GPU.

The full workload (10 fine steps to PCG 1e-12 at this size) takes hours. This tool
measures what the sweep is about: that every N fits in HBM, and the device throughput
at that size. Per N it reports:
  * peak device memory after the context and the batch are resident;
  * one Newton iteration of the first fine step for all N systems (PCG relaxed to
    --pcg-tol, Newton capped at one iteration, so the lanes stop with "Newton did not
    converge", which is expected here): time, PCG counts, algorithmic GB/s;
  * the standalone phase probes (SpMV and update phase) at this size.
Start states are N(0, 1e-3), generated on the device (torch, seeded).

  python tools/config5_sizing.py [--N 16 64 256] [--pcg-tol 1e-6]
  python tools/config5_sizing.py --N 16 --fine-steps 10 --newton-max 50 --pcg-tol 1e-12   (the real sweep at N = 16)
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1905_13076_b200 as ps  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, nargs="*", default=[16, 64, 256])
ap.add_argument("--nr", type=int, default=2000)
ap.add_argument("--ntheta", type=int, default=2048)
ap.add_argument("--pcg-tol", type=float, default=1e-2)
ap.add_argument("--pcg-max", type=int, default=5000)
ap.add_argument("--newton-max", type=int, default=1, help="1: one Newton iteration (stops with 'did not converge')")
ap.add_argument("--no-probes", action="store_true")
ap.add_argument("--fine-steps", type=int, default=1,
                help="1: the first fine step only (mesh N*10 x 1); 10: the full configs[4] subintervals (mesh N x 10)")
a = ap.parse_args()

t0 = time.perf_counter()
prob = ps.build_polar_cable(nr=a.nr, ntheta=a.ntheta, brauer_k2=4.0, current=8000.0)
build_s = time.perf_counter() - t0
d = prob.dim
dev = torch.device("cuda", 0)
peak = 6530.3
try:
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    pass
for N in a.N:
    torch.cuda.synchronize()
    mesh = ps.TimeMesh(N, 10, prob.period)
    newton = ps.NewtonSettings(tol_abs=1e-9, tol_rel=1e-10, max_iter=a.newton_max,
                               line_search=0 if a.newton_max == 1 else 30)
    pmesh = ps.TimeMesh(N * 10, 1, prob.period) if a.fine_steps == 1 else ps.TimeMesh(N, a.fine_steps, prob.period)
    prop = ps.Propagator(prob, pmesh, newton,
                         ps.KrylovSettings(tol_rel=a.pcg_tol, max_iter=a.pcg_max), max_batch=N)
    g = torch.Generator(device=dev)
    g.manual_seed(19051307 + N)
    U = torch.randn((N, d), generator=g, device=dev, dtype=torch.float64) * 1e-3
    out = torch.empty_like(U)
    t1 = time.perf_counter()
    try:
        prop.fine_propagate_batch_dev(1, N, U.data_ptr(), out.data_ptr())
    except ps.ParasteadyError as exc:  # one Newton iteration by design
        print(f"N={N}: {exc}", file=sys.stderr, flush=True)
    st = prop.last_status
    torch.cuda.synchronize()
    wall = time.perf_counter() - t1
    free, total = torch.cuda.mem_get_info(dev)
    probes = {}
    for mode in (() if a.no_probes else (1, 2, 3)):
        ms, by = C.c_double(0), C.c_double(0)
        prop._check(ps.lib().ps_phase_probe(prop._ctx, mode, 3, C.byref(ms), C.byref(by)))
        probes[f"mode{mode}"] = {"us": ms.value * 1e3, "GBps": by.value / (ms.value / 1e3) / 1e9,
                                 "frac": by.value / (ms.value / 1e3) / 1e9 / peak}
    what = ("one Newton iteration of the first fine step" if a.newton_max == 1 else
            f"the first fine step (Newton <= {a.newton_max} iterations)" if a.fine_steps == 1 else
            f"all {a.fine_steps} fine steps of every subinterval (Newton <= {a.newton_max} iterations per step)")
    line = {"measurement": f"BASELINE configs[4]: {what}, PCG rel {a.pcg_tol}",
            "nr": a.nr, "ntheta": a.ntheta, "dof": d, "nnz": prob.nnz, "N": N, "build_s": build_s,
            "device_used_GB": (total - free) / 1e9, "device_total_GB": total / 1e9,
            "step_wall_s": wall, "kernel_ms": st.kernel_ms, "newton_iterations": st.newton_iterations,
            "pcg_iterations": st.pcg_iterations, "pcg_tol": a.pcg_tol,
            "algorithmic_GBps": st.algorithmic_bytes / (st.kernel_ms / 1e3) / 1e9,
            "frac": st.algorithmic_bytes / (st.kernel_ms / 1e3) / 1e9 / peak, "phase_probes": probes,
            "status": st.code, "max_pcg_per_solve": st.max_pcg_iterations,
            "max_newton": st.max_newton_iterations, "newton_max": a.newton_max,
            "fine_steps": a.fine_steps,
            "dof_timesteps_per_s": (N * a.fine_steps * d / (st.kernel_ms / 1e3)) if a.newton_max > 1 and st.code == 0
            else None,
            "failed_residual": st.residual if st.code else None}
    print(json.dumps(line), flush=True)
    prop.close()
    del U, out
    torch.cuda.empty_cache()
