#!/usr/bin/env python3
"""BASELINE configs[3] (full PP-PC steady state) on one B200: the cable on the
nr = 1000 x ntheta = 1024 mesh (d = 1,022,977), 50 Hz + a 1 kHz square ripple at
10 % (five odd Fourier terms), N = 64 subintervals x 100 fine steps, multiharmonic
coarse solve over bins 0..32.  Prints one JSON line per
measurement.

  step       (bounded) the initial coarse sweep from zero, ONE fine step of all 64
             subintervals from it (Newton 1e-10 rel / 1e-9 abs, PCG 1e-12), the coarse
             batch and one multiharmonic correction (ps_pppc_correct) with that
             step's states standing in for F: time, iterations and bytes of each
             phase, and the fine-sweep cost extrapolated x100.
  iterations K   solve_pp_pc with max_iterations = K: the real PP-PC iterations with
             the per-iteration fine / spectral times and COCG counts.

  python tools/config3_iteration.py step [--current 2000]
  python tools/config3_iteration.py iterations 1 [--current 74.2]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1905_13076_b200 as ps  # noqa: E402

NEWTON = ps.NewtonSettings(tol_abs=1e-9, tol_rel=1e-10, max_iter=50, line_search=30)
PCG = ps.KrylovSettings(1e-12, 50000)


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6541.5


def problem(a):
    t0 = time.perf_counter()
    prob = ps.build_polar_cable(nr=a.nr, ntheta=a.ntheta, current=a.current, ripple_terms=5)
    return prob, time.perf_counter() - t0


def status_dict(st, peak_gbs):
    out = {"kernel_ms": st.kernel_ms, "newton_iterations": st.newton_iterations,
           "pcg_iterations": st.pcg_iterations, "max_pcg_per_solve": st.max_pcg_iterations,
           "lockstep_iterations": st.lockstep_pcg_iterations, "algorithmic_GB": st.algorithmic_bytes / 1e9}
    if st.kernel_ms > 0:
        out["algorithmic_GBps"] = st.algorithmic_bytes / (st.kernel_ms / 1e3) / 1e9
        out["frac"] = out["algorithmic_GBps"] / peak_gbs
    return out


def step(a):
    prob, build_s = problem(a)
    N, s = a.N, a.steps
    mesh = ps.TimeMesh(N, s, prob.period)
    pk = peak()
    prop = ps.Propagator(prob, mesh, NEWTON, PCG, ps.KrylovSettings(1e-12, 50000), max_batch=N)
    lin = prop.frozen()
    line = {"measurement": "BASELINE configs[3] one-step probe", "nr": a.nr, "ntheta": a.ntheta, "dof": prob.dim,
            "nnz": prob.nnz, "N": N, "fine_steps": s, "current_A": a.current, "build_s": build_s}
    t0 = time.perf_counter()
    U0 = lin.coarse_sweep()
    line["coarse_sweep"] = dict(wall_s=time.perf_counter() - t0, **status_dict(lin.last_status, pk))
    dt = mesh.fine_dt()
    t_next = np.array([mesh.boundary(n - 1) + dt for n in range(1, N + 1)])
    t0 = time.perf_counter()
    res = prop.newton_step_batch(U0, t_next, dt)
    fs = status_dict(prop.last_status, pk)
    fs["wall_s"] = time.perf_counter() - t0
    fs["newton_per_system"] = [r.iterations for r in res]
    fs["sweep_estimate_s"] = fs["kernel_ms"] / 1e3 * s
    line["fine_one_step"] = fs
    F = np.stack([r.state for r in res])
    t0 = time.perf_counter()
    G = lin.coarse_propagate_batch(1, U0)
    line["coarse_batch"] = dict(wall_s=time.perf_counter() - t0, **status_dict(lin.last_status, pk))
    lin.mh_setup(True)
    t0 = time.perf_counter()
    try:
        _, jump = lin.pppc_correct(F, G, U0)
        line["correction"] = dict(wall_s=time.perf_counter() - t0, jump=jump, bins=len(lin.mh_bins()),
                                  **status_dict(lin.last_status, pk))
    except ps.ParasteadyError as exc:
        line["correction"] = {"error": str(exc)}
    line["device_used_GB"] = device_used_gb()
    print(json.dumps(line), flush=True)


def device_used_gb():
    try:
        import torch
        free, total = torch.cuda.mem_get_info(0)
        return (total - free) / 1e9
    except Exception:
        return None


def iterations(a):
    prob, build_s = problem(a)
    mesh = ps.TimeMesh(a.N, a.steps, prob.period)
    es = ps.EngineSettings(mesh, tol=a.tol, max_iterations=a.k, newton=NEWTON, pcg=PCG,
                           cocg=ps.KrylovSettings(1e-12, 50000))
    t0 = time.perf_counter()
    try:
        res = ps.solve_pp_pc(prob, es)
        h, err = res.history, None
    except ps.ParasteadyError as exc:
        h, err = None, str(exc)
    wall = time.perf_counter() - t0
    line = {"measurement": f"BASELINE configs[3] PP-PC, max_iterations = {a.k}", "nr": a.nr, "ntheta": a.ntheta,
            "dof": prob.dim, "nnz": prob.nnz, "N": a.N, "fine_steps": a.steps, "current_A": a.current,
            "tol": a.tol, "wall_s": wall, "build_s": build_s}
    if err:
        line["error"] = err
    else:
        line.update(iterations=h["iterations"], converged=h["converged"], jumps=h["jumps"],
                    fine_ms=h["fine_ms"], coarse_ms=h["coarse_ms"], spectral_ms=h["spectral_ms"],
                    total_ms=h["total_ms"], fine_pcg_iterations=h["fine_pcg_iterations"],
                    newton_iterations=h["newton_iterations"], cocg_iterations=h["cocg_iterations"],
                    cocg_per_iteration=h["cocg_per_iteration"], fine_ms_per_iteration=h["fine_ms_per_iteration"],
                    spectral_ms_per_iteration=h["spectral_ms_per_iteration"],
                    fine_algorithmic_GBps=h["fine_bytes"] / (h["fine_ms"] / 1e3) / 1e9,
                    dof_timesteps_per_s=a.N * a.steps * prob.dim * h["iterations"] / (h["fine_ms"] / 1e3))
        line["fine_frac"] = line["fine_algorithmic_GBps"] / peak()
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["step", "iterations"])
    ap.add_argument("k", type=int, nargs="?", default=1)
    ap.add_argument("--current", type=float, default=2000.0)
    ap.add_argument("--nr", type=int, default=1000)
    ap.add_argument("--ntheta", type=int, default=1024)
    ap.add_argument("--N", type=int, default=64)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--tol", type=float, default=1e-8)
    a = ap.parse_args()
    step(a) if a.what == "step" else iterations(a)


if __name__ == "__main__":
    main()
