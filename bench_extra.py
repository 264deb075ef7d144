#!/usr/bin/env python3
"""Secondary measurements (not the driver's bench line): BASELINE configs[0]
full PP-PC wall time and configs[2] multiharmonic coarse solve, each with the
oracle timed beside it.  Prints one JSON object per measurement.

  python bench_extra.py [config1] [config3] [--no-cpu]
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1905_13076_b200 as ps  # noqa: E402

NEWTON = ps.NewtonSettings(tol_abs=1e-9, tol_rel=1e-10, max_iter=50, line_search=30)


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def config1(cpu=True):
    prob = ps.build_polar_cable(current=20.0)
    mesh = ps.TimeMesh(20, 50, prob.period)
    es = ps.EngineSettings(mesh, tol=1e-6, max_iterations=30, newton=NEWTON)
    ps.solve_pp_pc(prob, es)  # warm-up (context, module load)
    t0 = time.perf_counter()
    res = ps.solve_pp_pc(prob, es)
    wall = time.perf_counter() - t0
    h = res.history
    out = {"measurement": "PP-PC wall time, BASELINE configs[0] geometry (I0 = 20 A, DESIGN.md §2)",
           "d": prob.dim, "N": 20, "s": 50, "iterations": h["iterations"], "converged": h["converged"],
           "jumps": h["jumps"], "wall_s": wall, "device_total_ms": h["total_ms"], "fine_ms": h["fine_ms"],
           "coarse_ms": h["coarse_ms"], "spectral_ms": h["spectral_ms"],
           "fine_pcg_iterations": h["fine_pcg_iterations"], "newton_iterations": h["newton_iterations"],
           "fine_achieved_GBps": h["fine_bytes"] / (h["fine_ms"] / 1e3) / 1e9,
           "dof_timesteps_per_s_fine": 20 * 50 * prob.dim * h["iterations"] / (h["fine_ms"] / 1e3)}
    if cpu:
        from oracle import pyoracle as po
        orc = po.Oracle(prob)
        for mode, name in ((po.DIRECT, "direct LDL^T (reference algorithm)"), (po.ITERATIVE, "Jacobi-PCG")):
            t0 = time.perf_counter()
            U, ho, _ = orc.solve_pp_pc(es, mode=mode)
            out[f"cpu_{'direct' if mode == po.DIRECT else 'pcg'}"] = {
                "wall_s": time.perf_counter() - t0, "iterations": ho["iterations"], "cores": os.cpu_count(),
                "kind": "port", "what": name}
    return out


def config3(cpu=True, full_bins=False):
    nr, nt, N = 500, 512, 256
    prob = ps.build_polar_cable(nr=nr, ntheta=nt)
    d = prob.dim
    mesh = ps.TimeMesh(N, 1, prob.period)
    u_ref = ps.seeded_normal(19051307, d, 1e-3)
    lin = ps.Propagator(prob, mesh, max_batch=N).frozen(u_ref)
    if full_bins:
        mask, shift, label = None, 0, "reference bins 0..128, discrete symbol"
    else:
        mask = np.zeros(N, dtype=np.int32)
        mask[1:64:2] = 1
        shift, label = 1, "odd harmonics 1..63, K + j w M (BASELINE wording)"
    lin.mh_setup(True, mask, shift)
    g = ps.seeded_uniform(19051308, d, 0.5, 1.5)
    eps = ps.seeded_normal(19051309, N * d, 1e-4).reshape(N, d)
    rhs = np.sin(2 * np.pi * np.arange(N) / N)[:, None] * g[None, :] + eps
    lin.mh_solve(rhs)  # warm-up
    t0 = time.perf_counter()
    U = lin.mh_solve(rhs)
    wall = time.perf_counter() - t0
    st = lin.last_status
    out = {"measurement": f"multiharmonic coarse solve, BASELINE configs[2] ({label})", "d": d, "nnz": prob.nnz,
           "N": N, "bins": int(N // 2 + 1 if mask is None else mask.sum()), "cocg_iterations": st.pcg_iterations,
           "max_cocg_per_bin": st.max_pcg_iterations, "lockstep_iterations": st.lockstep_pcg_iterations,
           "kernel_ms": st.kernel_ms, "wall_s_with_host_copies": wall,
           "achieved_GBps": st.algorithmic_bytes / (st.kernel_ms / 1e3) / 1e9, "peak_GBps": peak()}
    out["frac"] = out["achieved_GBps"] / out["peak_GBps"]
    if cpu:
        from oracle import pyoracle as po
        orc = po.Oracle(prob).frozen(u_ref)
        t0 = time.perf_counter()
        sub_mask = np.zeros(N, dtype=np.int32)
        sub_mask[1] = 1  # one bin as the bounded CPU sample
        orc.mh_solve(mesh, rhs, bin_mask=sub_mask, shift_kind=shift, mode=po.ITERATIVE)
        el = time.perf_counter() - t0
        out["cpu_one_bin_s"] = el
        out["cpu_extrapolated_s"] = el * out["bins"] / min(out["bins"], os.cpu_count() or 1)
    return out


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    cpu = "--no-cpu" not in sys.argv
    which = args or ["config1", "config3"]
    for w in which:
        if w == "config1":
            print(json.dumps(config1(cpu)), flush=True)
        elif w == "config3":
            print(json.dumps(config3(cpu)), flush=True)
        elif w == "config3full":
            print(json.dumps(config3(cpu, full_bins=True)), flush=True)


if __name__ == "__main__":
    main()
