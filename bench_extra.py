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


# the most saturated current at which PP-PC with the reference's frozen-at-zero
# coarse operator converges (profiles/r02_config0_current_bisect.jsonl); BASELINE's
# 2000 A diverges (tests/test_gpu_baseline_configs.py)
CONFIG0_CURRENT = 74.2


def config1(cpu=True):
    prob = ps.build_polar_cable(current=CONFIG0_CURRENT)
    mesh = ps.TimeMesh(20, 50, prob.period)
    es = ps.EngineSettings(mesh, tol=1e-6, max_iterations=40, newton=NEWTON)
    ps.solve_pp_pc(prob, es)  # warm-up (context, module load)
    t0 = time.perf_counter()
    res = ps.solve_pp_pc(prob, es)
    wall = time.perf_counter() - t0
    h = res.history
    out = {"measurement": f"PP-PC wall time, BASELINE configs[0] (I0 = {CONFIG0_CURRENT} A, DESIGN.md §2)",
           "d": prob.dim, "N": 20, "s": 50, "iterations": h["iterations"], "converged": h["converged"],
           "jumps": h["jumps"], "wall_s": wall, "device_total_ms": h["total_ms"], "fine_ms": h["fine_ms"],
           "coarse_ms": h["coarse_ms"], "spectral_ms": h["spectral_ms"],
           "fine_pcg_iterations": h["fine_pcg_iterations"], "newton_iterations": h["newton_iterations"],
           "fine_achieved_GBps": h["fine_bytes"] / (h["fine_ms"] / 1e3) / 1e9,
           "dof_timesteps_per_s_fine": 20 * 50 * prob.dim * h["iterations"] / (h["fine_ms"] / 1e3)}
    out["cocg_per_iteration"] = h["cocg_per_iteration"]
    if cpu:
        from oracle import pyoracle as po
        orc = po.Oracle(po.build_polar_cable(current=CONFIG0_CURRENT))  # the oracle's own builder
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
        mask = np.zeros(N // 2 + 1, dtype=np.int32)  # bins 0..N/2 (conjugate symmetry)
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
        orc = po.Oracle(po.build_polar_cable(nr=nr, ntheta=nt)).frozen(u_ref)
        cores = os.cpu_count() or 1
        # the reference's algorithm: a sparse factorization per solved bin once
        # (proj/src/spectral.cpp:233-255), then one back-substitution per bin in
        # every PP-PC iteration (:257-279); bins in parallel on all host cores
        t0 = time.perf_counter()
        U_d = orc.mh_solve(mesh, rhs, bin_mask=mask, shift_kind=shift, mode=po.DIRECT,
                           workers=min(cores, out["bins"]))
        el = time.perf_counter() - t0
        tm = orc.last_direct_timing
        busy = tm["factor_s"] + tm["solve_s"]
        out["cpu_direct"] = {"kind": "port", "cores": cores, "wall_s": el, "factor_s_summed": tm["factor_s"],
                             "solve_s_summed": tm["solve_s"],
                             "per_iteration_solve_wall_s": tm["wall_s"] * tm["solve_s"] / busy if busy else None,
                             "factor_once_wall_s": tm["wall_s"] * tm["factor_s"] / busy if busy else None,
                             "rel_l2_vs_gpu": float(np.linalg.norm(U - U_d) / np.linalg.norm(U_d))}
        # the same Jacobi-COCG on one bin as a bounded single-core sample
        t0 = time.perf_counter()
        sub_mask = np.zeros(N // 2 + 1, dtype=np.int32)
        sub_mask[1] = 1
        orc.mh_solve(mesh, rhs, bin_mask=sub_mask, shift_kind=shift, mode=po.ITERATIVE, workers=1)
        el = time.perf_counter() - t0
        out["cpu_cocg_one_bin_s"] = el
        out["cpu_cocg_extrapolated_s"] = el * out["bins"] / min(out["bins"], cores)
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
