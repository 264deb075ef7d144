"""configs[0] (nr=40 x ntheta=64, N=20 x 50 steps, PP-PC tol 1e-6) on the CPU
oracle (direct LDL^T, the reference algorithm): does PP-PC with the reference's
frozen-at-zero coarse operator (proj/src/engine.cpp:66-74) converge at a given
current?  Prints one JSON line per run; `bisect` searches the most saturated
convergent current between two bounds.

  python tools/current_bisect.py run 2000 [--ref quarter] [--iters 8]
  python tools/current_bisect.py bisect 20 2000 [--steps 8]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle as po  # noqa: E402
from paper_1905_13076_b200.api import EngineSettings, KrylovSettings, NewtonSettings, TimeMesh  # noqa: E402

NEWTON = NewtonSettings(tol_abs=1e-9, tol_rel=1e-10, max_iter=50, line_search=30)


def run(current, ref_kind="zero", iters=40, mode=po.DIRECT):
    prob = po.build_polar_cable(nr=40, ntheta=64, current=float(current))
    mesh = TimeMesh(20, 50, prob.period)
    orc = po.Oracle(prob)
    ref = None
    if ref_kind == "quarter":
        # the state at the T/4 current peak of one sequential period from zero
        U, _, _, _ = orc.sequential_steady_state(mesh, 1e-300, 1, newton=NEWTON, mode=mode)
        ref = U[5]
    es = EngineSettings(mesh=mesh, tol=1e-6, max_iterations=iters, newton=NEWTON,
                        pcg=KrylovSettings(1e-12, 50000), cocg=KrylovSettings(1e-12, 50000), frozen_reference=ref)
    t0 = time.time()
    out = dict(current=float(current), frozen_reference=ref_kind, mode="direct" if mode == po.DIRECT else "iterative")
    try:
        U, h, its = orc.solve_pp_pc(es, mode=mode, keep_iterates=True)
        out.update(converged=h["converged"], iterations=h["iterations"], jumps=h["jumps"],
                   iterate_max_norm=[float(np.abs(x).max()) for x in its])
    except po.ParasteadyError as e:
        out.update(converged=False, error=str(e))
        # the iterates up to the failing iteration: rerun with fewer iterations
        for k in range(iters - 1, 0, -1):
            es.max_iterations = k
            try:
                U, h, its = orc.solve_pp_pc(es, mode=mode, keep_iterates=True)
            except po.ParasteadyError:
                continue
            out.update(failed_in_iteration=k + 1, jumps=h["jumps"],
                       iterate_max_norm=[float(np.abs(x).max()) for x in its])
            break
    out["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["run", "bisect"])
    ap.add_argument("a", type=float)
    ap.add_argument("b", type=float, nargs="?")
    ap.add_argument("--ref", default="zero", choices=["zero", "quarter"])
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--steps", type=int, default=8)
    args = ap.parse_args()
    if args.what == "run":
        run(args.a, args.ref, args.iters)
        return
    lo, hi = args.a, args.b   # lo converges, hi does not
    for _ in range(args.steps):
        mid = round(0.5 * (lo + hi), 1)
        if run(mid, args.ref, args.iters)["converged"]:
            lo = mid
        else:
            hi = mid
    print(json.dumps({"most_saturated_convergent_current": lo, "first_divergent_current": hi}))


if __name__ == "__main__":
    main()
