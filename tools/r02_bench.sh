#!/bin/bash
# One default bench line plus the per-interval timing breakdown of one step.
mkdir -p gpurun_out
PPPC_DEBUG_TIMING=1 timeout 900 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/bench_dbg.log 2>&1; echo dbg_rc=$?
grep -v "^{" gpurun_out/bench_dbg.log | tail -30
timeout 1500 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench_default.log
