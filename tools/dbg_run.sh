#!/bin/bash
# Debug-timing run: per-phase work / wait, action shares and per-group interval
# counts of the config-2 propagation (PPPC_DEBUG_TIMING), plus a default bench.
mkdir -p gpurun_out
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/it_bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/it_bench.log | cut -c1-250
fi
PPPC_DEBUG_TIMING=1 timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 1 ${DBG_ARGS:---fine-steps 2} > gpurun_out/it_dbg.log 2>&1; echo dbg_rc=$?
grep -v "^{" gpurun_out/it_dbg.log | tail -12
