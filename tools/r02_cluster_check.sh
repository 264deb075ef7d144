#!/bin/bash
# System-per-cluster engine check: engine parity tests (all engines, forced cluster
# sizes), then one configs[1] bench step per cluster size and for the lane engine.
mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests/test_gpu_parity.py -q -x -k "both_engines" --timeout 300 > gpurun_out/cl_tests.log 2>&1; echo cl_tests_rc=$?
tail -15 gpurun_out/cl_tests.log
for c in ${CL_SIZES:-0 6 8}; do
  PPPC_CLUSTER=$c PPPC_DEBUG_TIMING=1 PPPC_ENGINE=cluster timeout -k 10 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/cl_bench_$c.log 2>&1; echo bench_${c}_rc=$?
  grep "pppc cluster" gpurun_out/cl_bench_$c.log | head -1
  tail -1 gpurun_out/cl_bench_$c.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('C=$c', d['value'], d['ms_per_step'], d.get('solver'), d.get('roofline'))"
done
