#!/bin/bash
# System-per-cluster engine check: engine parity tests (all engines, forced cluster
# sizes), then one configs[1] bench step per library variant / cluster size.
mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests/test_gpu_parity.py -q -x -k "both_engines" --timeout 300 > gpurun_out/cl_tests.log 2>&1; echo cl_tests_rc=$?
tail -5 gpurun_out/cl_tests.log
for v in ${CL_VARIANTS:-main}; do
  lib=""; [ "$v" != main ] && lib=xvariants/$v.so
  for c in ${CL_SIZES:-0}; do
    PPPC_LIB=$lib PPPC_CLUSTER=$c PPPC_DEBUG_TIMING=1 PPPC_ENGINE=cluster timeout -k 10 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/cl_bench_${v}_$c.log 2>&1; echo bench_${v}_${c}_rc=$?
    grep "pppc cluster" gpurun_out/cl_bench_${v}_$c.log | head -1
    tail -1 gpurun_out/cl_bench_${v}_$c.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v C=$c', d['value'], d['ms_per_step'], d.get('solver'))"
  done
done
