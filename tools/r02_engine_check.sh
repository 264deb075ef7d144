#!/bin/bash
# System-per-block engine check: parity suites under the default engine, the
# bitwise batch-split test and configs[0]/configs[1] parity under both engines,
# then one bench step per engine.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q -x --durations=5 > gpurun_out/eng_sys_tests.log 2>&1; echo sys_tests_rc=$?
tail -8 gpurun_out/eng_sys_tests.log
timeout 900 python -m pytest tests/test_gpu_baseline_configs.py -q -x --durations=5 > gpurun_out/eng_sys_baseline.log 2>&1; echo sys_baseline_rc=$?
tail -8 gpurun_out/eng_sys_baseline.log
for e in sys lane; do
  PPPC_ENGINE=$e timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/eng_bench_$e.log 2>&1; echo bench_${e}_rc=$?
  tail -1 gpurun_out/eng_bench_$e.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', d['value'], d['ms_per_step'], d['solver'])"
done
