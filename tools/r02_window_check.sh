#!/bin/bash
# Phase-A sliding window: phase probes at run lengths 1/2/4/8, quick parity, short bench A/B.
O=gpurun_out/window; mkdir -p $O
for R in 1 2 4 8; do echo "run=$R"; PPPC_RUN=$R timeout 300 python tools/phase_probe.py --reps 20; done > $O/probe.log 2>&1; cat $O/probe.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -x > $O/pytest.log 2>&1; echo pytest_rc=$?; tail -2 $O/pytest.log
for R in 1 8; do PPPC_RUN=$R timeout 600 python bench.py --steps 1 --warmup 1 --fine-steps 5 --no-cpu-baseline > $O/bench_run$R.log 2>&1; echo bench_run$R rc=$?; tail -1 $O/bench_run$R.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['solver'])"; done
