#!/bin/bash
# One-call validation of HEAD on a B200: the whole -m gpu suite, smoke(), the default bench line.
O=gpurun_out/validate; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench.log 2>&1; echo bench_rc=$?; tail -1 $O/bench.log | cut -c1-400
