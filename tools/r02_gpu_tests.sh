#!/bin/bash
# Round-2 parity additions on one B200: the kernel probes, the BASELINE-config
# parity cases (with timings), then the whole -m gpu suite.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/pytest_kernels.log 2>&1; echo kernels_rc=$?
tail -3 gpurun_out/pytest_kernels.log
timeout 2400 python -m pytest tests/test_gpu_baseline_configs.py -q --durations=0 ${BASELINE_K:+-k "$BASELINE_K"} > gpurun_out/pytest_baseline.log 2>&1; echo baseline_rc=$?
tail -15 gpurun_out/pytest_baseline.log
