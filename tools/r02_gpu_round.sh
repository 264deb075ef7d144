#!/bin/bash
# Round-2 GPU pass: kernel probes, BASELINE-config parity, the whole -m gpu
# suite, then one default bench line.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/pytest_kernels.log 2>&1; echo kernels_rc=$?
tail -3 gpurun_out/pytest_kernels.log
timeout 2400 python -m pytest tests/test_gpu_baseline_configs.py -q --durations=0 ${BASELINE_K:+-k "$BASELINE_K"} > gpurun_out/pytest_baseline.log 2>&1; echo baseline_rc=$?
tail -15 gpurun_out/pytest_baseline.log
timeout 1800 python -m pytest tests -m gpu -q --durations=15 --deselect tests/test_gpu_baseline_configs.py > gpurun_out/pytest_gpu.log 2>&1; echo gpu_rc=$?
tail -20 gpurun_out/pytest_gpu.log
