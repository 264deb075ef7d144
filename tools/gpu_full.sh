#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_full.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_full.log
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1"
timeout 1500 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:propagate_kernel -c 1 --csv --log-file gpurun_out/traffic_full.csv $B > gpurun_out/ncu_traffic_full.log 2>&1; echo traffic_rc=$?
tail -2 gpurun_out/ncu_traffic_full.log | cut -c1-1500
grep -v "^==" gpurun_out/traffic_full.csv | cut -d, -f5,13,15
