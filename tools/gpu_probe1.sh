#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/wave_probe.py --waves 100 50 34 32 25 20 16 > gpurun_out/wave_probe.log 2>&1; echo wave_rc=$?
cat gpurun_out/wave_probe.log
S="python bench.py --steps 1 --warmup 0 --fine-steps 1 --pcg-tol 1e-6 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:propagate_kernel -c 1 --csv --log-file gpurun_out/traffic.csv $S > gpurun_out/ncu_traffic.log 2>&1; echo traffic_rc=$?
cat gpurun_out/traffic.csv | tail -5
