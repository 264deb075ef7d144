#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python bench_extra.py config1 config3 config3full > gpurun_out/bench_extra.log 2>&1; echo extra_rc=$?
cat gpurun_out/bench_extra.log | cut -c1-600
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_config3.csv python bench_extra.py config3 --no-cpu > gpurun_out/ncu_c3.log 2>&1; echo ncu_c3_rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"dft|assemble" -c 4 -o gpurun_out/spectral_full python bench_extra.py config3 --no-cpu > gpurun_out/ncu_c3full.log 2>&1; echo ncu_c3full_rc=$?
