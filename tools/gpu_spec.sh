#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_spec.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_spec.log
timeout 900 python bench_extra.py config1 config3 --no-cpu > gpurun_out/bench_spec.log 2>&1; echo c3_rc=$?
cut -c1-900 gpurun_out/bench_spec.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"dft|assemble|jump" --csv --log-file gpurun_out/launches_spec.csv python bench_extra.py config3 --no-cpu > gpurun_out/ncu_spec.log 2>&1; echo ncu_rc=$?
grep -v "^==" gpurun_out/launches_spec.csv | cut -d, -f5,13,15 | head -30
