#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_spec2.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_spec2.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"dft|jump" --csv --log-file gpurun_out/launches_spec2.csv python bench_extra.py config3 --no-cpu > gpurun_out/ncu_spec2.log 2>&1; echo ncu_rc=$?
grep -v "^==" gpurun_out/launches_spec2.csv | cut -d, -f5,13,15 | grep -v bytes | head -12
PPPC_DEBUG_TIMING=1 timeout 600 python tools/wave_probe.py --waves 100 > gpurun_out/dbg_timing.log 2>&1; echo dbg_rc=$?
cat gpurun_out/dbg_timing.log | head -40
