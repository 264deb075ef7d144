#!/bin/bash
# One GPU call: parity tests, smoke, default bench line, ncu launch list and the
# application-replay DRAM traffic of the persistent propagation kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench_default.log
S="python bench.py --steps 1 --warmup 1 --fine-steps 1 --no-cpu-baseline"
timeout 300 $S > gpurun_out/short_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $S > gpurun_out/ncu_launch.log 2>&1; echo launch_rc=$?
timeout 1200 bash tools/profile_cmd.sh gpurun_out/prof > gpurun_out/prof_cmd.log 2>&1; echo prof_rc=$?
