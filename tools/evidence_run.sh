#!/bin/bash
# Round evidence: default bench line, ncu launch list, ncu DRAM traffic of the
# persistent kernel (single-pass metric group on a shortened launch), and a
# full ncu capture of the phase-probe kernels.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench_default.log
S="python bench.py --steps 1 --warmup 1 --fine-steps 1 --no-cpu-baseline"
timeout 300 $S > gpurun_out/short_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $S > gpurun_out/ncu_launch.log 2>&1; echo launch_rc=$?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:propagate_kernel -c 1 --csv --log-file gpurun_out/traffic.csv $S > gpurun_out/ncu_traffic.log 2>&1; echo traffic_rc=$?
timeout 300 python tools/phase_probe.py > gpurun_out/probe_plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on -k regex:phase_probe -c 3 -o gpurun_out/probe_full python tools/phase_probe.py --reps 1 > gpurun_out/probe_ncu.log 2>&1; echo probe_rc=$?
