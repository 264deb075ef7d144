#!/bin/bash
# Round-2 end evidence in one call: tests, smoke, default bench line, reference arm,
# ncu launch list + DRAM/L2 traffic of the timed launch, the COCG kernel's traffic at
# configs[2], phase-probe --set full capture, bench_extra.  Outputs under gpurun_out/final2/.
O=gpurun_out/final2; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
nproc > $O/host.txt; free -g >> $O/host.txt
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log
timeout 1200 python bench.py > $O/bench.log 2>&1; echo bench_rc=$?; tail -1 $O/bench.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > $O/bench_ref.log 2>&1; echo ref_rc=$?; tail -1 $O/bench_ref.log | cut -c1-300
S="python bench.py --steps 1 --warmup 1 --fine-steps 1 --no-cpu-baseline"
timeout 300 $S > $O/short_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $S > $O/ncu_launch.log 2>&1; echo launch_rc=$?
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1"
timeout 1800 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:propagate_kernel -c 1 --csv --log-file $O/traffic_full.csv $B > $O/ncu_traffic.log 2>&1; echo traffic_rc=$?
C="python bench_extra.py config3 --no-cpu"
timeout 600 ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:cocg_kernel -c 1 --csv --log-file $O/cocg_traffic.csv $C > $O/ncu_cocg.log 2>&1; echo cocg_rc=$?
timeout 300 python tools/phase_probe.py > $O/probe_plain.log 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:phase_probe -c 3 -o $O/probe_full python tools/phase_probe.py --reps 1 > $O/probe_ncu.log 2>&1; echo probe_rc=$?
timeout 1500 python bench_extra.py config1 config3 > $O/bench_extra.log 2>&1; echo extra_rc=$?
