#!/bin/bash
# Final round-2 evidence on the final code: -m gpu suite, smoke(), default bench line,
# reference arm, PPPC_DEBUG_TIMING breakdown, ncu launch list, ncu --set full of the
# cluster kernel on one wave of 15 systems (first fine step), DRAM/L2 bytes of one
# full timed launch.
mkdir -p gpurun_out
timeout -k 10 2400 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/r02f_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/r02f_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/r02f_smoke.log
timeout 1500 python bench.py > gpurun_out/r02f_bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/r02f_bench.log > gpurun_out/r02f_bench.json; cut -c1-330 gpurun_out/r02f_bench.json
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/r02f_bench_reference.log 2>&1; echo ref_rc=$?
tail -1 gpurun_out/r02f_bench_reference.log > gpurun_out/r02f_bench_reference.json
PPPC_DEBUG_TIMING=1 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02f_timing.log 2>&1; echo timing_rc=$?
grep -h "pppc cluster" gpurun_out/r02f_timing.log | sort | uniq -c | tee gpurun_out/r02f_cluster_timing.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02f_launches.log 2>&1; echo launches_rc=$?
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum --clock-control none -k regex:syscluster -c 1 --csv --log-file gpurun_out/r02f_traffic.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02f_traffic.log 2>&1; echo traffic_rc=$?
tail -4 gpurun_out/r02f_traffic.csv | cut -c150-
W="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --subintervals 15 --fine-steps 1 --e2e-steps 0"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:syscluster -c 1 -f -o gpurun_out/r02f_cluster_ncu $W > gpurun_out/r02f_ncu.log 2>&1; echo ncu_rc=$?
