#!/bin/bash
# Round-2 evidence with the cluster engine as the configs[1] default: the whole
# -m gpu suite, smoke(), the default bench line, the reference arm, the ncu launch
# list of the bench command and the DRAM/L2 bytes of one timed launch.
mkdir -p gpurun_out
timeout -k 10 2400 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/r02c_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -12 gpurun_out/r02c_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/r02c_smoke.log
timeout 1500 python bench.py > gpurun_out/r02c_bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/r02c_bench.log > gpurun_out/r02c_bench.json; cut -c1-400 gpurun_out/r02c_bench.json
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/r02c_bench_reference.log 2>&1; echo ref_rc=$?
tail -1 gpurun_out/r02c_bench_reference.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02c_launches.log 2>&1; echo launches_rc=$?
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum --clock-control none -k regex:syscluster -c 1 --csv --log-file gpurun_out/r02c_traffic.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02c_traffic.log 2>&1; echo traffic_rc=$?
tail -5 gpurun_out/r02c_traffic.csv
