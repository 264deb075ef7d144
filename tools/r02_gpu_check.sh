mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
PPPC_DEBUG_TIMING=1 timeout 900 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/bench_dbg.log 2>&1; echo dbg_rc=$?
timeout 1200 python bench.py --steps 2 --warmup 1 > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench_default.log
