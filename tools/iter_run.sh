#!/bin/bash
# Iteration run on the GPU box: gpu parity (fast set), phase probes, short bench,
# optional ncu capture of one probe mode (PROBE_NCU=<mode>).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/it_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/it_tests.log
timeout 300 python tools/phase_probe.py > gpurun_out/it_probe.log 2>&1; echo probe_rc=$?
cat gpurun_out/it_probe.log | grep mode
timeout 900 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/it_bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/it_bench.log | cut -c1-400
if [ -n "$PROBE_NCU" ]; then
  timeout 600 ncu --set full --import-source on -k regex:phase_probe -c 1 -f -o gpurun_out/it_probe \
    python tools/phase_probe.py --reps 1 --mode $PROBE_NCU > gpurun_out/it_probe_ncu.log 2>&1; echo ncu_rc=$?
fi
