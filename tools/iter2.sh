#!/bin/bash
# GPU parity (fast set) then the debug-timing run.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/it_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/it_tests.log
bash tools/dbg_run.sh
