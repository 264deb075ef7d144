#!/bin/bash
mkdir -p gpurun_out
PPPC_SEQ=1 timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_seq.log 2>&1; echo pytest_seq_rc=$?
tail -3 gpurun_out/pytest_seq.log
timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_conc.log 2>&1; echo pytest_conc_rc=$?
tail -2 gpurun_out/pytest_conc.log
for sq in 0 1; do echo "SEQ=$sq"; PPPC_SEQ=$sq timeout 600 python tools/wave_probe.py --waves 100 2>&1 | tail -1; done
PPPC_SEQ=1 PPPC_DEBUG_TIMING=1 timeout 600 python tools/wave_probe.py --waves 100 > gpurun_out/dbg_seq.log 2>&1; head -12 gpurun_out/dbg_seq.log
