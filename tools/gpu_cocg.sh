#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "multiharmonic or pppc or dft or jump or harmonic" > gpurun_out/pytest_cocg.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_cocg.log
timeout 900 python bench_extra.py config3 config3full --no-cpu > gpurun_out/bench_c3.log 2>&1; echo c3_rc=$?
cut -c1-700 gpurun_out/bench_c3.log
