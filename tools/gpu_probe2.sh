#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/phase_probe.py > gpurun_out/probe_plain.log 2>&1; echo probe_rc=$?
cat gpurun_out/probe_plain.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:phase_probe -c 3 -o gpurun_out/probe_full python tools/phase_probe.py --reps 1 > gpurun_out/probe_ncu.log 2>&1; echo probe_ncu_rc=$?
tail -3 gpurun_out/probe_ncu.log
