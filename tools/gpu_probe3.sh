#!/bin/bash
mkdir -p gpurun_out
for n in 100 32 25; do
  echo "== phase probe N=$n"; timeout 300 python tools/phase_probe.py --N $n 2>&1 | tail -3
  echo "== phase probe N=$n no L2 persist"; PPPC_NO_L2_PERSIST=1 timeout 300 python tools/phase_probe.py --N $n 2>&1 | tail -3
done
echo "== waves, no L2 persist"; PPPC_NO_L2_PERSIST=1 timeout 600 python tools/wave_probe.py --waves 100 32 25 2>&1
