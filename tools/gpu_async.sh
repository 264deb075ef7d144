#!/bin/bash
for n in 100 32; do
  echo "-- N=$n"; timeout 300 python tools/phase_probe.py --N $n --mode 1 4 1 4 2>&1 | tail -4
done
