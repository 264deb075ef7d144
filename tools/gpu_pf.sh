#!/bin/bash
for pf in 0 2 4 8; do
  echo "PF=$pf"; PPPC_PF=$pf timeout 600 python tools/wave_probe.py --waves 100 2>&1 | tail -1
done
