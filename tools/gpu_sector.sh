#!/bin/bash
PPPC_SEQ=1 PPPC_SECTOR=1 timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" 2>&1 | tail -2
for v in "1 0" "1 1"; do set -- $v; echo "SEQ=$1 SECTOR=$2"; PPPC_SEQ=$1 PPPC_SECTOR=$2 timeout 600 python tools/wave_probe.py --waves 100 2>&1 | tail -1; done
PPPC_SEQ=1 PPPC_SECTOR=1 PPPC_DEBUG_TIMING=1 timeout 600 python tools/wave_probe.py --waves 100 2>&1 | head -3
