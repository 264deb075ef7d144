#!/bin/bash
PPPC_SEQ=1 timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" 2>&1 | tail -2
for sq in 1 0; do echo "SEQ=$sq"; PPPC_SEQ=$sq timeout 600 python tools/wave_probe.py --waves 100 2>&1 | tail -1; done
PPPC_SEQ=1 PPPC_DEBUG_TIMING=1 timeout 600 python tools/wave_probe.py --waves 100 2>&1 | head -3
