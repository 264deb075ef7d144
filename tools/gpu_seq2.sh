#!/bin/bash
for sq in 1 0; do echo "SEQ=$sq"; PPPC_SEQ=$sq timeout 600 python tools/wave_probe.py --waves 100 2>&1 | tail -1; done
PPPC_SEQ=1 PPPC_DEBUG_TIMING=1 timeout 600 python tools/wave_probe.py --waves 100 2>&1 | head -3
