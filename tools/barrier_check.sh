#!/bin/bash
# group-barrier diagnostics: per-interval work / wait / arrival-to-release (2 fine steps)
for sq in 0 1; do echo "SEQ=$sq"; PPPC_SEQ=$sq PPPC_DEBUG_TIMING=1 timeout 600 python tools/wave_probe.py --waves 100 2>&1 | head -3; done
