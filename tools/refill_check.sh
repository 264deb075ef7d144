#!/bin/bash
# refill-path change check: parity, 2-step wave timing, per-interval timing
timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" 2>&1 | tail -2
timeout 600 python tools/wave_probe.py --waves 100 2>&1 | tail -1
PPPC_DEBUG_TIMING=1 timeout 600 python tools/wave_probe.py --waves 100 2>&1 | head -3
