#!/bin/bash
# COCG change check: spectral parity tests and the configs[2] coarse solve
timeout 900 python -m pytest tests -m gpu -x -q -k "multiharmonic or pppc or harmonic or files or cyclic" 2>&1 | tail -2
timeout 900 python bench_extra.py config3 config3full --no-cpu 2>&1 | python -c 'import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d["bins"], d["kernel_ms"], d["frac"], d["lockstep_iterations"])'
