#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -x -q -k "not fullsize" 2>&1 | tail -3
for cl in 1 0 1; do echo "CLUSTER=$cl"; PPPC_CLUSTER=$cl timeout 600 python bench_extra.py config1 --no-cpu 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["wall_s"], d["fine_ms"], d["coarse_ms"], d["spectral_ms"], d["iterations"], d["jumps"][-1])'; done
