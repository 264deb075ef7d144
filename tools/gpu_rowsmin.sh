#!/bin/bash
for rm in 64 32 16; do echo "ROWS_MIN=$rm"; PPPC_ROWS_MIN=$rm timeout 600 python bench_extra.py config1 --no-cpu 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print("config1", d["wall_s"], d["fine_ms"], d["coarse_ms"], d["iterations"])'; done
