#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -x -q -k "not fullsize" 2>&1 | tail -2
timeout 600 python bench_extra.py config1 --no-cpu 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print("config1", d["wall_s"], d["fine_ms"], d["iterations"])'
timeout 600 python tools/wave_probe.py --waves 100 2>&1 | tail -1
