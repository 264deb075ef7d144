#!/bin/bash
mkdir -p gpurun_out
for sq in 1 0 1; do PPPC_SEQ=$sq timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_seq$sq.log 2>&1; echo "SEQ=$sq $(tail -1 gpurun_out/bench_seq$sq.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"], d["e2e"]["value"], d["roofline"]["frac"], d["solver"]["lockstep_pcg_iterations"])')"; done
