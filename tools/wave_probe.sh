#!/bin/bash
# Time per system-step of the fine batch as a function of the batch (wave) size.
mkdir -p gpurun_out
for n in ${WAVES:-8 16 25 32 50 100}; do
  timeout 600 python bench.py --steps 2 --warmup 1 --fine-steps ${FS:-2} --subintervals $n --no-cpu-baseline > gpurun_out/wave_$n.log 2>&1
  echo "N=$n rc=$? $(tail -1 gpurun_out/wave_$n.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"], d["roofline"]["frac"], d["solver"])' 2>&1)"
done
