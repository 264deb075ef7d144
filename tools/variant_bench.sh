#!/bin/bash
# Time kernel variants (variants/*.so) on a shortened config-2 bench run.
for v in ${VARIANTS:-$(ls variants/*.so)}; do
  r=$(PPPC_LIB=$v timeout 600 python bench.py --no-cpu-baseline --steps 1 --warmup 1 ${VB_ARGS:---fine-steps 2} 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['solver']['lockstep_pcg_iterations'])" 2>&1)
  echo "$v $r"
done
