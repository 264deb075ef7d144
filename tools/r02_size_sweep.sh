#!/bin/bash
# Cluster engine against the lane engine across mesh sizes (100 subintervals x 5 fine
# steps each, bench settings otherwise): where the automatic choice pays.
mkdir -p gpurun_out
for m in "100 128" "200 256" "300 256" "400 256"; do
  set -- $m
  for e in cluster lane; do
    PPPC_ENGINE=$e PPPC_DEBUG_TIMING=1 timeout -k 10 900 python bench.py --nr $1 --ntheta $2 --fine-steps 5 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/sweep_$1x$2_$e.log 2>&1
    echo "nr=$1 ntheta=$2 engine=$e rc=$?"
    grep "pppc cluster\]" gpurun_out/sweep_$1x$2_$e.log | head -1
    tail -1 gpurun_out/sweep_$1x$2_$e.log | python3 -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print(json.dumps({'nr':$1,'ntheta':$2,'dof':d['config']['dof'],'requested':'$e','engine':d.get('engine'),'ms_per_step':d['ms_per_step'],'dof_timesteps_per_s':d['value'],'pcg_iterations':d['solver']['pcg_iterations'],'canonical_frac':d['roofline']['frac']}))
except Exception as ex: print('no json', ex)" | tee -a gpurun_out/r02g_size_sweep.jsonl
  done
done
