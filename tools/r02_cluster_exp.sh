#!/bin/bash
# Cluster engine: parity tests + bench step of the current library, then the
# timing-only experiment builds (PPPC_CL_EXP: results are wrong by design; only
# the cycle counters of PPPC_DEBUG_TIMING are read) on one wave of 15 systems.
mkdir -p gpurun_out
CL_VARIANTS="main" CL_SIZES="0" bash tools/r02_cluster_check.sh
grep -h "cluster timing" gpurun_out/cl_bench_main_0.log | tail -1
W="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --subintervals 15 --fine-steps 1 --e2e-steps 0"
PPPC_DEBUG_TIMING=1 timeout -k 10 300 $W > gpurun_out/cl_exp_base.log 2>&1; echo base_rc=$?
grep -h "cluster timing" gpurun_out/cl_exp_base.log | tail -1
for e in ${CL_EXPS:-1 2 4 6}; do
  PPPC_LIB=xvariants/cl_exp$e.so PPPC_DEBUG_TIMING=1 timeout -k 10 300 $W > gpurun_out/cl_exp_$e.log 2>&1; echo exp${e}_rc=$?
  grep -h "cluster timing" gpurun_out/cl_exp_$e.log | tail -1
done
