#!/bin/bash
# BASELINE configs[4], N = 16, the first fine step of every subinterval to full Newton
# convergence (1e-10 rel / 1e-9 abs, max 50, backtracking), PCG 1e-12, lane engine.
O=gpurun_out/config4; mkdir -p $O
timeout 3300 python tools/config5_sizing.py --N 16 --fine-steps 1 --newton-max 50 --pcg-tol 1e-12 --pcg-max 50000 \
   --no-probes > $O/c4_n16_step1.jsonl 2> $O/c4_n16_step1.err; echo a_rc=$?; tail -c 1200 $O/c4_n16_step1.jsonl; tail -2 $O/c4_n16_step1.err
