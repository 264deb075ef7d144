#!/bin/bash
# BASELINE configs[4] on one B200 (k2 = 4.0, I0 = 8000 A, d = 4,093,953), lane engine:
#  a) N = 16: the first fine step of every subinterval to full Newton convergence
#     (1e-10 rel / 1e-9 abs, max 50, backtracking), PCG 1e-12 -> Newton / PCG counts
#  b) N = 64 and 256: one Newton iteration of the first fine step at PCG 1e-12
#     (memory fit and throughput at scale)
#  c) N = 16: all 10 fine steps of every subinterval -> DOF-timesteps/s
O=gpurun_out/config4; mkdir -p $O
timeout 1500 python tools/config5_sizing.py --N 16 --fine-steps 1 --newton-max 50 --pcg-tol 1e-12 --pcg-max 50000 \
   --no-probes > $O/c4_n16_step1.jsonl 2> $O/c4_n16_step1.err; echo a_rc=$?; tail -c 1200 $O/c4_n16_step1.jsonl; tail -2 $O/c4_n16_step1.err
timeout 1500 python tools/config5_sizing.py --N 64 256 --newton-max 1 --pcg-tol 1e-12 --pcg-max 50000 \
   > $O/c4_n64_256.jsonl 2> $O/c4_n64_256.err; echo b_rc=$?; tail -c 2500 $O/c4_n64_256.jsonl; tail -2 $O/c4_n64_256.err
timeout 3300 python tools/config5_sizing.py --N 16 --fine-steps 10 --newton-max 50 --pcg-tol 1e-12 --pcg-max 50000 \
   --no-probes > $O/c4_n16_10steps.jsonl 2> $O/c4_n16_10steps.err; echo c_rc=$?; tail -c 1200 $O/c4_n16_10steps.jsonl; tail -2 $O/c4_n16_10steps.err
