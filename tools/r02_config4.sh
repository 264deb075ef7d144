#!/bin/bash
# BASELINE configs[4] on one B200 (bounded): the first fine step of N = 16 with the real
# Newton / PCG 1e-12, then one Newton iteration (step solve to PCG 1e-12) at N = 64 and 256.
mkdir -p gpurun_out
case "$1" in
  a) timeout 3300 python tools/config5_sizing.py --N 16 --newton-max 50 --pcg-tol 1e-12 --pcg-max 50000 --no-probes \
       > gpurun_out/c4_n16.jsonl 2> gpurun_out/c4_n16.err; echo rc=$?; tail -2 gpurun_out/c4_n16.err ;;
  b) timeout 3300 python tools/config5_sizing.py --N 256 64 --newton-max 1 --pcg-tol 1e-12 --pcg-max 50000 \
       > gpurun_out/c4_n256_64.jsonl 2> gpurun_out/c4_n256_64.err; echo rc=$?; tail -2 gpurun_out/c4_n256_64.err ;;
esac
