#!/bin/bash
# ownership x cache-hint variants: phase probes (N=100, N=32) and the 2-step wave probe
mkdir -p gpurun_out
for lib in paper_1905_13076_b200/libpppc_b200.so variants/hints.so; do
  for ct in 0 1; do
    echo "=== lib=$lib contig=$ct"
    for n in 100 32; do
      echo "-- phase probe N=$n"; PPPC_LIB=$lib PPPC_CONTIG=$ct timeout 300 python tools/phase_probe.py --N $n --mode 1 2 2>&1 | tail -2
    done
    PPPC_LIB=$lib PPPC_CONTIG=$ct timeout 600 python tools/wave_probe.py --waves 100 25 2>&1 | tail -2
  done
done
