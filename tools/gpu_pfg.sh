#!/bin/bash
for lib in paper_1905_13076_b200/libpppc_b200.so variants/pfg.so; do
 for pf in 1 2 4; do
  echo "lib=$lib PF=$pf"; PPPC_LIB=$lib PPPC_PF=$pf timeout 300 python tools/phase_probe.py --mode 1 1 2>&1 | tail -1
 done
done
for lib in paper_1905_13076_b200/libpppc_b200.so variants/pfg.so; do
 for pf in 0 2; do echo "wave lib=$lib PF=$pf"; PPPC_LIB=$lib PPPC_PF=$pf timeout 600 python tools/wave_probe.py --waves 100 2>&1 | tail -1; done
done
