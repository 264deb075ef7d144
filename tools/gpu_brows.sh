#!/bin/bash
PPPC_BROWS=1 timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" 2>&1 | tail -2
for b in 0 1; do echo "BROWS=$b"; PPPC_BROWS=$b timeout 300 python tools/phase_probe.py --mode 2 2 2>&1 | tail -1; PPPC_BROWS=$b timeout 600 python tools/wave_probe.py --waves 100 2>&1 | tail -1; done
for b in 0 1; do echo "BROWS=$b config5 N=64"; PPPC_BROWS=$b timeout 600 python tools/config5_sizing.py --N 64 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["kernel_ms"], d["pcg_iterations"], d["algorithmic_GBps"], d["phase_probes"])'; done
