for pf in 0 1 2 3 4 6; do echo "pf=$pf"; PPPC_PF=$pf python tools/phase_probe.py --mode 1 2 2>&1 | grep mode; done
