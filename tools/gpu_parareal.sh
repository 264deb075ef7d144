#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "parareal or pp_ic" 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" 2>&1 | tail -2
