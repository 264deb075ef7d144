#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q -k "multiharmonic or pppc or harmonic or files" 2>&1 | tail -3
timeout 900 python bench_extra.py config3 config3full --no-cpu 2>&1 | cut -c1-600
