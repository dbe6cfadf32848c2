#!/bin/bash
# parity probe of the TC path, GPU tests, per-kernel times (CUDA events, L2 flushed)
timeout 120 python tests/tc_check.py 2 100 2>&1 | tail -4
timeout 120 python tests/tc_check.py 8 515 2>&1 | tail -4
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 120 python tools/ktime.py 2>&1 | tail -1
timeout 120 python tools/ktime.py 2>&1 | tail -1
