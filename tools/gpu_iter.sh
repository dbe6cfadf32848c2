#!/bin/bash
# quick iteration: parity check, fault probe, per-kernel times (default build + variants)
timeout 300 python tools/tc_check.py 8 515 2>&1 | tail -4
N=3 OP=fwd bash tools/gpu_var.sh default 2>/dev/null; N=3 OP=bwd bash tools/gpu_var.sh default 2>/dev/null
timeout 120 python tools/ktime.py 2>&1 | tail -1
for v in "$@"; do SWR_LIB=$PWD/build/var/libswr_$v.so timeout 120 python tools/ktime.py 2>&1 | tail -1; done
