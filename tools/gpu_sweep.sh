#!/bin/bash
# per-kernel times of each variant build (tools/ktime.py), then the fault probe on the default build
for v in "$@"; do SWR_LIB=$PWD/build/var/libswr_$v.so timeout 120 python tools/ktime.py 2>&1 | tail -1; done
timeout 120 python tools/ktime.py 2>&1 | tail -1
N=6 OP=fwd bash tools/gpu_var.sh a; N=4 OP=bwd bash tools/gpu_var.sh a
timeout 300 python tools/tc_check.py 8 515 2>&1 | tail -4
