#!/bin/bash
# build/var/libswr_<tag>.so with extra nvcc flags (A/B experiments; load with SWR_LIB=...)
tag=$1; shift
cd "$(dirname "$0")/.."
mkdir -p build/var
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr "$@" \
  -shared -o build/var/libswr_$tag.so paper_2512_13921_b200/csrc/*.cu -I include 2>&1 | grep -iE "error|warning" || true
