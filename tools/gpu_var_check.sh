#!/bin/bash
# parity probe + kernel times of the default build and each build/var/libswr_<tag>.so given
timeout 100 python tests/tc_check.py 2 100 2>&1 | tail -4
timeout 100 python tools/ktime.py 2>&1 | tail -1
for v in "$@"; do
  SWR_LIB=$PWD/build/var/libswr_$v.so timeout 100 python tests/tc_check.py 2 100 2>&1 | tail -4
  SWR_LIB=$PWD/build/var/libswr_$v.so timeout 100 python tools/ktime.py 2>&1 | tail -1
done
