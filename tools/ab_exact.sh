#!/bin/bash
# A/B of builds (build/var/libswr_<tag>.so) with tools/exact_time.py
for v in "$@"; do SWR_LIB=$PWD/build/var/libswr_$v.so timeout 200 python tools/exact_time.py 2>&1 | head -2 | sed "s/^/$v /"; done
