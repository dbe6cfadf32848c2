#!/bin/bash
# A/B of FFMA-path builds (build/var/libswr_<tag>.so) with tools/ffma_time.py, alternated twice
for i in 1 2; do for v in "$@"; do SWR_LIB=$PWD/build/var/libswr_$v.so timeout 120 python tools/ffma_time.py 2>&1 | tail -1 | sed "s/^/$v /"; done; done
