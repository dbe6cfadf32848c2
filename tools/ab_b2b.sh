#!/bin/bash
# A/B of back-to-back step times: default build vs build/var/libswr_<tag>.so, alternated 3x
# usage: tools/ab_b2b.sh [op] tag1 tag2 ...
op=swr
if [ "$1" = swr ] || [ "$1" = mix ]; then op=$1; shift; fi
for i in 1 2 3; do
  for v in default "$@"; do
    if [ "$v" = default ]; then unset SWR_LIB; else export SWR_LIB=$PWD/build/var/libswr_$v.so; fi
    timeout 120 python tools/b2b_step.py $op
  done
done
unset SWR_LIB
