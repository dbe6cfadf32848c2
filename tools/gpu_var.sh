#!/bin/bash
# run the fwd race probe against each variant build, N times each
N=${N:-4}
for v in "$@"; do
  ok=0; fail=0
  for i in $(seq $N); do
    r=$( ([ "$v" = default ] || export SWR_LIB=$PWD/build/var/libswr_$v.so; timeout 120 python tools/race_probe.py ${OP:-fwd}) 2>&1 | grep -E "OK|FAIL" | tail -1)
    case "$r" in *OK*) ok=$((ok+1));; *) fail=$((fail+1));; esac
  done
  echo "$v ok=$ok fail=$fail"
done
