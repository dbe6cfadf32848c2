#!/bin/bash
# A/B: default build vs build/var/libswr_$1.so, bench.py value alternated 3x
for i in 1 2 3; do
  for v in default "$@"; do
    if [ "$v" = default ]; then unset SWR_LIB; else export SWR_LIB=$PWD/build/var/libswr_$v.so; fi
    echo "$v $(timeout 200 python bench.py --steps 50 --warmup 10 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), round(d['fwd_ms']*1e3,1), round(d['bwd_ms']*1e3,1))")"
  done
done
unset SWR_LIB
