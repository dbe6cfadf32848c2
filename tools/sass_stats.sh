#!/bin/bash
# static SASS opcode counts of the TC kernels in libswr.so (proxy for instruction mix)
for op in 0 1 2 3; do
  cuobjdump -sass -fun "_ZN3swr2tc13swr_tc_kernelILi${op}EEEvNS0_4MapsENS_6ParamsE" ${1:-paper_2512_13921_b200/libswr.so} \
   | grep -E "^\s+/\*[0-9a-f]+\*/" | awk '{op=$2; if (op ~ /^@/) op=$3; sub(/\..*/,"",op); sub(/;/,"",op); c[op]++; n++} END {printf "OP'$op' total %d:", n; for (k in c) if (c[k] > 25) printf " %s=%d", k, c[k]; print ""}'
done
