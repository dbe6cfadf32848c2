#!/bin/bash
# one ncu --set full capture of the TC kernels (fwd, bwd; mix with MIX=1) on the bench config
K=${K:-regex:swr_tc_kernel}
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -s ${S:-2} -c ${C:-2} -o gpurun_out/prof_${TAG:-tc} \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${ARGS} > gpurun_out/ncu_${TAG:-tc}.log 2>&1; echo "ncu rc=$?"
