#!/bin/bash
# bench lines for every single-GPU config (no cpu baseline / e2e), one JSON line each
for c in layer4k L8k L16k L32k L4k_b16 paper_d16; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/cfg_$c.json
done
for c in layer4k L32k paper_d16; do
  timeout 300 python bench.py --config $c --op mix --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/cfgmix_$c.json
done
