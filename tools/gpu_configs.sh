#!/bin/bash
# bench lines for every single-GPU config (no cpu baseline / e2e), one JSON line each
for c in layer4k L8k L16k L32k L4k_b16 paper_d16 layer4k_f32; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/cfg_$c.json
done
for c in layer4k L32k paper_d16 layer4k_f32; do
  timeout 300 python bench.py --config $c --op mix --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/cfgmix_$c.json
done
# the FFMA family on the graded bf16 shape, for comparison with the tensor-core path
timeout 300 python bench.py --config layer4k --path ffma --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/cfgffma_layer4k.json
timeout 300 python bench.py --config layer4k --op mix --path ffma --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/cfgffmamix_layer4k.json
