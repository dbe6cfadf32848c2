# every bench config x op (back to back timing where inputs exceed 2x L2) -> gpurun_out/cfg_*.json
rm -f gpurun_out/cfg_*.json
run() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-extra "$@" 2>/dev/null | tail -1; }
for c in layer4k L8k L16k L32k L4k_b16 bxh paper_d16 layer4k_f32 tiny; do
  for op in swr mix layer; do
    run --config $c --op $op > gpurun_out/cfg_${c}_${op}.json
  done
done
for op in swr mix; do run --config layer4k --op $op --path ffma > gpurun_out/cfg_layer4k_${op}_ffma.json; done
ls gpurun_out/cfg_*.json | wc -l
