# round-2 (second half) profiles: launch list of the default bench command, full captures of
# the paired layer backward on the tensor cores (layer4k, G = 8) and of the staged narrow-head
# backward at the paper's head shape (d = 16, h = 128): SWR, mixer, layer (G = 8)
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extra"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02b_launches.csv $B > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:swr_tc_kernel -s 6 -c 2 -o gpurun_out/r02b_layer_full $B --op layer > gpurun_out/ncu_l.log 2>&1; echo "layer full rc=$?"
for op in swr mix layer; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_stream|bwd_staged" -s 6 -c 2 -o gpurun_out/r02b_d16${op}_full $B --config paper_d16 --op $op > gpurun_out/ncu_d16$op.log 2>&1; echo "d16 $op full rc=$?"
done
