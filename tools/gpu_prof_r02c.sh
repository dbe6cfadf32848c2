# final captures of the staged narrow-head backward at d = 16 (mixer and layer after the FFMA2 change)
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extra"
for op in mix layer; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bwd_staged" -s 3 -c 1 -o gpurun_out/r02c_d16${op}_full $B --config paper_d16 --op $op > gpurun_out/ncu_c$op.log 2>&1; echo "d16 $op rc=$?"
done
