set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
for path in tc ffma; do
  timeout 300 python bench.py --steps 50 --warmup 5 --path $path --no-cpu-baseline > gpurun_out/bench_swr_$path.json 2>&1; echo "bench $path rc=$?"
  cat gpurun_out/bench_swr_$path.json
  timeout 300 python bench.py --steps 50 --warmup 5 --op mix --path $path --no-cpu-baseline --no-e2e > gpurun_out/bench_mix_$path.json 2>&1
  cat gpurun_out/bench_mix_$path.json
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tc.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:swr_tc_kernel -s 2 -c 2 -o gpurun_out/prof_tc python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_tc.log 2>&1; echo "ncu2 rc=$?"
