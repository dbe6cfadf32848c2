set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_swr.json 2> gpurun_out/bench_swr.err; echo "bench rc=$?"
cat gpurun_out/bench_swr.json; tail -3 gpurun_out/bench_swr.err
timeout 300 python bench.py --steps 20 --warmup 5 --op mix --no-cpu-baseline > gpurun_out/bench_mix.json 2>&1; echo "bench mix rc=$?"
cat gpurun_out/bench_mix.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_ffma -s 2 -c 1 -o gpurun_out/prof_bwd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bwd.log 2>&1; echo "ncu2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_ffma -s 2 -c 1 -o gpurun_out/prof_fwd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_fwd.log 2>&1; echo "ncu3 rc=$?"
