set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 300 python bench.py --steps 100 --warmup 10 > gpurun_out/bench_swr.json 2> gpurun_out/bench_swr.err; echo "bench rc=$?"
cat gpurun_out/bench_swr.json
timeout 300 python bench.py --steps 100 --warmup 10 --op mix --no-cpu-baseline > gpurun_out/bench_mix.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 10 -c 12 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:swr_tc_kernel -s 2 -c 2 -o gpurun_out/prof_tc_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
