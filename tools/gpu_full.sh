# full GPU pass: tests, smoke, bench lines, back-to-back probe, launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 300 python bench.py --steps 100 --warmup 10 > gpurun_out/bench_swr.json 2> gpurun_out/bench_swr.err; echo "bench rc=$?"
cat gpurun_out/bench_swr.json; tail -3 gpurun_out/bench_swr.err
timeout 300 python bench.py --steps 100 --warmup 10 --op mix --no-cpu-baseline > gpurun_out/bench_mix.json 2>&1; cat gpurun_out/bench_mix.json
timeout 300 python bench.py --steps 50 --warmup 10 --op layer --no-cpu-baseline > gpurun_out/bench_layer.json 2>&1; cat gpurun_out/bench_layer.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 10 -c 12 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu1 rc=$?"
