timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python tools/host_cost.py swr 2>&1 | grep -v Trace
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_swr.json 2> gpurun_out/bench_swr.err; echo "bench rc=$?"; cat gpurun_out/bench_swr.json; tail -3 gpurun_out/bench_swr.err
timeout 300 python bench.py --config paper_d16 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_d16.json 2>&1; cat gpurun_out/bench_d16.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_ffma_vec -s 3 -c 1 -o gpurun_out/prof_d16_bwd2 python bench.py --config paper_d16 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/ncu_d16.log 2>&1; echo "ncu rc=$?"
