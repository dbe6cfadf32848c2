# parity after the ring-depth change, b2b traces, bench, d16 FFMA bwd profile
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for op in fwd bwd; do SWR_LIB=$PWD/build/var/libswr_trace.so B2B=1 timeout 120 python tools/tc_trace.py $op 2>&1 | grep -v "^span\|^ *[0-9]" ; done > gpurun_out/trace_b2b.txt; cat gpurun_out/trace_b2b.txt
timeout 600 python bench.py --steps 50 --warmup 10 > gpurun_out/bench_swr.json 2> gpurun_out/bench_swr.err; echo "bench rc=$?"; cat gpurun_out/bench_swr.json; tail -3 gpurun_out/bench_swr.err
timeout 300 python bench.py --config paper_d16 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_d16.json 2>&1; cat gpurun_out/bench_d16.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_ffma_vec -s 3 -c 1 -o gpurun_out/prof_d16_bwd python bench.py --config paper_d16 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_d16.log 2>&1; echo "ncu rc=$?"
