timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python __graft_entry__.py smoke 2>&1 | tail -1 | cut -c1-300
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_swr.json 2> gpurun_out/bench_swr.err; echo "bench rc=$?"; cat gpurun_out/bench_swr.json; tail -3 gpurun_out/bench_swr.err
for c in paper_d16 layer4k_f32; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']/1e6,1), 'Mtok/s fwd', round(d['fwd_ms']*1e3,1), 'bwd', round(d['bwd_ms']*1e3,1), 'us', d['config']['last_path'])"; done
timeout 300 python bench.py --op mix --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-extra > gpurun_out/bench_mix.json 2>&1; cat gpurun_out/bench_mix.json | cut -c1-600
for t in memcheck racecheck synccheck initcheck; do echo "== $t"; timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py ext 2>&1 | tail -12; done > gpurun_out/sanitizer.txt 2>&1; cat gpurun_out/sanitizer.txt
