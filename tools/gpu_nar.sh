# staged narrow-head backward: parity tests (FFMA family at d = 16 / 32) and bench lines
timeout 600 python -m pytest tests/test_parity.py tests/test_props.py tests/test_fuzz.py tests/test_graph.py -x -q --timeout 120 > gpurun_out/t_nar.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/t_nar.log
for op in swr mix; do
  timeout 300 python bench.py --config paper_d16 --op $op --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$op', round(d['value']/1e6,1), 'fwd', round(d['fwd_ms']*1e3,1), 'bwd', round(d['bwd_ms']*1e3,1), d['hbm_gbs'])"
done
