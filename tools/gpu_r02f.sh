compute-sanitizer --tool racecheck tools/mbar_race_probe > gpurun_out/san_racecheck_mbar_probe.log 2>&1; tail -5 gpurun_out/san_racecheck_mbar_probe.log
timeout 900 python -m pytest tests/test_parity.py tests/test_props.py tests/test_layer.py tests/test_decode.py -m gpu -x -q 2>&1 | tail -2
for v in base mixg2 mixg8 default; do
  if [ $v = default ]; then unset SWR_LIB; else export SWR_LIB=$PWD/build/var/libswr_$v.so; fi
  for c in paper_d16 layer4k_f32; do timeout 300 python bench.py --config $c --op mix --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v mix $c', round(d['value']/1e6,1), 'Mtok/s fwd', round(d['fwd_ms']*1e3,1), 'bwd', round(d['bwd_ms']*1e3,1), 'us', d['config']['last_path'])"; done
done
unset SWR_LIB
for c in paper_d16 layer4k_f32; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('swr $c', round(d['value']/1e6,1), 'Mtok/s fwd', round(d['fwd_ms']*1e3,1), 'bwd', round(d['bwd_ms']*1e3,1), 'us', d['config']['last_path'])"; done
