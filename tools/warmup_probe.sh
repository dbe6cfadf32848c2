for i in 1 2 3; do for w in 3 10 30; do
  echo "w=$w $(timeout 200 python bench.py --steps 50 --warmup $w --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), round(d['fwd_ms']*1e3,1), round(d['bwd_ms']*1e3,1))")"
done; done
