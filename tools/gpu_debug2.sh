for i in 1 2 3 4 5; do timeout 120 python bench.py --steps 20 --warmup 3 --path tc --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-120; done
timeout 600 compute-sanitizer --tool synccheck python tools/tc_check.py 8 512 fwd,bwd 2>&1 | tail -6
