timeout 60 python tools/tc_check.py 2 100 || exit 1
timeout 120 python tools/tc_check.py 8 4096 || exit 1
for op in fwd bwd mixf mixb; do timeout 120 python tools/tc_trace.py $op 2>&1 | grep -v "^ *[0-9]"; done
timeout 300 python bench.py --steps 50 --warmup 5 --path tc --no-cpu-baseline --no-e2e
timeout 300 python bench.py --steps 50 --warmup 5 --path tc --op mix --no-cpu-baseline --no-e2e
