set -x
timeout 60 python tools/tc_check.py 1 32 fwd; echo rc=$?
timeout 60 python tools/tc_check.py 2 100; echo rc=$?
timeout 120 python tools/tc_check.py 8 4096; echo rc=$?
timeout 300 python bench.py --steps 50 --warmup 5 --path tc --no-cpu-baseline --no-e2e; echo rc=$?
timeout 300 python bench.py --steps 50 --warmup 5 --path tc --op mix --no-cpu-baseline --no-e2e; echo rc=$?
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
