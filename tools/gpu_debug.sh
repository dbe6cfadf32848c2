for i in 1 2 3; do CUDA_LAUNCH_BLOCKING=1 timeout 120 python bench.py --steps 20 --warmup 3 --path tc --no-cpu-baseline --no-e2e 2>&1 | tail -2 | cut -c1-300; done
CUDA_LAUNCH_BLOCKING=1 timeout 120 python bench.py --steps 20 --warmup 3 --path tc --op mix --no-cpu-baseline --no-e2e 2>&1 | tail -2 | cut -c1-200
timeout 300 compute-sanitizer --tool memcheck python tools/tc_check.py 2 100 2>&1 | tail -15
