set -x
timeout 900 python -m pytest tests/test_layer.py -x -q --timeout 60 > gpurun_out/t_layer.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/t_layer.log
timeout 120 python tools/layer_time.py > gpurun_out/layer_time.txt 2>&1; cat gpurun_out/layer_time.txt
