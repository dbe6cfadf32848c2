for op in fwd bwd mixf mixb; do timeout 120 python tools/tc_trace.py $op; done
