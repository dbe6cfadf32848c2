set -x
timeout 60 python tools/tc_check.py 1 32 fwd; echo rc=$?
timeout 60 python tools/tc_check.py 2 100 fwd,bwd; echo rc=$?
timeout 60 python tools/tc_check.py 2 100 mixf,mixb; echo rc=$?
timeout 120 python tools/tc_check.py 8 4096; echo rc=$?
