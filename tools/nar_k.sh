timeout 300 python -m pytest tests/test_narrow.py -x -q --timeout 120 2>&1 | tail -1
for v in k57 k30 k20 k16; do SWR_LIB=build/var/libswr_$v.so timeout 60 python tools/nar_time.py; done
