# staged narrow-head backward against the register-staged kernels (SWR_NAR_OFF build)
for D in 16 32; do for v in main off; do L=build/var/libswr_$v.so; [ $v = main ] && L=paper_2512_13921_b200/libswr.so
  SWR_LIB=$L timeout 60 python tools/nar_time.py 8 8192 $((2048 / D)) $D; done; done
for v in main off; do L=build/var/libswr_$v.so; [ $v = main ] && L=paper_2512_13921_b200/libswr.so
  echo $v; SWR_LIB=$L timeout 100 python tools/layer_time.py 8 8192 128 16 2>&1 | grep 'path 0' | grep -v mix_bwd; done
