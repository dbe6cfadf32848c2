# TC layer backward (pairs of heads, layer4k G = 8) ring / warp-count variants, back to back
for v in main ${VARS}; do L=build/var/libswr_$v.so; [ $v = main ] && L=paper_2512_13921_b200/libswr.so
  echo -n "$v: "; SWR_LIB=$L timeout 60 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2512_13921_b200 as P
from swr_inputs import layer_inputs
g={k:v.cuda() for k,v in layer_inputs(8,4096,16,128,8,8,dtype=torch.bfloat16,seed=1).items()}
f=lambda: P.phalanx_layer_mix_bwd(g['q'],g['zk'],g['v'],g['za'],g['dy'])
for _ in range(5): f()
torch.cuda.synchronize(); e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): f()
e1.record(); torch.cuda.synchronize(); print(round(e0.elapsed_time(e1)*50,1),'us', P.last_path())
"; done
