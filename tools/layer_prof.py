"""One launch each of the TC mixer backward and the TC layer backward (logits off, on),
for ncu: ncu -k regex:swr_tc_kernel python tools/layer_prof.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2512_13921_b200 as P
from swr_inputs import layer_inputs

g = {k: v.cuda() for k, v in layer_inputs(8, 4096, 16, 128, dtype=torch.bfloat16, seed=1).items()}
for _ in range(3):
    P.phalanx_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"])
    P.phalanx_layer_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"], logit_a=False, logit_k=False)
    P.phalanx_layer_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"])
torch.cuda.synchronize()
