"""One paper-shape layer backward (d=16, h=128, G groups) for ncu: python tools/nar_layer_prof.py [G]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2512_13921_b200 as P
from swr_inputs import layer_inputs

G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
g = {k: v.cuda() for k, v in layer_inputs(8, 8192, 128, 16, G, G, dtype=torch.bfloat16, seed=1).items()}
for _ in range(2):
    P.phalanx_layer_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"])
torch.cuda.synchronize()
