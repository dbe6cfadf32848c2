"""One swr_exact_fwd at the layer shape, for ncu's launch list (kernel times of the
tensor-core first pass, the look-back scan and the output pass)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2512_13921_b200 as P
from swr_inputs import swr_inputs

B, L = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (8, 4096)
g = {k: v.cuda() for k, v in swr_inputs(B, L, 16, 128, dtype=torch.bfloat16, seed=1).items()}
for _ in range(4):
    P.swr_exact_fwd(g["u"], g["a"])
torch.cuda.synchronize()
