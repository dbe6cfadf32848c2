import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2512_13921_b200 as P
from swr_inputs import swr_inputs
op = sys.argv[1]
P.set_path(P.SWR_PATH_TC)
g = {k: v.cuda() for k, v in swr_inputs(8, 4096, 16, 128, seed=1).items()}
flush = torch.empty(64 << 20, device="cuda")
for it in range(60):
    flush.zero_()
    if op in ("fwd", "both"): P.swr_fwd(g["u"], g["a"])
    if op in ("bwd", "both"): P.swr_bwd(g["u"], g["a"], g["G"])
try:
    torch.cuda.synchronize(); print(op, "OK")
except Exception as e:
    print(op, "FAIL", str(e)[:80])
