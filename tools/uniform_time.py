"""Uniform-window forward (swr_uniform_fwd) time at the layer shape for k = 4, 16, 32 (L2 flushed)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2512_13921_b200 as P
from swr_inputs import swr_inputs
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn):
    for _ in range(3): fn()
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    return sorted(ts)[5]
g = {k: v.cuda() for k, v in swr_inputs(8, 4096, 16, 128, dtype=torch.bfloat16, seed=1).items()}
print(os.environ.get("SWR_LIB", "default")[-16:], " ".join(f"k={k}: {t(lambda: P.swr_uniform_fwd(g['u'], g['a'], k)):.0f}us" for k in (4, 16, 32)), flush=True)
