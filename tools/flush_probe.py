"""fwd/bwd event times under different L2 flush recipes (write / write+read / none)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2512_13921_b200 as P
from swr_inputs import swr_inputs
s = {k: v.cuda() for k, v in swr_inputs(8, 4096, 16, 128, dtype=torch.bfloat16, seed=1).items()}
fl = torch.empty(64 << 20, device="cuda")
rd = torch.empty(64 << 20, device="cuda")
sink = torch.empty(1, device="cuda")
def w(): fl.zero_()
def wr(): fl.zero_(); sink.copy_(rd.sum())
def none(): pass
for name, f in [("write", w), ("write+read", wr), ("none", none), ("write", w)]:
    tf, tb = [], []
    for it in range(40):
        f()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(); P.swr_fwd(s["u"], s["a"]); e[1].record(); P.swr_bwd(s["u"], s["a"], s["G"]); e[2].record()
        torch.cuda.synchronize()
        if it >= 5: tf.append(e[0].elapsed_time(e[1]) * 1e3); tb.append(e[1].elapsed_time(e[2]) * 1e3)
    tf.sort(); tb.sort()
    print(f"{name:12s} fwd {tf[len(tf)//2]:.1f}us bwd {tb[len(tb)//2]:.1f}us", flush=True)
