"""fwd and bwd timed back to back (the bench step) and each alone after an L2 flush."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2512_13921_b200 as P
from swr_inputs import swr_inputs, mix_inputs
op = sys.argv[1] if len(sys.argv) > 1 else "swr"
B, L, H, D = 8, 4096, 16, 128
if op == "swr":
    g = {k: v.cuda() for k, v in swr_inputs(B, L, H, D, dtype=torch.bfloat16, seed=1).items()}
    f = lambda: P.swr_fwd(g["u"], g["a"]); b = lambda: P.swr_bwd(g["u"], g["a"], g["G"])
else:
    g = {k: v.cuda() for k, v in mix_inputs(B, L, H, D, dtype=torch.bfloat16, seed=1).items()}
    f = lambda: P.phalanx_mix(g["q"], g["k"], g["v"], g["a"]); b = lambda: P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.zeros(64 << 20, device="cuda"); sink = torch.empty(1, device="cuda")
def fl(): flush.zero_(); sink.copy_(rd.sum())
for _ in range(3): fl(); f(); b()
E = lambda: torch.cuda.Event(enable_timing=True)
tf, tb, ta, tb2 = [], [], [], []
for _ in range(20):
    fl(); e = [E() for _ in range(3)]
    e[0].record(); f(); e[1].record(); b(); e[2].record(); torch.cuda.synchronize()
    tf.append(e[0].elapsed_time(e[1]) * 1e3); tb.append(e[1].elapsed_time(e[2]) * 1e3)
    fl(); e = [E() for _ in range(2)]
    e[0].record(); b(); e[1].record(); torch.cuda.synchronize(); tb2.append(e[0].elapsed_time(e[1]) * 1e3)
med = lambda x: sorted(x)[len(x) // 2]
print(f"{os.path.basename(os.environ.get('SWR_LIB', 'default'))} {op} step: fwd {med(tf):.1f} + bwd {med(tb):.1f} = {med(tf)+med(tb):.1f} us"
      f" ({B*L/(med(tf)+med(tb))/1e0:.1f} Mtok/s); bwd alone {med(tb2):.1f} us", flush=True)
