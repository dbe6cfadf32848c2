"""FFMA-path kernel times at the paper's head shape (d=16, h=128) and fp32 layer shape (MIX=1: the mixer)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2512_13921_b200 as P
from swr_inputs import swr_inputs, mix_inputs
P.set_path(P.SWR_PATH_FFMA)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.zeros(64 << 20, device="cuda"); sink = torch.empty(1, device="cuda")
def t(fn):
    for _ in range(3): fn()
    ts = []
    for _ in range(10):
        flush.zero_(); sink.copy_(rd.sum())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    return sorted(ts)[len(ts) // 2]
out = []
for (B, L, H, D, dt) in [(8, 8192, 128, 16, torch.bfloat16), (8, 4096, 16, 128, torch.float32)]:
    g = {k: v.cuda() for k, v in swr_inputs(B, L, H, D, dtype=dt, seed=1).items()}
    e = 2 if dt == torch.bfloat16 else 4
    n = B * L * H
    if os.environ.get("MIX"):
        g = {k: v.cuda() for k, v in mix_inputs(B, L, H, D, dtype=dt, seed=1).items()}
        tf = t(lambda: P.phalanx_mix(g["q"], g["k"], g["v"], g["a"]))
        tb = t(lambda: P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"]))
        bf, bb = (4 * D + 1) * e, (7 * D + 2) * e
    else:
        tf = t(lambda: P.swr_fwd(g["u"], g["a"])); tb = t(lambda: P.swr_bwd(g["u"], g["a"], g["G"]))
        bf, bb = (2 * D + 1) * e, (3 * D + 2) * e
    out.append(f"d{D}{'bf16' if e == 2 else 'f32'} fwd {tf:.0f}us {n*bf/tf/1e3:.0f}GB/s bwd {tb:.0f}us {n*bb/tb/1e3:.0f}GB/s")
print(os.path.basename(os.environ.get("SWR_LIB", "default")), " | ".join(out), flush=True)
