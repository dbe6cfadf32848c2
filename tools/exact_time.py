"""What B2P's truncation saves (and the uniform window k = 16 beside it): the exact full-range recurrence (swr_exact_fwd,
Alg. 2's three stages) against the truncated B2P forward (swr_fwd) at the layer
shape, each after an L2 flush (CUDA events, median of 10)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
for (B, L, H, D, dt) in [(8, 4096, 16, 128, torch.bfloat16), (2, 32768, 16, 128, torch.bfloat16),
                         (8, 8192, 128, 16, torch.bfloat16), (8, 4096, 16, 128, torch.float32)]:
    g = {k: v.cuda() for k, v in swr_inputs(B, L, H, D, dtype=dt, seed=1).items()}
    te = t(lambda: P.swr_exact_fwd(g["u"], g["a"]))
    tt = t(lambda: P.swr_fwd(g["u"], g["a"]))
    tbe = t(lambda: P.swr_exact_bwd(g["u"], g["a"], g["G"]))
    tbt = t(lambda: P.swr_bwd(g["u"], g["a"], g["G"]))
    path = {1: "ffma", 2: "tc"}[P.last_path()]
    tu = t(lambda: P.swr_uniform_fwd(g["u"], g["a"], 16))
    e = g["u"].element_size()
    n = B * L * H
    print(f"B={B} L={L} H={H} d={D} {str(dt)[6:]}: exact {te:.0f} us ({n * (2 * D + 1) * e / te / 1e3:.0f} GB/s "
          f"algorithmic), B2P swr_fwd [{path}] {tt:.0f} us -> exact/B2P {te / tt:.2f}x; backward exact {tbe:.0f} us "
          f"vs B2P {tbt:.0f} us ({tbe / tbt:.2f}x); uniform k=16 fwd {tu:.0f} us", flush=True)
