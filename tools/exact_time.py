"""What B2P's truncation saves: the exact full-range recurrence (swr_exact_fwd: one
pass with a decoupled look-back; swr_exact_bwd: five launches) against the truncated
B2P step (swr_fwd / swr_bwd), back to back (CUDA events, no flush; inputs > L2).
SWR_LIB selects a build (the round-1 three-launch forward: -DSWR_EXACT_3STAGE)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2512_13921_b200 as P
from swr_inputs import swr_inputs

E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def t(fn, n=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = E(), E()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


tag = os.path.basename(os.environ.get("SWR_LIB", "default"))
for (B, L, H, D, dt) in [(8, 4096, 16, 128, torch.bfloat16), (2, 32768, 16, 128, torch.bfloat16),
                         (8, 8192, 128, 16, torch.bfloat16), (8, 4096, 16, 128, torch.float32)]:
    g = {k: v.cuda() for k, v in swr_inputs(B, L, H, D, dtype=dt, seed=1).items()}
    te = t(lambda: P.swr_exact_fwd(g["u"], g["a"]))
    epath = {1: "ffma", 2: "tc"}[P.last_path()]
    tt = t(lambda: P.swr_fwd(g["u"], g["a"]))
    tbe = t(lambda: P.swr_exact_bwd(g["u"], g["a"], g["G"]))
    tbt = t(lambda: P.swr_bwd(g["u"], g["a"], g["G"]))
    path = {1: "ffma", 2: "tc"}[P.last_path()]
    e = g["u"].element_size()
    n = B * L * H
    print(f"{tag} B={B} L={L} H={H} d={D} {str(dt)[6:]}: exact fwd [{epath}] {te:.0f} us ({n * (2 * D + 1) * e / te / 1e3:.0f} GB/s"
          f" algorithmic), B2P swr_fwd [{path}] {tt:.0f} us -> {te / tt:.2f}x; exact bwd {tbe:.0f} us vs B2P {tbt:.0f} us"
          f" ({tbe / tbt:.2f}x)", flush=True)
