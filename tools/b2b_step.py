"""Back-to-back timing (no L2 flush; inputs > L2) of the fwd, the bwd and the fwd+bwd
step of one op on a bench config, so every deferred write-back is charged to some
launch.  SWR_LIB selects a build (A/B with tools/ab_b2b.sh).

    python tools/b2b_step.py [swr|mix] [B L H D]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2512_13921_b200 as P
from swr_inputs import mix_inputs, swr_inputs

op = sys.argv[1] if len(sys.argv) > 1 else "swr"
B, L, H, D = (int(x) for x in sys.argv[2:6]) if len(sys.argv) > 5 else (8, 4096, 16, 128)
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def b2b(fn, n=40, warm=8):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = E(), E()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


n = B * L * H
if op == "swr":
    g = {k: v.cuda() for k, v in swr_inputs(B, L, H, D, dtype=torch.bfloat16, seed=1).items()}
    f = lambda: P.swr_fwd(g["u"], g["a"])  # noqa: E731
    bw = lambda: P.swr_bwd(g["u"], g["a"], g["G"])  # noqa: E731
    by_f, by_b = n * (2 * D + 1) * 2, n * (3 * D + 2) * 2
else:
    g = {k: v.cuda() for k, v in mix_inputs(B, L, H, D, dtype=torch.bfloat16, seed=1).items()}
    f = lambda: P.phalanx_mix(g["q"], g["k"], g["v"], g["a"])  # noqa: E731
    bw = lambda: P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"])  # noqa: E731
    by_f, by_b = n * (4 * D + 1) * 2, n * (7 * D + 2) * 2
tf, tb, ts = b2b(f), b2b(bw), b2b(lambda: (f(), bw()))
print(f"{os.path.basename(os.environ.get('SWR_LIB', 'default')):24s} {op} fwd {tf:6.1f} us {by_f / tf / 1e3:5.0f} GB/s"
      f" | bwd {tb:6.1f} us {by_b / tb / 1e3:5.0f} GB/s | step {ts:6.1f} us {(by_f + by_b) / ts / 1e3:5.0f} GB/s"
      f" {B * L / ts:6.1f} Mtok/s", flush=True)
