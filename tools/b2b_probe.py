"""Back-to-back timing (no L2 flush between steps; inputs 4x the L2) of the SWR step
and of reference copies, so every deferred write-back is charged to some step.

    python tools/b2b_probe.py [op=swr|mix] [config=layer4k]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2512_13921_b200 as P
from swr_inputs import mix_inputs, swr_inputs

op = sys.argv[1] if len(sys.argv) > 1 else "swr"
B, L, H, D = 8, 4096, 16, 128
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def b2b(fn, n=30, warm=5):
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


# reference copies: torch copy_ of one d-tensor (128 MiB) and of 1 GiB elements (MEASURED_PEAKS)
for nbytes in (128 << 20, 256 << 20, 2 << 30):
    a = torch.empty(nbytes // 2, dtype=torch.bfloat16, device="cuda").normal_()
    b = torch.empty_like(a)
    t = b2b(lambda: b.copy_(a))
    print(f"copy_ {nbytes >> 20} MiB: {t:.1f} us  {2 * nbytes / t / 1e3:.0f} GB/s (read+write)", flush=True)
    del a, b
# read-only sum and write-only fill
a = torch.empty(128 << 20, dtype=torch.bfloat16, device="cuda").normal_()
t = b2b(lambda: a.sum())
print(f"read 256 MiB (sum): {t:.1f} us {256 * 2**20 / t / 1e3:.0f} GB/s", flush=True)
t = b2b(lambda: a.fill_(1.0))
print(f"write 256 MiB (fill): {t:.1f} us {256 * 2**20 / t / 1e3:.0f} GB/s", flush=True)
del a

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
tf = b2b(f)
tb = b2b(bw)
ts = b2b(lambda: (f(), bw()))
print(f"{op} fwd b2b {tf:.1f} us {by_f / tf / 1e3:.0f} GB/s | bwd b2b {tb:.1f} us {by_b / tb / 1e3:.0f} GB/s"
      f" | step b2b {ts:.1f} us {(by_f + by_b) / ts / 1e3:.0f} GB/s {B * L / ts:.1f} Mtok/s", flush=True)
