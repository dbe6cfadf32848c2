"""Back-to-back times of the backward kernels at the paper's head shape (d=16, h=128,
B=8, L=8192, bf16), SWR and mixer: python tools/nar_time.py [B L H D]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2512_13921_b200 as P
from swr_inputs import mix_inputs

B, L, H, D = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (8, 8192, 128, 16)
g = {k: v.cuda() for k, v in mix_inputs(B, L, H, D, dtype=torch.bfloat16, seed=1).items()}
P.set_path(P.SWR_PATH_FFMA)


def b2b(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


e = 2
tok = B * L * H
ts = b2b(lambda: P.swr_bwd(g["v"], g["a"], g["dy"]))
tm = b2b(lambda: P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"]))
bs = tok * ((2 * D + 1) * e + (D + 1) * e)
bm = tok * ((4 * D + 1) * e + (3 * D + 1) * e)
print(f"{os.environ.get('SWR_LIB', 'libswr.so')}: swr_bwd {ts:.1f} us {bs / ts / 1e3:.0f} GB/s | mix_bwd {tm:.1f} us {bm / tm / 1e3:.0f} GB/s")
