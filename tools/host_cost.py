"""Host (CPU) cost of one entry-point call: enqueue N calls behind a long GPU sleep so
nothing waits on the GPU, and divide the wall time.  Compare with the GPU time per
call: if the host is slower, back-to-back timings include GPU idle gaps.

    python tools/host_cost.py [swr|mix]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2512_13921_b200 as P
from paper_2512_13921_b200 import _lib, ops
from swr_inputs import mix_inputs, swr_inputs

op = sys.argv[1] if len(sys.argv) > 1 else "swr"
B, L, H, D = 8, 4096, 16, 128
if op == "swr":
    g = {k: v.cuda() for k, v in swr_inputs(B, L, H, D, dtype=torch.bfloat16, seed=1).items()}
    f = lambda: P.swr_fwd(g["u"], g["a"])  # noqa: E731
    bw = lambda: P.swr_bwd(g["u"], g["a"], g["G"])  # noqa: E731
else:
    g = {k: v.cuda() for k, v in mix_inputs(B, L, H, D, dtype=torch.bfloat16, seed=1).items()}
    f = lambda: P.phalanx_mix(g["q"], g["k"], g["v"], g["a"])  # noqa: E731
    bw = lambda: P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"])  # noqa: E731
x = f()
du, da, _ = bw() if op == "swr" else (None, None, None)
for _ in range(5):
    f(); bw()
torch.cuda.synchronize()
stream = torch.cuda.current_stream().cuda_stream
shape = ops._shape(g["u"] if op == "swr" else g["q"], g["a"])
N = 100
for name, fn in (("fwd (ops)", f), ("bwd (ops)", bw),
                 ("fwd (raw C ABI)", lambda: _lib.swr_fwd(g["u"].data_ptr(), g["a"].data_ptr(), x.data_ptr(), None,
                                                          None, shape, _lib.SWR_BF16, stream)) if op == "swr" else None,
                 ("event record", lambda: torch.cuda.Event(enable_timing=True).record())):
    if fn is None:
        continue
    torch.cuda._sleep(2_000_000_000)  # ~1 s of GPU work ahead of the calls
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    t = (time.perf_counter() - t0) / N * 1e6
    torch.cuda.synchronize()
    print(f"{op} {name}: {t:.1f} us host time per call", flush=True)
