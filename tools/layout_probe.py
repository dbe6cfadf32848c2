"""Does DRAM locality matter?  Time the TC kernels on the same total work with
different head counts (B*H fixed): H=1 makes every line contiguous in HBM."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2512_13921_b200 as P
from swr_inputs import swr_inputs
P.set_path(P.SWR_PATH_TC)
L, D = 4096, 128
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.zeros(64 << 20, device="cuda"); sink = torch.empty(1, device="cuda")
for H in (1, 2, 4, 8, 16, 32):
    B = 128 // H
    s = {k: v.cuda() for k, v in swr_inputs(B, L, H, D, dtype=torch.bfloat16, seed=1).items()}
    n = B * L * H
    res = []
    for name, fn, by in (("fwd", lambda: P.swr_fwd(s["u"], s["a"]), n * (2 * D + 1) * 2),
                         ("bwd", lambda: P.swr_bwd(s["u"], s["a"], s["G"]), n * (3 * D + 2) * 2)):
        for _ in range(3): fn()
        ts = []
        for _ in range(15):
            flush.zero_(); sink.copy_(rd.sum())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort(); med = ts[len(ts) // 2]
        res.append(f"{name} {med:.1f}us {by / med / 1e3:.0f}GB/s")
    print(f"B={B} H={H}: " + " | ".join(res), flush=True)
