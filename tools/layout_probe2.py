"""Same SWR work in the [B,L,H,D] layout and in a head-major physical layout
([B,H,L,D] storage viewed as [B,L,H,D]): does DRAM page locality limit the TC kernels?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2512_13921_b200 as P
B, L, H, D = 8, 4096, 16, 128
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.zeros(64 << 20, device="cuda"); sink = torch.empty(1, device="cuda")
def t(fn):
    for _ in range(20): fn()
    ts = []
    for _ in range(15):
        flush.zero_(); sink.copy_(rd.sum())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    return sorted(ts)[len(ts) // 2]
a = torch.sigmoid(torch.randn(B, L, H, device="cuda")).bfloat16()
for name, mk in [("BLHD", lambda: torch.randn(B, L, H, D, device="cuda").bfloat16()),
                 ("BHLD", lambda: torch.randn(B, H, L, D, device="cuda").bfloat16().transpose(1, 2))]:
    u, G = mk(), mk()
    x = torch.empty_like(u)
    tf = t(lambda: P.swr_fwd(u, a))
    tb = t(lambda: P.swr_bwd(u, a, G))
    print(name, "path", P.last_path(), f"fwd {tf:.1f}us bwd {tb:.1f}us", flush=True)
