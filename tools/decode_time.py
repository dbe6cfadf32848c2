"""Per-token time of the recurrence-mode decode step (swr_decode_step), eager and
captured in one CUDA graph of S steps, at the layer shape (B=8, H=16, d=128) and the
paper's head shape (B=8, H=128, d=16)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2512_13921_b200 as P

S = 256
for (B, H, D, dt) in [(8, 16, 128, torch.bfloat16), (8, 128, 16, torch.bfloat16), (256, 16, 128, torch.bfloat16)]:
    u = torch.randn(B, S, H, D, device="cuda").to(dt)
    a = torch.rand(B, S, H, device="cuda").to(dt)
    st = P.DecodeState(B, H, D, u.device)
    us = [u[:, n].contiguous() for n in range(S)]
    as_ = [a[:, n] for n in range(S)]
    def run():
        st.pos = 0
        for n in range(S):
            P.swr_decode_step(us[n], as_[n], st)
    for _ in range(2): run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) * 1e3 / S
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): run()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g): run()
    g.replay(); torch.cuda.synchronize()
    e0.record()
    for _ in range(5): g.replay()
    e1.record(); torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) * 1e3 / (5 * S)
    byts = B * H * (D * 2 + 2 + 3 * 4 * D + 4 + D * 2)  # u, a, w+v read, w write (+v at block start), x
    print(f"B={B} H={H} d={D}: eager {eager:.2f} us/token, graph {graph:.2f} us/token "
          f"({B * H / graph / 1e3:.1f} G token-heads/s, ~{byts / graph / 1e3:.0f} GB/s)", flush=True)
