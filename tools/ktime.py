"""Per-kernel timing (CUDA events, L2 flushed between launches) of each TC op on a
bench config; prints median us and algorithmic GB/s.  SWR_LIB selects a build."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2512_13921_b200 as P
from swr_inputs import swr_inputs, mix_inputs

B, L, H, D = 8, 4096, 16, 128
ops = sys.argv[1].split(",") if len(sys.argv) > 1 else ["fwd", "bwd", "mixf", "mixb"]
P.set_path(P.SWR_PATH_TC)
n = B * L * H
bytes_ = {"fwd": n * (2 * D + 1) * 2, "bwd": n * (3 * D + 2) * 2, "mixf": n * (4 * D + 1) * 2, "mixb": n * (7 * D + 2) * 2}
s = {k: v.cuda() for k, v in swr_inputs(B, L, H, D, dtype=torch.bfloat16, seed=1).items()}
m = {k: v.cuda() for k, v in mix_inputs(B, L, H, D, dtype=torch.bfloat16, seed=2).items()}
fn = {"fwd": lambda: P.swr_fwd(s["u"], s["a"]),
      "bwd": lambda: P.swr_bwd(s["u"], s["a"], s["G"]),
      "mixf": lambda: P.phalanx_mix(m["q"], m["k"], m["v"], m["a"]),
      "mixb": lambda: P.phalanx_mix_bwd(m["q"], m["k"], m["v"], m["a"], m["dy"])}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.zeros(64 << 20, device="cuda")
sink = torch.empty(1, device="cuda")
out = []
for op in ops:
    for _ in range(3): fn[op]()
    ts = []
    for _ in range(25):
        flush.zero_(); sink.copy_(flush_rd.sum())  # clean L2 (bench.py's flush)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn[op](); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort(); med = ts[len(ts) // 2]
    out.append(f"{op} {med:.1f}us {bytes_[op] / med / 1e3:.0f}GB/s")
print(os.path.basename(os.environ.get("SWR_LIB", "default")), " | ".join(out), flush=True)
