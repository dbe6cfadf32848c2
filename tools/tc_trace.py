"""Per-item pipeline timeline of CTA 0 of the TC kernels (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2512_13921_b200 as P
from paper_2512_13921_b200 import _lib
from swr_inputs import swr_inputs, mix_inputs

EV = ["prod_got", "prod_issued", "prep_full", "prep_done", "mma_full", "mma_issued", "ready",
      "epi_ready", "epi_done", "store_commit", "released"]
op = sys.argv[1] if len(sys.argv) > 1 else "fwd"
N = 64
P.set_path(P.SWR_PATH_TC)
if op in ("fwd", "bwd"):
    g = {k: v.cuda() for k, v in swr_inputs(8, 4096, 16, 128, seed=1).items()}
    run = (lambda: P.swr_fwd(g["u"], g["a"])) if op == "fwd" else (lambda: P.swr_bwd(g["u"], g["a"], g["G"]))
else:
    g = {k: v.cuda() for k, v in mix_inputs(8, 4096, 16, 128, seed=1).items()}
    run = (lambda: P.phalanx_mix(g["q"], g["k"], g["v"], g["a"])) if op == "mixf" else (
        lambda: P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"]))
for _ in range(int(os.environ.get("WARM", "5"))):
    run()
buf = torch.zeros(N * 16 + 4 * 160, dtype=torch.int64, device="cuda")
_lib.set_trace(buf.data_ptr(), N)
if os.environ.get("B2B"):  # traced launch right behind back-to-back launches (deferred write-back paid)
    for _ in range(4):
        run()
else:
    flush = torch.empty(64 << 20, device="cuda")
    flush.zero_()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); run(); e1.record()
torch.cuda.synchronize()
_lib.set_trace(None, 0)
print(op, "kernel ms", e0.elapsed_time(e1))
allb = buf.cpu().numpy()
span = allb[N * 16:].reshape(-1, 4)
span = span[span[:, 0] > 0]
order = np.argsort(span[:, 2])
d_sm = (span[order, 1] - span[order, 0]) / 1e3
print("span (us) / items by SM id:", " ".join(f"{int(span[i,2])}:{x:.0f}/{int(span[i,3])}" for i, x in zip(order, d_sm)))
st0 = span[:, 0].min()
dur = (span[:, 1] - span[:, 0]) / 1e3
ends = np.sort((span[:, 1] - span[:, 0].min()) / 1e3)
print("CTA end times (us) percentiles 0/10/50/90/100:", " ".join(f"{np.percentile(ends, q):.1f}" for q in (0, 10, 50, 90, 100)))
print(f"CTAs {len(span)}: start spread {(span[:,0].max()-st0)/1e3:.1f} us, span min/med/max {dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us, last end {(span[:,1].max()-st0)/1e3:.1f} us")
t = allb[:N * 16].reshape(N, 16).astype(np.int64)
valid = t[:, 0] > 0
t0 = t[valid][:, 0].min()
rel = np.where(t > 0, t - t0, -1)
print("item " + " ".join(f"{e[:10]:>10}" for e in EV))
for j in list(range(20, 36)):
    if j < N and valid[j]:
        print(f"{j:4d} " + " ".join(f"{x:10d}" for x in rel[j]))
# steady-state averages of stage-to-stage latencies (items 40..200)
sl = slice(8, 48)
def d(a, b):
    m = (t[sl, a] > 0) & (t[sl, b] > 0)
    return float(np.median(t[sl, b][m] - t[sl, a][m])) if m.any() else float("nan")
print("median latencies (cycles): prod_issued->prep_full", d(1, 2), " prep", d(2, 3), " prep_done->mma_full", d(3, 4),
      " mma_issued->ready", d(5, 6), " ready->epi_ready", d(6, 7), " epi", d(7, 8), " epi_done->commit", d(8, 9),
      " prod_got->released(own)", d(0, 10))
per = np.diff(t[sl, 1])
print("producer issue period cycles (median)", float(np.median(per)), " epi_ready period", float(np.median(np.diff(t[sl, 7][t[sl,7]>0]))))
# full timeline of CTA 0: item, producer got-stage time (us), prep_full latency, epi_done (us)
if os.environ.get("TIMELINE"):
    clk = 1.965e3  # cycles per us at the max SM clock
    for j in range(N):
        if not valid[j]: break
        print(f"tl {j:3d} got {rel[j,0]/clk:6.2f} issued {rel[j,1]/clk:6.2f} landed {rel[j,2]/clk:6.2f} prepped {rel[j,3]/clk:6.2f} mma {rel[j,5]/clk:6.2f} epi_in {rel[j,7]/clk:6.2f} epi_out {rel[j,8]/clk:6.2f} store {rel[j,9]/clk:6.2f} retired {rel[j,10]/clk:6.2f} dec_issue {rel[j,11]/clk:6.2f}")
