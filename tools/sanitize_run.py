"""One small call of every entry point on both kernel families, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2512_13921_b200 as P
from swr_inputs import layer_inputs, mix_inputs, swr_inputs

torch.cuda.set_device(0)


def run(path, dtype, D, B=1, L=100, H=16):
    P.set_path(path)
    s = {k: v.cuda() for k, v in swr_inputs(B, L, H, D, dtype=dtype, seed=1, carry=True).items()}
    x, co = P.swr_fwd(s["u"], s["a"], carry_in=s["carry_in"], return_carry=True)
    P.swr_bwd(s["u"], s["a"], s["G"], carry_in=s["carry_in"], mu_in=s["mu_in"])
    m = {k: v.cuda() for k, v in mix_inputs(B, L, H, D, dtype=dtype, seed=2, carry=True).items()}
    P.phalanx_mix(m["q"], m["k"], m["v"], m["a"], carry_in=m["carry_in"], return_carry=True)
    P.phalanx_mix_bwd(m["q"], m["k"], m["v"], m["a"], m["dy"], carry_in=m["carry_in"], mu_in=m["mu_in"])
    gq = H // 2  # shared groups: CUDA-core group sums, or TC with the per-head scratch
    y = {k: v.cuda() for k, v in layer_inputs(B, L, H, D, H // 2, H, dtype=dtype, seed=3).items()}
    P.phalanx_layer_mix(y["q"], y["zk"], y["v"], y["za"])
    yb = {k: v.cuda() for k, v in layer_inputs(B, L, H, D, gq, H, dtype=dtype, seed=4).items()}
    P.phalanx_layer_mix_bwd(yb["q"], yb["zk"], yb["v"], yb["za"], yb["dy"])
    torch.cuda.synchronize()
    print("ok", path, dtype, D, "last path", P.last_path(), flush=True)


which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "tc"):
    run(P.SWR_PATH_TC, torch.bfloat16, 128)
    run(P.SWR_PATH_TC, torch.bfloat16, 128, B=2, L=33, H=8)
if which in ("all", "ffma"):
    run(P.SWR_PATH_FFMA, torch.bfloat16, 16, H=8)
    run(P.SWR_PATH_FFMA, torch.float32, 128, H=4)
if which in ("all", "ext"):  # the CUDA-core extensions
    P.set_path(P.SWR_PATH_AUTO)
    s = {k: v.cuda() for k, v in swr_inputs(1, 100, 4, 32, dtype=torch.float32, seed=5).items()}
    P.swr_exact_fwd(s["u"], s["a"])
    P.swr_exact_bwd(s["u"], s["a"], s["G"])
    sl = {k: v.cuda() for k, v in swr_inputs(1, 16 * 1030, 2, 16, dtype=torch.float32, seed=6, carry=True).items()}
    P.swr_exact_fwd(sl["u"], sl["a"], carry_in=sl["carry_in"])  # look-back over many chunks
    P.swr_exact_bwd(sl["u"], sl["a"], sl["G"], carry_in=sl["carry_in"], mu_in=sl["mu_in"])  # look-back scans
    P.swr_uniform_fwd(s["u"], s["a"], 8)
    st = P.DecodeState(1, 4, 32, "cuda")
    for n in range(20):
        P.swr_decode_step(s["u"][:, n], s["a"][:, n], st)
    torch.cuda.synchronize()
    print("ok extensions", flush=True)
