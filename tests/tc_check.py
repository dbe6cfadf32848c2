"""Quick TC-path parity probe (test infrastructure: it calls oracle/): each op once on
bf16 D=128 inputs vs the fp64 oracle.  python tests/tc_check.py [B] [L] [ops]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_2512_13921_b200 as P
from swr_inputs import swr_inputs, mix_inputs, to64

def err(x, ref):
    x = x.detach().to("cpu", torch.float64).numpy()
    return float(np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-30))

P.set_path(P.SWR_PATH_TC)
B, L, H, D = int(sys.argv[1]) if len(sys.argv) > 1 else 2, int(sys.argv[2]) if len(sys.argv) > 2 else 100, 16, 128
ops = sys.argv[3].split(",") if len(sys.argv) > 3 else ["fwd", "bwd", "mixf", "mixb"]
inp = swr_inputs(B, L, H, D, dtype=torch.bfloat16, seed=3, carry=True)
g = {k: v.cuda() for k, v in inp.items()}
h = {k: to64(v) for k, v in inp.items()}
if "fwd" in ops:
    x, co = P.swr_fwd(g["u"], g["a"], carry_in=g["carry_in"], return_carry=True); torch.cuda.synchronize()
    rx, rco = oracle.swr_fwd(h["u"], h["a"], carry_in=h["carry_in"], carry_out=True)
    print("fwd path", P.last_path(), "x", err(x, rx), "co", err(co, rco), flush=True)
if "bwd" in ops:
    du, da, mo = P.swr_bwd(g["u"], g["a"], g["G"], carry_in=g["carry_in"], mu_in=g["mu_in"]); torch.cuda.synchronize()
    rdu, rda, rmo = oracle.swr_bwd(h["u"], h["a"], h["G"], carry_in=h["carry_in"], mu_in=h["mu_in"])
    print("bwd path", P.last_path(), "du", err(du, rdu), "da", err(da, rda), "mo", err(mo, rmo), flush=True)
inp = mix_inputs(B, L, H, D, dtype=torch.bfloat16, seed=4, carry=True)
g = {k: v.cuda() for k, v in inp.items()}
h = {k: to64(v) for k, v in inp.items()}
if "mixf" in ops:
    y, co = P.phalanx_mix(g["q"], g["k"], g["v"], g["a"], carry_in=g["carry_in"], return_carry=True); torch.cuda.synchronize()
    ry, rco = oracle.mix_fwd(h["q"], h["k"], h["v"], h["a"], carry_in=h["carry_in"], carry_out=True)
    print("mixf path", P.last_path(), "y", err(y, ry), "co", err(co, rco), flush=True)
if "mixb" in ops:
    r = P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"], carry_in=g["carry_in"], mu_in=g["mu_in"]); torch.cuda.synchronize()
    rr = oracle.mix_bwd(h["q"], h["k"], h["v"], h["a"], h["dy"], carry_in=h["carry_in"], mu_in=h["mu_in"])
    print("mixb path", P.last_path(), [round(err(a_, b_), 6) for a_, b_ in zip(r, rr)], flush=True)
