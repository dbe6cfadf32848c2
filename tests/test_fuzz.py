"""Seeded random configurations of every north-star entry point (and the layer mixer)
against the fp64 oracle: random B, L (ragged), H, d, dtype, kernel family, carries,
decay family and memory layout (contiguous, head-major storage, a slice of a wider
tensor).  Complements the structured sweeps of test_parity.py / test_tc_parity.py with
combinations nobody picked by hand.  Tolerance as test_parity.py (normwise)."""
import random

import numpy as np
import pytest
import torch

import oracle
from swr_inputs import DECAY_KINDS, layer_inputs, mix_inputs, swr_inputs, to64

pytestmark = pytest.mark.gpu
TOL = {torch.float32: 1e-5, torch.bfloat16: 2e-2}
N_CASES = 160


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from conftest import build_lib
    build_lib()
    import paper_2512_13921_b200 as P
    return P


def normwise(x, ref):
    x = x.detach().to("cpu", torch.float64).numpy()
    den = np.max(np.abs(ref)) if ref.size else 0.0
    num = np.max(np.abs(x - ref)) if ref.size else 0.0
    return num / den if den > 0 else num


def relayout(t, how, rng):
    """The same values in another memory layout the ABI accepts (D contiguous)."""
    if how == "contiguous" or t.dim() != 4:
        return t.cuda()
    if how == "head_major":  # storage [B, H, L, D], viewed as [B, L, H, D]
        return t.permute(0, 2, 1, 3).contiguous().cuda().permute(0, 2, 1, 3)
    # a slice of a tensor with extra heads on both sides
    B, L, H, D = t.shape
    big = torch.zeros(B, L, H + 3, D, dtype=t.dtype)
    big[:, :, 1:H + 1] = t
    return big.cuda()[:, :, 1:H + 1]


def case(i):
    rng = random.Random(1000 + i)
    op = rng.choice(["swr", "mix", "layer"])
    dtype = rng.choice([torch.float32, torch.bfloat16])
    D = rng.choice([16, 32, 64, 128])
    H = rng.choice([1, 2, 3, 4, 8, 16]) if op != "layer" else rng.choice([2, 4, 8, 16])
    B = rng.choice([1, 2, 3])
    L = rng.choice([1, 15, 16, 17, 31, 64, 100, 129, 256, 333])
    path = rng.choice(["auto", "ffma"])
    carry = rng.random() < 0.5
    decay = rng.choice(DECAY_KINDS)
    how = rng.choice(["contiguous", "head_major", "slice"])
    return dict(op=op, dtype=dtype, D=D, H=H, B=B, L=L, path=path, carry=carry, decay=decay, how=how,
                seed=2000 + i)


@pytest.mark.parametrize("i", range(N_CASES))
def test_fuzz(P, i):
    c = case(i)
    rng = random.Random(c["seed"])
    prev = P.set_path(P.SWR_PATH_AUTO if c["path"] == "auto" else P.SWR_PATH_FFMA)
    tol = TOL[c["dtype"]]
    try:
        if c["op"] == "swr":
            inp = swr_inputs(c["B"], c["L"], c["H"], c["D"], dtype=c["dtype"], seed=c["seed"], decay=c["decay"],
                             carry=c["carry"])
            g = {k: relayout(v, c["how"], rng) for k, v in inp.items()}
            x, co = P.swr_fwd(g["u"], g["a"], carry_in=g.get("carry_in"), return_carry=True)
            du, da, mo = P.swr_bwd(g["u"], g["a"], g["G"], carry_in=g.get("carry_in"), mu_in=g.get("mu_in"))
            torch.cuda.synchronize()
            h = {k: to64(v) for k, v in inp.items()}
            rx, rco = oracle.swr_fwd(h["u"], h["a"], carry_in=h.get("carry_in"), carry_out=True)
            rdu, rda, rmo = oracle.swr_bwd(h["u"], h["a"], h["G"], carry_in=h.get("carry_in"), mu_in=h.get("mu_in"))
            outs = {"x": (x, rx), "carry_out": (co, rco), "du": (du, rdu), "da": (da, rda), "mu_out": (mo, rmo)}
        elif c["op"] == "mix":
            inp = mix_inputs(c["B"], c["L"], c["H"], c["D"], dtype=c["dtype"], seed=c["seed"], decay=c["decay"],
                             carry=c["carry"])
            g = {k: relayout(v, c["how"], rng) for k, v in inp.items()}
            y, co = P.phalanx_mix(g["q"], g["k"], g["v"], g["a"], carry_in=g.get("carry_in"), return_carry=True)
            dq, dk, dv, da, mo = P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"], carry_in=g.get("carry_in"),
                                                   mu_in=g.get("mu_in"))
            torch.cuda.synchronize()
            h = {k: to64(v) for k, v in inp.items()}
            ry, rco = oracle.mix_fwd(h["q"], h["k"], h["v"], h["a"], carry_in=h.get("carry_in"), carry_out=True)
            rdq, rdk, rdv, rda, rmo = oracle.mix_bwd(h["q"], h["k"], h["v"], h["a"], h["dy"],
                                                     carry_in=h.get("carry_in"), mu_in=h.get("mu_in"))
            outs = {"y": (y, ry), "carry_out": (co, rco), "dq": (dq, rdq), "dk": (dk, rdk), "dv": (dv, rdv),
                    "da": (da, rda), "mu_out": (mo, rmo)}
        else:
            H = c["H"]
            Gq, Gk = rng.choice([g for g in (1, 2, 4, 8, 16) if H % g == 0]), rng.choice(
                [g for g in (1, 2, 4, 8, 16) if H % g == 0])
            inp = layer_inputs(c["B"], c["L"], H, c["D"], Gq, Gk, dtype=c["dtype"], seed=c["seed"], carry=c["carry"])
            g = {k: relayout(v, c["how"], rng) for k, v in inp.items()}
            hq, hk = H // Gq, H // Gk
            fits = all(x <= 256 // (c["D"] // 4) for x in (hq, hk)) or (
                c["dtype"] == torch.bfloat16 and c["D"] == 128 and H % 8 == 0 and c["path"] == "auto")
            y, co = P.phalanx_layer_mix(g["q"], g["zk"], g["v"], g["za"], carry_in=g.get("carry_in"), return_carry=True)
            if not fits:
                with pytest.raises(P.SwrError, match="UNSUPPORTED"):
                    P.phalanx_layer_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"])
                return
            dq, dzk, dv, dza, mo = P.phalanx_layer_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"],
                                                           carry_in=g.get("carry_in"), mu_in=g.get("mu_in"))
            torch.cuda.synchronize()
            h = {k: to64(v) for k, v in inp.items()}
            ry, rco = oracle.layer_mix_fwd(h["q"], h["zk"], h["v"], h["za"], carry_in=h.get("carry_in"), carry_out=True)
            rdq, rdzk, rdv, rdza, rmo = oracle.layer_mix_bwd(h["q"], h["zk"], h["v"], h["za"], h["dy"],
                                                             carry_in=h.get("carry_in"), mu_in=h.get("mu_in"))
            outs = {"y": (y, ry), "carry_out": (co, rco), "dq": (dq, rdq), "dzk": (dzk, rdzk), "dv": (dv, rdv),
                    "dza": (dza, rdza), "mu_out": (mo, rmo)}
    finally:
        P.set_path(prev)
    errs = {k: normwise(a, r) for k, (a, r) in outs.items()}
    bad = {k: e for k, e in errs.items() if e > tol}
    assert not bad, f"case {c}: {bad}"
