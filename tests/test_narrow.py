"""GPU parity of the staged narrow-head backward (csrc/swr_narrow.cu: bf16, D = 16 / 32,
TMA-addressable operands -- the paper's head shape d = 16, h = 128)
against the fp64 oracle.  These shapes take that kernel on the CUDA-core family
(SWR_PATH_FFMA, and AUTO since the tensor cores serve D = 128 only): H a multiple of
8 (16-byte decay rows), contiguous heads.  Covered: one block, ragged tails (15, 17,
33), chunk boundaries of the 32-block walk with their halo blocks (512, 513, 1100,
2049), head groups that overhang H (H = 24 with 16-head CTAs), carries in and out,
every decay family, batch > 1; the layer mixer backward with groups of 8 / 16 heads
(mixed q / k group sizes, D = 32, H = 48 / 64 / 128, L = 1 .. 700, each logit flag).
Tolerance as tests/test_parity.py (normwise 2e-2)."""
import numpy as np
import pytest
import torch

import oracle
from swr_inputs import DECAY_KINDS, mix_inputs, swr_inputs, to64

pytestmark = pytest.mark.gpu

TOL = 2e-2


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from conftest import build_lib
    build_lib()
    import paper_2512_13921_b200 as P
    prev = P.set_path(P.SWR_PATH_FFMA)
    yield P
    P.set_path(prev)


def normwise(x, ref):
    x = x.detach().to("cpu", torch.float64).numpy()
    den = np.max(np.abs(ref)) if ref.size else 0.0
    num = np.max(np.abs(x - ref)) if ref.size else 0.0
    return num / den if den > 0 else num


def check(outs, refs):
    errs = {k: normwise(outs[k], refs[k]) for k in outs}
    bad = {k: e for k, e in errs.items() if e > TOL}
    assert not bad, f"normwise errors above {TOL}: {bad} (all: {errs})"


SHAPES = [(1, 1, 8), (2, 15, 8), (1, 17, 16), (3, 33, 24), (1, 512, 8), (2, 513, 16), (1, 1100, 24),
          (1, 2049, 8), (2, 300, 128)]


@pytest.mark.parametrize("D", [16, 32])
@pytest.mark.parametrize("B,L,H", SHAPES)
@pytest.mark.parametrize("carry", [False, True])
def test_swr_bwd_narrow(P, B, L, H, D, carry):
    inp = swr_inputs(B, L, H, D, dtype=torch.bfloat16, seed=7 * L + H + D, carry=carry)
    g = {k: v.cuda() for k, v in inp.items()}
    du, da, mo = P.swr_bwd(g["u"], g["a"], g["G"], carry_in=g.get("carry_in"), mu_in=g.get("mu_in"))
    torch.cuda.synchronize()
    assert P.last_path() == 1
    h = {k: to64(v) for k, v in inp.items()}
    rdu, rda, rmo = oracle.swr_bwd(h["u"], h["a"], h["G"], carry_in=h.get("carry_in"), mu_in=h.get("mu_in"))
    check({"du": du, "da": da, "mu_out": mo}, {"du": rdu, "da": rda, "mu_out": rmo})


@pytest.mark.parametrize("D", [16, 32])
@pytest.mark.parametrize("B,L,H", SHAPES)
@pytest.mark.parametrize("carry", [False, True])
def test_mix_bwd_narrow(P, B, L, H, D, carry):
    inp = mix_inputs(B, L, H, D, dtype=torch.bfloat16, seed=5 * L + H + D, carry=carry)
    g = {k: v.cuda() for k, v in inp.items()}
    dq, dk, dv, da, mo = P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"], carry_in=g.get("carry_in"),
                                           mu_in=g.get("mu_in"))
    torch.cuda.synchronize()
    assert P.last_path() == 1
    h = {k: to64(v) for k, v in inp.items()}
    r = oracle.mix_bwd(h["q"], h["k"], h["v"], h["a"], h["dy"], carry_in=h.get("carry_in"), mu_in=h.get("mu_in"))
    check({"dq": dq, "dk": dk, "dv": dv, "da": da, "mu_out": mo},
          dict(zip(["dq", "dk", "dv", "da", "mu_out"], r)))


@pytest.mark.parametrize("decay", DECAY_KINDS)
@pytest.mark.parametrize("op", ["swr", "mix"])
def test_narrow_decays(P, decay, op):
    B, L, H, D = 2, 700, 16, 16
    if op == "swr":
        inp = swr_inputs(B, L, H, D, dtype=torch.bfloat16, seed=11, decay=decay, carry=True)
        g = {k: v.cuda() for k, v in inp.items()}
        out = P.swr_bwd(g["u"], g["a"], g["G"], carry_in=g["carry_in"], mu_in=g["mu_in"])
        h = {k: to64(v) for k, v in inp.items()}
        ref = oracle.swr_bwd(h["u"], h["a"], h["G"], carry_in=h["carry_in"], mu_in=h["mu_in"])
        names = ["du", "da", "mu_out"]
    else:
        inp = mix_inputs(B, L, H, D, dtype=torch.bfloat16, seed=13, decay=decay, carry=True)
        g = {k: v.cuda() for k, v in inp.items()}
        out = P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"], carry_in=g["carry_in"], mu_in=g["mu_in"])
        h = {k: to64(v) for k, v in inp.items()}
        ref = oracle.mix_bwd(h["q"], h["k"], h["v"], h["a"], h["dy"], carry_in=h["carry_in"], mu_in=h["mu_in"])
        names = ["dq", "dk", "dv", "da", "mu_out"]
    torch.cuda.synchronize()
    check(dict(zip(names, out)), dict(zip(names, ref)))


def test_narrow_deterministic(P):
    """Fixed-order da reduction: repeated launches give the same bits."""
    inp = mix_inputs(2, 3000, 32, 16, dtype=torch.bfloat16, seed=3)
    g = {k: v.cuda() for k, v in inp.items()}
    r1 = P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"])
    r2 = P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"])
    torch.cuda.synchronize()
    for x1, x2 in zip(r1, r2):
        assert torch.equal(x1, x2)


def test_narrow_paper_shape_sampled(P):
    """The bench's paper_d16 workload (B=8, L=8192, H=128, d=16) in the bench's launch
    configuration: four sampled (b, h) lines of the SWR and mixer backward against the
    oracle run on those lines alone (lines are independent)."""
    B, L, H, D = 8, 8192, 128, 16
    inp = mix_inputs(B, L, H, D, dtype=torch.bfloat16, seed=1)
    g = {k: v.cuda() for k, v in inp.items()}
    du, da, _ = P.swr_bwd(g["v"], g["a"], g["dy"])
    dq, dk, dv, dam, _ = P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"])
    torch.cuda.synchronize()
    for b, hh in [(0, 0), (3, 57), (7, 127), (5, 64)]:
        s = lambda x: to64(x[b:b + 1, :, hh:hh + 1])  # noqa: E731
        rdu, rda, _ = oracle.swr_bwd(s(inp["v"]), s(inp["a"]), s(inp["dy"]))
        check({"du": du[b:b + 1, :, hh:hh + 1], "da": da[b:b + 1, :, hh:hh + 1]}, {"du": rdu, "da": rda})
        r = oracle.mix_bwd(s(inp["q"]), s(inp["k"]), s(inp["v"]), s(inp["a"]), s(inp["dy"]))
        check({"dq": dq[b:b + 1, :, hh:hh + 1], "dk": dk[b:b + 1, :, hh:hh + 1], "dv": dv[b:b + 1, :, hh:hh + 1],
               "da": dam[b:b + 1, :, hh:hh + 1]}, dict(zip(["dq", "dk", "dv", "da"], r[:4])))


# ---------------------------------------------------------------------------
# the layer mixer backward on the staged kernel: q / zk shared by groups of >= 8 heads
# inside the CTA's 16 heads (the paper's d = 16 models: 8 groups of 16 heads)
# ---------------------------------------------------------------------------
def _layer_run(P, inp, logit_a=True, logit_k=True):
    from test_layer import run
    return run(P, inp, logit_a=logit_a, logit_k=logit_k)


@pytest.mark.parametrize("B,L,H,D,Gq,Gk", [(1, 64, 128, 16, 8, 8), (2, 100, 128, 16, 16, 8), (1, 513, 32, 16, 2, 4),
                                           (2, 33, 16, 16, 1, 2), (1, 1, 16, 16, 1, 1), (1, 700, 64, 32, 4, 8),
                                           (3, 17, 48, 16, 3, 6)])
@pytest.mark.parametrize("carry", [False, True])
def test_layer_bwd_narrow(P, B, L, H, D, Gq, Gk, carry):
    from swr_inputs import layer_inputs
    from test_layer import check as lcheck
    inp = layer_inputs(B, L, H, D, Gq, Gk, dtype=torch.bfloat16, seed=L + H + Gq + D, carry=carry)
    outs, refs = _layer_run(P, inp)
    assert P.last_path() == 1
    lcheck(outs, refs, TOL)


@pytest.mark.parametrize("logit_a,logit_k", [(False, True), (True, False), (False, False)])
def test_layer_bwd_narrow_flags(P, logit_a, logit_k):
    from swr_inputs import layer_inputs
    from test_layer import check as lcheck
    inp = layer_inputs(2, 300, 128, 16, 8, 8, dtype=torch.bfloat16, seed=9, carry=True)
    if not logit_a:
        inp["za"] = torch.sigmoid(inp["za"].float()).to(torch.bfloat16)
    if not logit_k:
        inp["zk"] = torch.sigmoid(inp["zk"].float()).to(torch.bfloat16)
    outs, refs = _layer_run(P, inp, logit_a=logit_a, logit_k=logit_k)
    lcheck(outs, refs, TOL)


def test_layer_bwd_narrow_deterministic(P):
    from swr_inputs import layer_inputs
    inp = layer_inputs(2, 1000, 128, 16, 8, 8, dtype=torch.bfloat16, seed=4)
    g = {k: v.cuda() for k, v in inp.items()}
    r1 = P.phalanx_layer_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"])
    r2 = P.phalanx_layer_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"])
    torch.cuda.synchronize()
    for x1, x2 in zip(r1, r2):
        assert torch.equal(x1, x2)
