"""GPU parity of the Phalanx layer mixer (include/swr.h
phalanx_layer_mix / phalanx_layer_mix_bwd) against the fp64 oracle
(oracle.layer_mix_fwd / layer_mix_bwd): sigma on the decay and key logits
 and q / k shared by groups of heads.
Tolerance as tests/test_parity.py (normwise; 1e-5 fp32, 2e-2 bf16)."""
import numpy as np
import pytest
import torch

import oracle
from swr_inputs import layer_inputs, to64

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-5, torch.bfloat16: 2e-2}


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


def check(outs, refs, tol):
    errs = {k: normwise(outs[k], refs[k]) for k in outs}
    bad = {k: e for k, e in errs.items() if e > tol}
    assert not bad, f"normwise errors above {tol}: {bad} (all: {errs})"
    return errs


def logit(a):
    """za with sigma(za) = a (to feed the logit oracle a decay / gate given directly)."""
    return np.log(a) - np.log1p(-a)


def run(P, inp, logit_a=True, logit_k=True, carry=False):
    g = {k: v.cuda() for k, v in inp.items()}
    ci, mi = g.get("carry_in"), g.get("mu_in")
    y, co = P.phalanx_layer_mix(g["q"], g["zk"], g["v"], g["za"], carry_in=ci, return_carry=True,
                                logit_a=logit_a, logit_k=logit_k)
    dq, dzk, dv, dza, mo = P.phalanx_layer_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"], carry_in=ci,
                                                   mu_in=mi, logit_a=logit_a, logit_k=logit_k)
    torch.cuda.synchronize()
    h = {k: to64(v) for k, v in inp.items()}
    za = h["za"] if logit_a else logit(h["za"])
    zk = h["zk"] if logit_k else logit(h["zk"])
    ry, rco = oracle.layer_mix_fwd(h["q"], zk, h["v"], za, carry_in=h.get("carry_in"), carry_out=True)
    rdq, rdzk, rdv, rdza, rmo = oracle.layer_mix_bwd(h["q"], zk, h["v"], za, h["dy"],
                                                     carry_in=h.get("carry_in"), mu_in=h.get("mu_in"))
    if not logit_a:  # gradients w.r.t. a itself: dza / sigma'(za)
        s = oracle.sigmoid(za)
        rdza = rdza / (s * (1.0 - s))
    if not logit_k:
        s = oracle.sigmoid(zk)
        rdzk = rdzk / (s * (1.0 - s))
    return ({"y": y, "carry_out": co, "dq": dq, "dzk": dzk, "dv": dv, "dza": dza, "mu_out": mo},
            {"y": ry, "carry_out": rco, "dq": rdq, "dzk": rdzk, "dv": rdv, "dza": rdza, "mu_out": rmo})


# (B, L, H, D, Gq, Gk): no sharing, 2, 4 and 8 heads per group, the paper's 8 groups
# at d = 16 (16 heads per group) and a single group
CASES = [
    (2, 100, 4, 128, 4, 4), (2, 100, 8, 128, 4, 4), (1, 65, 16, 128, 8, 8), (1, 48, 16, 128, 2, 8),
    (2, 77, 16, 64, 4, 2), (1, 200, 8, 32, 1, 2), (1, 64, 128, 16, 8, 8), (2, 33, 32, 16, 4, 32),
    (1, 16, 6, 128, 3, 6), (1, 1, 4, 16, 2, 1), (1, 32, 16, 128, 1, 16),
]


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("B,L,H,D,Gq,Gk", CASES)
def test_layer_mix_parity(P, dtype, B, L, H, D, Gq, Gk):
    inp = layer_inputs(B, L, H, D, Gq, Gk, dtype=dtype, seed=B * 7 + L + H + D + Gq, carry=True)
    hq, hk = H // Gq, H // Gk
    # CUDA-core group sums within one CTA, or the tensor cores with the per-head scratch
    fits = all(x & (x - 1) == 0 and x <= 256 // (D // 4) for x in (hq, hk)) or (
        dtype == torch.bfloat16 and D == 128 and H % 8 == 0)
    if not fits:
        with pytest.raises(P.SwrError, match="UNSUPPORTED"):
            run(P, inp)
        return
    outs, refs = run(P, inp)
    check(outs, refs, TOL[dtype])


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("logit_a,logit_k", [(True, False), (False, True), (False, False)])
def test_layer_mix_logit_flags(P, dtype, logit_a, logit_k):
    """logit_a / logit_k off: za / zk are a / k themselves (then the reference's
    logit-gradients are divided back by sigma')."""
    inp = layer_inputs(2, 80, 8, 32, 4, 2, dtype=dtype, seed=11)
    if not logit_a:
        inp["za"] = torch.sigmoid(inp["za"].float()).to(dtype)
    if not logit_k:
        inp["zk"] = torch.sigmoid(inp["zk"].float()).to(dtype)
    outs, refs = run(P, inp, logit_a, logit_k)
    check(outs, refs, TOL[dtype])


def test_layer_mix_reduces_to_mixer(P):
    """G = H and logits off: bitwise the plain mixer's kernels (same FFMA arithmetic)."""
    inp = layer_inputs(2, 96, 4, 64, dtype=torch.float32, seed=5)
    g = {k: v.cuda() for k, v in inp.items()}
    prev = P.set_path(P.SWR_PATH_FFMA)
    try:
        y0 = P.phalanx_mix(g["q"], g["zk"], g["v"], g["za"])
        y1 = P.phalanx_layer_mix(g["q"], g["zk"], g["v"], g["za"], logit_a=False, logit_k=False)
        b0 = P.phalanx_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"])
        b1 = P.phalanx_layer_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"], logit_a=False, logit_k=False)
    finally:
        P.set_path(prev)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)
    for x0, x1 in zip(b0[:4], b1[:4]):
        assert torch.equal(x0, x1)


def test_layer_mix_extreme_logits(P):
    """Saturating logits (|z| up to 40: sigma = 0 or 1 exactly in fp32) stay finite."""
    inp = layer_inputs(1, 64, 8, 32, 2, 4, dtype=torch.float32, seed=3)
    inp["za"] = inp["za"] * 20.0
    inp["zk"] = inp["zk"] * 20.0
    outs, refs = run(P, inp)
    for k, v in outs.items():
        assert torch.isfinite(v).all(), k
    check(outs, refs, 1e-5)


def test_layer_mix_autograd(P):
    """torch.autograd through layer_mix returns the group-summed logit gradients."""
    inp = layer_inputs(1, 50, 8, 16, 2, 4, dtype=torch.float32, seed=9)
    g = {k: v.cuda().requires_grad_(k != "dy") for k, v in inp.items()}
    y = P.layer_mix(g["q"], g["zk"], g["v"], g["za"])
    (y * g["dy"]).sum().backward()
    h = {k: to64(v) for k, v in inp.items()}
    rdq, rdzk, rdv, rdza, _ = oracle.layer_mix_bwd(h["q"], h["zk"], h["v"], h["za"], h["dy"])
    for name, x, r in (("dq", g["q"].grad, rdq), ("dzk", g["zk"].grad, rdzk), ("dv", g["v"].grad, rdv),
                       ("dza", g["za"].grad, rdza)):
        assert normwise(x, r) <= 1e-5, name


# ---------------------------------------------------------------------------
# tensor-core family (bf16, D = 128, H a multiple of 8): forward with sigma and
# group-shared q / k through the TMA maps; backward with sigma when no head shares
# a group (the group sums run on the CUDA-core family)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("B,L,H,Gq,Gk", [(2, 100, 16, 8, 4), (1, 4096, 16, 8, 8), (3, 33, 8, 1, 2),
                                         (1, 1, 24, 24, 24), (2, 200, 16, 16, 16)])
@pytest.mark.parametrize("carry", [False, True])
def test_layer_mix_tc_forward(P, B, L, H, Gq, Gk, carry):
    inp = layer_inputs(B, L, H, 128, Gq, Gk, dtype=torch.bfloat16, seed=L + H + Gq, carry=carry)
    g = {k: v.cuda() for k, v in inp.items()}
    prev = P.set_path(P.SWR_PATH_TC)
    try:
        y, co = P.phalanx_layer_mix(g["q"], g["zk"], g["v"], g["za"], carry_in=g.get("carry_in"), return_carry=True)
        assert P.last_path() == 2
    finally:
        P.set_path(prev)
    torch.cuda.synchronize()
    h = {k: to64(v) for k, v in inp.items()}
    ry, rco = oracle.layer_mix_fwd(h["q"], h["zk"], h["v"], h["za"], carry_in=h.get("carry_in"), carry_out=True)
    check({"y": y, "carry_out": co}, {"y": ry, "carry_out": rco}, 2e-2)


@pytest.mark.parametrize("B,L,H", [(2, 100, 16), (1, 4096, 16), (1, 17, 8), (2, 300, 24)])
@pytest.mark.parametrize("carry", [False, True])
def test_layer_mix_tc_backward(P, B, L, H, carry):
    inp = layer_inputs(B, L, H, 128, dtype=torch.bfloat16, seed=3 * L + H, carry=carry)
    prev = P.set_path(P.SWR_PATH_TC)
    try:
        outs, refs = run(P, inp)
        assert P.last_path() == 2
    finally:
        P.set_path(prev)
    check(outs, refs, 2e-2)


@pytest.mark.parametrize("B,L,H,Gq,Gk", [(2, 100, 16, 4, 4), (1, 4096, 16, 4, 8), (2, 33, 16, 2, 16),
                                         (1, 200, 24, 24, 3), (1, 17, 8, 1, 1)])
def test_layer_mix_tc_backward_groups(P, B, L, H, Gq, Gk):
    """Shared groups on the tensor cores: per-head dq / dk into the scratch the binding
    allocates (phalanx_layer_workspace_bytes), summed per group by a second kernel."""
    inp = layer_inputs(B, L, H, 128, Gq, Gk, dtype=torch.bfloat16, seed=L + 7 * Gq + Gk, carry=True)
    prev = P.set_path(P.SWR_PATH_TC)
    try:
        outs, refs = run(P, inp)
        assert P.last_path() == 2
    finally:
        P.set_path(prev)
    check(outs, refs, 2e-2)


# q and k shared by pairs of heads (the paper's 8 groups at H = 16): the walk
# interleaves a group's two heads block by block and the kernel sums dq / dz_k itself.
# Shapes: one line pair, ragged tails, L = 1 and 15/16/17, item counts below and above
# the SM count, long lines (weighted split, halo super-items), H = 8 / 24.
@pytest.mark.parametrize("B,L,H", [(2, 100, 16), (1, 4096, 16), (1, 1, 16), (3, 15, 8), (2, 16, 8), (1, 17, 24),
                                   (4, 1000, 16), (2, 2049, 24), (8, 512, 16)])
@pytest.mark.parametrize("carry", [False, True])
def test_layer_mix_tc_backward_pairs(P, B, L, H, carry):
    from paper_2512_13921_b200 import _lib, ops
    inp = layer_inputs(B, L, H, 128, H // 2, H // 2, dtype=torch.bfloat16, seed=5 * L + H + carry, carry=carry)
    g = {k: v for k, v in inp.items()}
    assert _lib.phalanx_layer_workspace_bytes(ops._shape(g["v"], g["za"]), ops._layer(g["q"], g["zk"], True, True),
                                              _lib.SWR_BF16) == 0
    prev = P.set_path(P.SWR_PATH_TC)
    try:
        outs, refs = run(P, inp)
        assert P.last_path() == 2
    finally:
        P.set_path(prev)
    check(outs, refs, 2e-2)


@pytest.mark.parametrize("za_shift", [-8.0, -2.0, 3.0, 8.0])
def test_layer_mix_tc_backward_pairs_decays(P, za_shift):
    """Decays from near 0 (sigma(N(0,1) - 8)) to long memory (sigma(N(0,1) + 8)) through
    the paired walk, carries on."""
    inp = layer_inputs(2, 300, 16, 128, 8, 8, dtype=torch.bfloat16, seed=17, carry=True, za_shift=za_shift)
    prev = P.set_path(P.SWR_PATH_TC)
    try:
        outs, refs = run(P, inp)
        assert P.last_path() == 2
    finally:
        P.set_path(prev)
    check(outs, refs, 2e-2)


def test_layer_mix_tc_backward_pairs_repeatable(P):
    """Fixed head order in the fused sums: repeated launches (which move the weighted
    split's range boundaries) give the same bits."""
    inp = layer_inputs(4, 2000, 16, 128, 8, 8, dtype=torch.bfloat16, seed=23)
    g = {k: v.cuda() for k, v in inp.items()}
    prev = P.set_path(P.SWR_PATH_TC)
    try:
        r1 = P.phalanx_layer_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"])
        for _ in range(10):
            r2 = P.phalanx_layer_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"])
    finally:
        P.set_path(prev)
    torch.cuda.synchronize()
    for x1, x2 in zip(r1, r2):
        assert torch.equal(x1, x2)


def test_layer_mix_tc_backward_groups_need_workspace(P):
    """Without the scratch a grouped backward is refused when SWR_PATH_TC is forced (no
    silent fallback) and runs on the CUDA-core family under AUTO."""
    from paper_2512_13921_b200 import _lib, ops
    inp = layer_inputs(1, 64, 16, 128, 4, 4, dtype=torch.bfloat16, seed=1)
    g = {k: v.cuda() for k, v in inp.items()}
    q, zk, v, za, dy = g["q"], g["zk"], g["v"], g["za"], g["dy"]
    outs = [torch.empty_like(q), torch.empty_like(zk), torch.empty_like(v), torch.empty_like(za)]
    mo = torch.empty(1, 16, 128, device="cuda")
    args = (q.data_ptr(), zk.data_ptr(), v.data_ptr(), za.data_ptr(), dy.data_ptr(), *[o.data_ptr() for o in outs],
            None, None, mo.data_ptr(), ops._shape(v, za), ops._layer(q, zk, True, True), _lib.SWR_BF16,
            torch.cuda.current_stream().cuda_stream)
    prev = P.set_path(P.SWR_PATH_TC)
    try:
        assert _lib.raw_status("phalanx_layer_mix_bwd", *args) == 8  # SWR_ERR_UNSUPPORTED
    finally:
        P.set_path(prev)
    P.set_path(P.SWR_PATH_AUTO)
    try:
        assert _lib.raw_status("phalanx_layer_mix_bwd", *args) == 0
        assert P.last_path() == 1
    finally:
        P.set_path(prev)


@pytest.mark.parametrize("path", ["auto", "ffma"])
def test_layer_mix_bwd_deterministic(P, path):
    """The group sums run in a fixed head order on both families: two runs give the
    same bits."""
    inp = layer_inputs(2, 300, 16, 128, 8, 4, dtype=torch.bfloat16, seed=21)
    g = {k: v.cuda() for k, v in inp.items()}
    prev = P.set_path(P.SWR_PATH_AUTO if path == "auto" else P.SWR_PATH_FFMA)
    try:
        r1 = P.phalanx_layer_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"])
        r2 = P.phalanx_layer_mix_bwd(g["q"], g["zk"], g["v"], g["za"], g["dy"])
    finally:
        P.set_path(prev)
    torch.cuda.synchronize()
    for x1, x2 in zip(r1, r2):
        assert torch.equal(x1, x2)
