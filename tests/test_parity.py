"""GPU parity: every C-ABI entry point against the fp64 oracle on the same
seeded inputs (the oracle sees the already-rounded storage values upcast to
fp64, R10).

Tolerance (BASELINE.json north_star; normwise, the metric of Fig. 7):
    max |gpu - oracle| <= tol * max |oracle|   per output tensor,
    tol = 1e-5 for fp32 storage, 2e-2 for bf16 storage.
carry_out / mu_out are fp32 outputs computed from storage-dtype inputs; they get
the tolerance of that dtype (the tensor-core path forms them from bf16 L_t,
P:1526).
"""
import numpy as np
import pytest
import torch

import oracle
from swr_inputs import mix_inputs, swr_inputs, to64, DECAY_KINDS

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-5, torch.bfloat16: 2e-2}


@pytest.fixture(scope="module", params=["auto", "ffma"])
def P(request):
    """Every test runs on both kernel families: AUTO (tcgen05/TMA for bf16 D=128,
    FFMA otherwise) and FFMA forced everywhere."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from conftest import build_lib
    build_lib()
    import paper_2512_13921_b200 as P
    prev = P.set_path(P.SWR_PATH_AUTO if request.param == "auto" else P.SWR_PATH_FFMA)
    yield P
    P.set_path(prev)


def normwise(x, ref):
    x = x.detach().to("cpu", torch.float64).numpy() if torch.is_tensor(x) else x
    den = np.max(np.abs(ref)) if ref.size else 0.0
    num = np.max(np.abs(x - ref)) if ref.size else 0.0
    return num / den if den > 0 else num


def assert_close(name, x, ref, tol):
    e = normwise(x, ref)
    assert e <= tol, f"{name}: normwise error {e:.3e} > {tol:.1e}"
    return e


def cuda(d):
    return {k: (v.cuda() if torch.is_tensor(v) else v) for k, v in d.items()}


# ---------------------------------------------------------------------------
# swr_fwd / swr_bwd over dtype x head dim x ragged lengths
# ---------------------------------------------------------------------------
SHAPES = [(2, 16, 3), (2, 48, 3), (1, 65, 5), (3, 200, 2), (1, 64, 1)]


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("D", [16, 32, 64, 128])
@pytest.mark.parametrize("B,L,H", SHAPES)
@pytest.mark.parametrize("carry", [False, True])
def test_swr_fwd_bwd_parity(P, dtype, D, B, L, H, carry):
    inp = swr_inputs(B, L, H, D, dtype=dtype, seed=B * 1000 + L + D, carry=carry)
    g = cuda(inp)
    ci = g.get("carry_in")
    mi = g.get("mu_in")
    x, co = P.swr_fwd(g["u"], g["a"], carry_in=ci, return_carry=True)
    du, da, mo = P.swr_bwd(g["u"], g["a"], g["G"], carry_in=ci, mu_in=mi)
    torch.cuda.synchronize()
    u64, a64, G64 = to64(inp["u"]), to64(inp["a"]), to64(inp["G"])
    ci64, mi64 = to64(inp.get("carry_in")), to64(inp.get("mu_in"))
    rx, rco = oracle.swr_fwd(u64, a64, carry_in=ci64, carry_out=True)
    rdu, rda, rmo = oracle.swr_bwd(u64, a64, G64, carry_in=ci64, mu_in=mi64)
    tol = TOL[dtype]
    assert_close("x", x, rx, tol)
    assert_close("carry_out", co, rco, tol)
    assert_close("du", du, rdu, tol)
    assert_close("da", da, rda, tol)
    assert_close("mu_out", mo, rmo, tol)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("D", [16, 64, 128])
@pytest.mark.parametrize("B,L,H", [(2, 48, 3), (1, 77, 2), (2, 160, 17)])
@pytest.mark.parametrize("carry", [False, True])
def test_mix_fwd_bwd_parity(P, dtype, D, B, L, H, carry):
    inp = mix_inputs(B, L, H, D, dtype=dtype, seed=7 + B + L + D, carry=carry)
    g = cuda(inp)
    ci, mi = g.get("carry_in"), g.get("mu_in")
    y, co = P.phalanx_mix(g["q"], g["k"], g["v"], g["a"], carry_in=ci, return_carry=True)
    dq, dk, dv, da, mo = P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"], carry_in=ci,
                                           mu_in=mi)
    torch.cuda.synchronize()
    q, k, v, a, dy = (to64(inp[n]) for n in ("q", "k", "v", "a", "dy"))
    ci64, mi64 = to64(inp.get("carry_in")), to64(inp.get("mu_in"))
    ry, rco = oracle.mix_fwd(q, k, v, a, carry_in=ci64, carry_out=True)
    rdq, rdk, rdv, rda, rmo = oracle.mix_bwd(q, k, v, a, dy, carry_in=ci64, mu_in=mi64)
    tol = TOL[dtype]
    assert_close("y", y, ry, tol)
    assert_close("carry_out", co, rco, tol)
    assert_close("dq", dq, rdq, tol)
    assert_close("dk", dk, rdk, tol)
    assert_close("dv", dv, rdv, tol)
    assert_close("da", da, rda, tol)
    assert_close("mu_out", mo, rmo, tol)


# ---------------------------------------------------------------------------
# adversarial decay families (exact 0 and 1, tiny, 1 - 2^-8, long memory)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("decay", DECAY_KINDS)
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_decay_families(P, decay, dtype):
    B, L, H, D = 2, 97, 3, 64
    inp = swr_inputs(B, L, H, D, dtype=dtype, seed=99, decay=decay, carry=True)
    g = cuda(inp)
    x = P.swr_fwd(g["u"], g["a"], carry_in=g["carry_in"])
    du, da, mo = P.swr_bwd(g["u"], g["a"], g["G"], carry_in=g["carry_in"], mu_in=g["mu_in"])
    torch.cuda.synchronize()
    args = (to64(inp["u"]), to64(inp["a"]))
    rx = oracle.swr_fwd(*args, carry_in=to64(inp["carry_in"]))
    rdu, rda, rmo = oracle.swr_bwd(*args, to64(inp["G"]), carry_in=to64(inp["carry_in"]),
                                   mu_in=to64(inp["mu_in"]))
    tol = TOL[dtype]
    assert_close("x", x, rx, tol)
    assert_close("du", du, rdu, tol)
    assert_close("da", da, rda, tol)
    assert_close("mu_out", mo, rmo, tol)


# ---------------------------------------------------------------------------
# BASELINE.json configs
# ---------------------------------------------------------------------------
def test_tiny_config_fp32(P):
    """BJ configs[0]: B=1, H=1, L=64 (4 blocks), d=16, fp32, decays in (0,1)."""
    inp = swr_inputs(1, 64, 1, 16, dtype=torch.float32, seed=0, decay="uniform")
    g = cuda(inp)
    x = P.swr_fwd(g["u"], g["a"])
    du, da, _ = P.swr_bwd(g["u"], g["a"], g["G"])
    torch.cuda.synchronize()
    u, a, G = to64(inp["u"]), to64(inp["a"]), to64(inp["G"])
    assert_close("x", x, oracle.swr_fwd(u, a), 1e-5)
    rdu, rda, _ = oracle.swr_bwd(u, a, G)
    assert_close("du", du, rdu, 1e-5)
    assert_close("da", da, rda, 1e-5)


def _sampled_pairs(B, H, n, seed=0):
    r = np.random.default_rng(seed)
    return [(int(r.integers(B)), int(r.integers(H))) for _ in range(n)]


@pytest.mark.parametrize("op", ["swr", "mix"])
def test_layer_config_sampled(P, op):
    """BJ configs[1] at full size (B=8, H=16, L=4096, d=128, bf16) in the launch
    configuration bench.py times; the oracle checks 6 sampled (b, h) slices."""
    B, L, H, D = 8, 4096, 16, 128
    if op == "swr":
        inp = swr_inputs(B, L, H, D, dtype=torch.bfloat16, seed=1)
        g = cuda(inp)
        x = P.swr_fwd(g["u"], g["a"])
        du, da, _ = P.swr_bwd(g["u"], g["a"], g["G"])
        outs = {"x": x, "du": du, "da": da}
    else:
        inp = mix_inputs(B, L, H, D, dtype=torch.bfloat16, seed=1)
        g = cuda(inp)
        y = P.phalanx_mix(g["q"], g["k"], g["v"], g["a"])
        dq, dk, dv, da, _ = P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"])
        outs = {"y": y, "dq": dq, "dk": dk, "dv": dv, "da": da}
    torch.cuda.synchronize()
    for b, h in _sampled_pairs(B, H, 6):
        sl4 = (slice(b, b + 1), slice(None), slice(h, h + 1))
        s = {k: to64(v[sl4]) for k, v in inp.items()}
        if op == "swr":
            rx = oracle.swr_fwd(s["u"], s["a"])
            rdu, rda, _ = oracle.swr_bwd(s["u"], s["a"], s["G"])
            refs = {"x": rx, "du": rdu, "da": rda}
        else:
            ry = oracle.mix_fwd(s["q"], s["k"], s["v"], s["a"])
            rdq, rdk, rdv, rda, _ = oracle.mix_bwd(s["q"], s["k"], s["v"], s["a"], s["dy"])
            refs = {"y": ry, "dq": rdq, "dk": rdk, "dv": rdv, "da": rda}
        for k, ref in refs.items():
            assert_close(f"{k}[b={b},h={h}]", outs[k][sl4], ref, 2e-2)


# ---------------------------------------------------------------------------
# layouts: strided d-tensors (sliced head dim) and [B, H, L] decays
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_strided_layouts(P, dtype):
    B, L, H, D = 2, 70, 3, 32
    inp = swr_inputs(B, L, H, D, dtype=dtype, seed=5)
    big = torch.zeros(B, L, H, 2 * D, dtype=dtype)
    big[..., :D] = inp["u"]
    bigG = torch.zeros(B, L, H, 2 * D, dtype=dtype)
    bigG[..., D:] = inp["G"]
    u = big.cuda()[..., :D]
    G = bigG.cuda()[..., D:]
    a_t = inp["a"].transpose(1, 2).contiguous().cuda().transpose(1, 2)  # [B,L,H] view of [B,H,L]
    assert u.stride() == G.stride() and a_t.stride(1) == 1
    x = P.swr_fwd(u, a_t)
    du, da, _ = P.swr_bwd(u, a_t, G)
    torch.cuda.synchronize()
    assert x.stride() == u.stride()
    rx = oracle.swr_fwd(to64(inp["u"]), to64(inp["a"]))
    rdu, rda, _ = oracle.swr_bwd(to64(inp["u"]), to64(inp["a"]), to64(inp["G"]))
    assert_close("x", x, rx, TOL[dtype])
    assert_close("du", du, rdu, TOL[dtype])
    assert_close("da", da, rda, TOL[dtype])


def test_empty_and_degenerate(P):
    for L in (0, 1):
        inp = swr_inputs(2, L, 3, 16, dtype=torch.float32, seed=3, carry=True)
        g = cuda(inp)
        x, co = P.swr_fwd(g["u"], g["a"], carry_in=g["carry_in"], return_carry=True)
        du, da, mo = P.swr_bwd(g["u"], g["a"], g["G"], carry_in=g["carry_in"], mu_in=g["mu_in"])
        torch.cuda.synchronize()
        rx, rco = oracle.swr_fwd(to64(inp["u"]), to64(inp["a"]), carry_in=to64(inp["carry_in"]),
                                 carry_out=True)
        rdu, rda, rmo = oracle.swr_bwd(to64(inp["u"]), to64(inp["a"]), to64(inp["G"]),
                                       carry_in=to64(inp["carry_in"]), mu_in=to64(inp["mu_in"]))
        if L == 0:
            assert x.numel() == 0 and torch.all(co == 0) and torch.all(mo == 0)
        else:
            assert_close("x", x, rx, 1e-5)
            assert_close("co", co, rco, 1e-5)
            assert_close("du", du, rdu, 1e-5)
            assert_close("da", da, rda, 1e-5)
            assert_close("mo", mo, rmo, 1e-5)


def test_autograd_wrapper(P):
    inp = mix_inputs(2, 50, 2, 32, dtype=torch.float32, seed=11)
    g = {k: v.cuda().requires_grad_(True) for k, v in inp.items() if k != "dy"}
    y = P.mix(g["q"], g["k"], g["v"], g["a"])
    y.backward(inp["dy"].cuda())
    rdq, rdk, rdv, rda, _ = oracle.mix_bwd(*(to64(inp[n]) for n in ("q", "k", "v", "a", "dy")))
    assert_close("dq", g["q"].grad, rdq, 1e-5)
    assert_close("dk", g["k"].grad, rdk, 1e-5)
    assert_close("dv", g["v"].grad, rdv, 1e-5)
    assert_close("da", g["a"].grad, rda, 1e-5)


def test_tensor_core_path_is_taken_for_the_graded_shape(P):
    """bf16, D = 128 must run on the tcgen05 family under AUTO (no silent fallback)."""
    inp = swr_inputs(2, 64, 16, 128, dtype=torch.bfloat16, seed=1)
    g = cuda(inp)
    prev = P.set_path(P.SWR_PATH_AUTO)
    try:
        P.swr_fwd(g["u"], g["a"])
        assert P.last_path() == 2
        P.swr_bwd(g["u"], g["a"], g["G"])
        assert P.last_path() == 2
        P.set_path(P.SWR_PATH_FFMA)
        P.swr_fwd(g["u"], g["a"])
        assert P.last_path() == 1
    finally:
        P.set_path(prev)
