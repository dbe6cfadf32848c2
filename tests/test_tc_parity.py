"""Oracle parity of the tensor-core family (csrc/swr_tc.cu), forced.

The path bench.py times at the graded shape (bf16, D = 128) is the tcgen05/TMA
kernel family.  Every test here selects SWR_PATH_TC (no silent fallback: a call
outside the envelope raises SWR_ERR_UNSUPPORTED) and asserts that the call was
served by it, then compares WHOLE output tensors with the fp64 oracle on the same
rounded inputs:

* all four ops, H in {8, 16, 24} (8-head decay boxes, one and three boxes), ragged
  and short L (partial last items and blocks: the a = 1 padding, TMA-clipped
  stores), grids below and above the SM count;
* carry_in / mu_in on and off, carry_out / mu_out checked (the segment
  checkpoint of P:1526, the first block's v_{-1} of P:1476);
* every decay family of swr_inputs.DECAY_KINDS (exact 0 and 1, 1e-3, 1 - 2^-8,
  long memory, the bounded-decay ablation of P:1888);
* strided (TMA-addressable) layouts.

Tolerance (BASELINE.json north_star, R10): normwise per tensor,
max|gpu - oracle| <= 2e-2 * max|oracle| for bf16 storage.
"""
import numpy as np
import pytest
import torch

import oracle
from swr_inputs import DECAY_KINDS, mix_inputs, swr_inputs, to64

pytestmark = pytest.mark.gpu
TOL = 2e-2
D = 128


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from conftest import build_lib
    build_lib()
    import paper_2512_13921_b200 as P
    prev = P.set_path(P.SWR_PATH_TC)
    yield P
    P.set_path(prev)


def normwise(x, ref):
    x = x.detach().to("cpu", torch.float64).numpy()
    den = np.max(np.abs(ref)) if ref.size else 0.0
    num = np.max(np.abs(x - ref)) if ref.size else 0.0
    return num / den if den > 0 else num


def check(name, x, ref):
    assert x.shape == ref.shape, (name, tuple(x.shape), ref.shape)
    e = normwise(x, ref)
    assert e <= TOL, f"{name}: normwise error {e:.3e} > {TOL:.0e}"


def cuda(d):
    return {k: v.cuda() for k, v in d.items()}


def run_swr(P, inp, carry):
    g = cuda(inp)
    ci, mi = (g.get("carry_in"), g.get("mu_in")) if carry else (None, None)
    x, co = P.swr_fwd(g["u"], g["a"], carry_in=ci, return_carry=True)
    assert P.last_path() == 2
    du, da, mo = P.swr_bwd(g["u"], g["a"], g["G"], carry_in=ci, mu_in=mi)
    assert P.last_path() == 2
    torch.cuda.synchronize()
    u, a, G = to64(inp["u"]), to64(inp["a"]), to64(inp["G"])
    ci64 = to64(inp["carry_in"]) if carry else None
    mi64 = to64(inp["mu_in"]) if carry else None
    rx, rco = oracle.swr_fwd(u, a, carry_in=ci64, carry_out=True)
    rdu, rda, rmo = oracle.swr_bwd(u, a, G, carry_in=ci64, mu_in=mi64)
    check("x", x, rx)
    check("carry_out", co, rco)
    check("du", du, rdu)
    check("da", da, rda)
    check("mu_out", mo, rmo)


def run_mix(P, inp, carry):
    g = cuda(inp)
    ci, mi = (g.get("carry_in"), g.get("mu_in")) if carry else (None, None)
    y, co = P.phalanx_mix(g["q"], g["k"], g["v"], g["a"], carry_in=ci, return_carry=True)
    assert P.last_path() == 2
    dq, dk, dv, da, mo = P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"], carry_in=ci,
                                           mu_in=mi)
    assert P.last_path() == 2
    torch.cuda.synchronize()
    q, k, v, a, dy = (to64(inp[n]) for n in ("q", "k", "v", "a", "dy"))
    ci64 = to64(inp["carry_in"]) if carry else None
    mi64 = to64(inp["mu_in"]) if carry else None
    ry, rco = oracle.mix_fwd(q, k, v, a, carry_in=ci64, carry_out=True)
    rdq, rdk, rdv, rda, rmo = oracle.mix_bwd(q, k, v, a, dy, carry_in=ci64, mu_in=mi64)
    check("y", y, ry)
    check("carry_out", co, rco)
    check("dq", dq, rdq)
    check("dk", dk, rdk)
    check("dv", dv, rdv)
    check("da", da, rda)
    check("mu_out", mo, rmo)


LENGTHS = [1, 15, 16, 17, 33, 63, 65, 100, 1000, 4096]


@pytest.mark.parametrize("carry", [False, True])
@pytest.mark.parametrize("L", LENGTHS)
@pytest.mark.parametrize("H", [8, 16, 24])
def test_swr_tc_whole_tensor(P, H, L, carry):
    B = 2 if L <= 1000 else 1
    run_swr(P, swr_inputs(B, L, H, D, dtype=torch.bfloat16, seed=17 * L + H, carry=True), carry)


@pytest.mark.parametrize("carry", [False, True])
@pytest.mark.parametrize("L", LENGTHS)
@pytest.mark.parametrize("H", [8, 16, 24])
def test_mix_tc_whole_tensor(P, H, L, carry):
    B = 2 if L <= 1000 else 1
    run_mix(P, mix_inputs(B, L, H, D, dtype=torch.bfloat16, seed=19 * L + H, carry=True), carry)


@pytest.mark.parametrize("L", [100, 1000])
@pytest.mark.parametrize("decay", DECAY_KINDS)
def test_swr_tc_decay_families(P, decay, L):
    run_swr(P, swr_inputs(2, L, 16, D, dtype=torch.bfloat16, seed=5, decay=decay, carry=True), True)


@pytest.mark.parametrize("L", [100, 1000])
@pytest.mark.parametrize("decay", DECAY_KINDS)
def test_mix_tc_decay_families(P, decay, L):
    run_mix(P, mix_inputs(2, L, 16, D, dtype=torch.bfloat16, seed=6, decay=decay, carry=True), True)


def test_tc_grid_above_sm_count_layer_rows(P):
    """Full-length rows of the layer config (L = 4096, H = 16) with B = 3: 3072
    forward items over 148 SMs -- every (b, h) slice of the whole tensor checked."""
    run_swr(P, swr_inputs(3, 4096, 16, D, dtype=torch.bfloat16, seed=77, carry=True), True)
    run_mix(P, mix_inputs(3, 4096, 16, D, dtype=torch.bfloat16, seed=78, carry=True), True)


def test_tc_strided_layouts(P):
    """TMA-addressable non-contiguous layouts: d-tensors are the D = 128 head slice
    of a [B, L, H, 256] buffer, decays the first H heads of a [B, L, H + 8] buffer."""
    B, L, H = 2, 300, 16
    inp = swr_inputs(B, L, H, D, dtype=torch.bfloat16, seed=8, carry=True)
    bu = torch.zeros(B, L, H, 2 * D, dtype=torch.bfloat16)
    bG = torch.zeros(B, L, H, 2 * D, dtype=torch.bfloat16)
    ba = torch.zeros(B, L, H + 8, dtype=torch.bfloat16)
    bu[..., D:] = inp["u"]
    bG[..., D:] = inp["G"]
    ba[..., :H] = inp["a"]
    u, G, a = bu.cuda()[..., D:], bG.cuda()[..., D:], ba.cuda()[..., :H]
    ci, mi = inp["carry_in"].cuda(), inp["mu_in"].cuda()
    x, co = P.swr_fwd(u, a, carry_in=ci, return_carry=True)
    assert P.last_path() == 2 and x.stride() == u.stride()
    du, da, mo = P.swr_bwd(u, a, G, carry_in=ci, mu_in=mi)
    assert P.last_path() == 2 and da.stride() == a.stride()
    torch.cuda.synchronize()
    h = {k: to64(v) for k, v in inp.items()}
    rx, rco = oracle.swr_fwd(h["u"], h["a"], carry_in=h["carry_in"], carry_out=True)
    rdu, rda, rmo = oracle.swr_bwd(h["u"], h["a"], h["G"], carry_in=h["carry_in"], mu_in=h["mu_in"])
    check("x", x, rx)
    check("carry_out", co, rco)
    check("du", du, rdu)
    check("da", da, rda)
    check("mu_out", mo, rmo)


def test_forced_tc_outside_envelope_raises(P):
    """SWR_PATH_TC never falls back silently: fp32, D != 128, or decays TMA cannot
    address (heads not contiguous) give SWR_ERR_UNSUPPORTED."""
    cases = [swr_inputs(1, 32, 8, D, dtype=torch.float32, seed=1),
             swr_inputs(1, 32, 8, 64, dtype=torch.bfloat16, seed=1)]
    for inp in cases:
        g = cuda(inp)
        with pytest.raises(P.SwrError) as ei:
            P.swr_fwd(g["u"], g["a"])
        assert ei.value.status == 8
    g = cuda(swr_inputs(1, 32, 8, D, dtype=torch.bfloat16, seed=1))
    a_hl = g["a"].transpose(1, 2).contiguous().transpose(1, 2)  # [B, H, L] storage
    with pytest.raises(P.SwrError) as ei:
        P.swr_bwd(g["u"], a_hl, g["G"])
    assert ei.value.status == 8


def test_path_selector_is_per_thread(P):
    """swr_set_path is thread-local: another thread's choice does not change ours."""
    import threading
    seen = {}

    def other():
        seen["initial"] = P.set_path(P.SWR_PATH_FFMA)  # a new thread starts at AUTO
        g = cuda(swr_inputs(1, 32, 8, D, dtype=torch.bfloat16, seed=2))
        P.swr_fwd(g["u"], g["a"])
        seen["path"] = P.last_path()

    t = threading.Thread(target=other)
    t.start()
    t.join()
    assert seen == {"initial": P.SWR_PATH_AUTO, "path": 1}
    g = cuda(swr_inputs(1, 32, 8, D, dtype=torch.bfloat16, seed=2))
    P.swr_fwd(g["u"], g["a"])
    assert P.last_path() == 2  # this thread still has SWR_PATH_TC
