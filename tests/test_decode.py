"""Recurrence-mode decoding (include/swr.h swr_decode_step; SURVEY 8(f)
NEXT-3) on the GPU: a sequence decoded one token at a time matches the fp64 oracle's
plain definition of the whole-sequence operator (oracle.swr_fwd / mix_fwd) within
the north-star tolerance, and is bitwise the CUDA-core forward (same ops, same
order)."""
import numpy as np
import pytest
import torch

import oracle
from swr_inputs import mix_inputs, swr_inputs, to64

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
    x = x.detach().double().cpu().numpy()
    return np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("D,H", [(16, 3), (32, 1), (128, 16), (64, 5)])
@pytest.mark.parametrize("carry", [False, True])
def test_swr_decode_matches_oracle_and_forward(P, dtype, D, H, carry):
    B, L = 2, 40
    inp = swr_inputs(B, L, H, D, dtype=dtype, seed=300 + D + H, carry=carry)
    u, a = inp["u"].cuda(), inp["a"].cuda()
    ci = inp["carry_in"].cuda() if carry else None
    st = P.DecodeState(B, H, D, u.device, carry_in=ci)
    launches = P.launch_count()
    x = torch.stack([P.swr_decode_step(u[:, n], a[:, n], st) for n in range(L)], dim=1)
    assert P.launch_count() - launches == L
    assert st.pos == L
    # the plain definition: x~ = L~ u of the whole sequence (the jagged operator)
    ref = oracle.swr_fwd(to64(inp["u"]), to64(inp["a"]), carry_in=to64(inp.get("carry_in")))
    assert normwise(x, ref) <= TOL[dtype]
    prev = P.set_path(P.SWR_PATH_FFMA)
    try:
        xf, co = P.swr_fwd(u, a, carry_in=ci, return_carry=True)
    finally:
        P.set_path(prev)
    assert torch.equal(x, xf)
    # the state after L tokens: w is carry_out (the local state at token L-1)
    assert torch.equal(st.w, co)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("D,H", [(16, 4), (128, 8)])
def test_mix_decode_matches_oracle_and_forward(P, dtype, D, H):
    B, L = 2, 37
    inp = mix_inputs(B, L, H, D, dtype=dtype, seed=400 + D, carry=True)
    q, k, v, a = (inp[n].cuda() for n in ("q", "k", "v", "a"))
    ci = inp["carry_in"].cuda()
    st = P.DecodeState(B, H, D, q.device, carry_in=ci)
    y = torch.stack([P.phalanx_mix_decode_step(q[:, n], k[:, n], v[:, n], a[:, n], st) for n in range(L)],
                    dim=1)
    ref = oracle.mix_fwd(*(to64(inp[n]) for n in ("q", "k", "v", "a")), carry_in=to64(inp["carry_in"]))
    assert normwise(y, ref) <= TOL[dtype]
    prev = P.set_path(P.SWR_PATH_FFMA)
    try:
        yf = P.phalanx_mix(q, k, v, a, carry_in=ci)
    finally:
        P.set_path(prev)
    assert torch.equal(y, yf)


@pytest.mark.parametrize("P_len", [0, 5, 16, 37, 64])
def test_prefill_then_decode_continues_the_forward(P, P_len):
    """State seeded from a prompt (at most its last 31 tokens) + decoding the rest
    gives bitwise the CUDA-core forward of the whole sequence from position P on."""
    B, L, H, D = 2, 80, 3, 32
    dtype = torch.bfloat16
    inp = swr_inputs(B, L, H, D, dtype=dtype, seed=700 + P_len, carry=True)
    u, a, ci = inp["u"].cuda(), inp["a"].cuda(), inp["carry_in"].cuda()
    st = P.DecodeState(B, H, D, u.device, carry_in=ci).prefill(u[:, :P_len], a[:, :P_len])
    assert st.pos == P_len
    x = torch.stack([P.swr_decode_step(u[:, n], a[:, n], st) for n in range(P_len, L)], dim=1)
    prev = P.set_path(P.SWR_PATH_FFMA)
    try:
        xf = P.swr_fwd(u, a, carry_in=ci)
        mq, mk, mv = (torch.randn(B, L, H, D, device="cuda").to(dtype) for _ in range(3))
        yf = P.phalanx_mix(mq, mk, mv, a, carry_in=ci)
    finally:
        P.set_path(prev)
    assert torch.equal(x, xf[:, P_len:])
    sm = P.DecodeState(B, H, D, u.device, carry_in=ci).prefill(None, a[:, :P_len], k=mk[:, :P_len],
                                                                 v=mv[:, :P_len])
    y = torch.stack([P.phalanx_mix_decode_step(mq[:, n], mk[:, n], mv[:, n], a[:, n], sm)
                     for n in range(P_len, L)], dim=1)
    assert torch.equal(y, yf[:, P_len:])
