"""Exact full-range recurrence (include/swr.h swr_exact_fwd; Alg. 2 P:684-708;
SURVEY 8(f) NEXT-2) against the fp64 Eq. 2.1 oracle (oracle.linrec_fwd, pinned to
the dense operator and the geometric closed form in test_oracle.py)."""
import numpy as np
import pytest
import torch

import oracle
from swr_inputs import swr_inputs, to64

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
@pytest.mark.parametrize("D", [16, 64, 128])
@pytest.mark.parametrize("B,L,H", [(2, 16, 3), (1, 77, 5), (2, 1000, 16), (1, 4096, 2)])
@pytest.mark.parametrize("carry", [False, True])
def test_exact_matches_full_recurrence(P, dtype, D, B, L, H, carry):
    inp = swr_inputs(B, L, H, D, dtype=dtype, seed=600 + L + D, carry=carry)
    u, a = inp["u"].cuda(), inp["a"].cuda()
    ci = inp["carry_in"].cuda() if carry else None
    x, co = P.swr_exact_fwd(u, a, carry_in=ci, return_carry=True)
    torch.cuda.synchronize()
    rx, rlast = oracle.linrec_fwd(to64(inp["u"]), to64(inp["a"]), to64(inp.get("carry_in")))
    assert normwise(x, rx) <= TOL[dtype]
    assert normwise(co, rlast) <= TOL[dtype]


def test_exact_differs_from_truncated_only_past_two_blocks(P):
    inp = swr_inputs(2, 200, 4, 32, dtype=torch.float32, seed=9)
    u, a = inp["u"].cuda(), inp["a"].cuda()
    xe = P.swr_exact_fwd(u, a)
    xs = P.swr_fwd(u, a)
    assert torch.allclose(xe[:, :32], xs[:, :32], rtol=1e-6, atol=1e-6)
    assert not torch.allclose(xe[:, 32:], xs[:, 32:], rtol=1e-6, atol=1e-6)


def test_exact_empty(P):
    u = torch.zeros(2, 0, 3, 16, device="cuda")
    a = torch.zeros(2, 0, 3, device="cuda")
    ci = torch.randn(2, 3, 16, device="cuda")
    x, co = P.swr_exact_fwd(u, a, carry_in=ci, return_carry=True)
    assert x.shape == u.shape and torch.count_nonzero(co) == 0


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("D", [16, 32, 128])
@pytest.mark.parametrize("B,L,H", [(2, 16, 3), (1, 77, 5), (2, 1000, 16), (1, 4096, 2)])
@pytest.mark.parametrize("carry", [False, True])
def test_exact_backward_matches_oracle(P, dtype, D, B, L, H, carry):
    inp = swr_inputs(B, L, H, D, dtype=dtype, seed=800 + L + D, carry=carry)
    u, a, G = inp["u"].cuda(), inp["a"].cuda(), inp["G"].cuda()
    ci = inp["carry_in"].cuda() if carry else None
    mi = inp["mu_in"].cuda() if carry else None
    du, da, mo = P.swr_exact_bwd(u, a, G, carry_in=ci, mu_in=mi)
    torch.cuda.synchronize()
    rdu, rda, rmo = oracle.linrec_bwd(to64(inp["u"]), to64(inp["a"]), to64(inp["G"]),
                                      to64(inp.get("carry_in")), to64(inp.get("mu_in")))
    assert normwise(du, rdu) <= TOL[dtype]
    assert normwise(da, rda) <= TOL[dtype]
    assert normwise(mo, rmo) <= TOL[dtype]


def test_exact_autograd(P):
    inp = swr_inputs(2, 100, 3, 16, dtype=torch.float32, seed=5, carry=True)
    u = inp["u"].cuda().requires_grad_()
    a = inp["a"].cuda().requires_grad_()
    c = inp["carry_in"].cuda().requires_grad_()
    G = inp["G"].cuda()
    x = P.swr_exact(u, a, c)
    (x * G).sum().backward()
    du, da, mo = P.swr_exact_bwd(u.detach(), a.detach(), G, carry_in=c.detach())
    assert torch.equal(u.grad, du) and torch.equal(a.grad, da) and torch.equal(c.grad, mo)


@pytest.mark.parametrize("L", [17, 33, 48, 8192])
@pytest.mark.parametrize("decay", ["sigmoid3", "one", "zero"])
def test_exact_lookback_chains(P, L, decay):
    """The single-pass forward's decoupled look-back (include/swr.h swr_exact_fwd):
    long memory (decays near or at 1) carries the state across every chunk; a = 0
    cuts it; short sequences have one to three 16-token blocks (one or two chunks).
    Called twice: the flags are reset per launch."""
    inp = swr_inputs(2, L, 4, 32, dtype=torch.float32, seed=L, decay=decay, carry=True)
    u, a, ci = inp["u"].cuda(), inp["a"].cuda(), inp["carry_in"].cuda()
    rx, rlast = oracle.linrec_fwd(to64(inp["u"]), to64(inp["a"]), to64(inp["carry_in"]))
    for _ in range(2):
        x, co = P.swr_exact_fwd(u, a, carry_in=ci, return_carry=True)
        torch.cuda.synchronize()
        assert normwise(x, rx) <= 1e-5
        assert normwise(co, rlast) <= 1e-5


@pytest.mark.parametrize("L", [16 * 1024 + 5, 16 * 1100])
def test_exact_bwd_lookback_scans(P, L):
    """From 1024 blocks per line the backward resolves both carrier chains by decoupled
    look-back scans (include/swr.h swr_exact_bwd); long-memory decays carry the adjoint
    across every chunk."""
    inp = swr_inputs(1, L, 2, 16, dtype=torch.float32, seed=L, decay="sigmoid3", carry=True)
    u, a, G = inp["u"].cuda(), inp["a"].cuda(), inp["G"].cuda()
    ci, mi = inp["carry_in"].cuda(), inp["mu_in"].cuda()
    du, da, mo = P.swr_exact_bwd(u, a, G, carry_in=ci, mu_in=mi)
    torch.cuda.synchronize()
    rdu, rda, rmo = oracle.linrec_bwd(to64(inp["u"]), to64(inp["a"]), to64(inp["G"]), to64(inp["carry_in"]),
                                      to64(inp["mu_in"]))
    assert normwise(du, rdu) <= 1e-5
    assert normwise(da, rda) <= 1e-5
    assert normwise(mo, rmo) <= 1e-5


@pytest.mark.parametrize("L", [1, 16, 100, 4096, 16 * 1030 + 3])
@pytest.mark.parametrize("decay", ["sigmoid", "sigmoid3", "one"])
def test_exact_fwd_tensor_cores(P, L, decay):
    """bf16, d = 128: the look-back scan's per-block carriers, then the B2P forward's
    tensor-core Pass I with the exact carrier (swr_tc.cu Cfg<6>)."""
    inp = swr_inputs(1, L, 16, 128, dtype=torch.bfloat16, seed=L + 5, decay=decay, carry=True)
    u, a, ci = inp["u"].cuda(), inp["a"].cuda(), inp["carry_in"].cuda()
    prev = P.set_path(P.SWR_PATH_TC)
    try:
        x, co = P.swr_exact_fwd(u, a, carry_in=ci, return_carry=True)
        assert P.last_path() == 2
    finally:
        P.set_path(prev)
    torch.cuda.synchronize()
    rx, rlast = oracle.linrec_fwd(to64(inp["u"]), to64(inp["a"]), to64(inp["carry_in"]))
    assert normwise(x, rx) <= 2e-2
    assert normwise(co, rlast) <= 2e-2
