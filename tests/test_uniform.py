"""Uniform-window recurrence (include/swr.h swr_uniform_fwd; Eq. banded_L P:1104-1113;
SURVEY 8(f) NEXT-4) against the fp64 early-stopped Kogge-Stone oracle (pinned to the
dense banded operator in test_oracle.py)."""
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
@pytest.mark.parametrize("k", [1, 4, 16, 32])
@pytest.mark.parametrize("D", [16, 128])
@pytest.mark.parametrize("B,L,H", [(2, 7, 3), (1, 100, 5), (2, 1000, 16)])
def test_uniform_matches_oracle(P, dtype, k, D, B, L, H):
    inp = swr_inputs(B, L, H, D, dtype=dtype, seed=1000 + k + L)
    x = P.swr_uniform_fwd(inp["u"].cuda(), inp["a"].cuda(), k)
    torch.cuda.synchronize()
    ref = oracle.uniform_fwd(to64(inp["u"]), to64(inp["a"]), k)
    assert normwise(x, ref) <= TOL[dtype]


def test_uniform_rejects_bad_window(P):
    u = torch.zeros(1, 16, 1, 16, device="cuda")
    a = torch.zeros(1, 16, 1, device="cuda")
    for k in (0, 3, 64):
        with pytest.raises(P.SwrError):
            P.swr_uniform_fwd(u, a, k)
