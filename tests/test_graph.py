"""CUDA-graph capture of the C-ABI calls: a captured fwd+bwd step, replayed on new
inputs copied into its static tensors, gives bitwise the same outputs as the eager
calls.  Captured tensor-core launches cannot use the per-SM weighted split (its
claim epoch would repeat on replay), so they take the uniform split by CTA index;
the results do not depend on the split (test_props.py)."""
import pytest
import torch

from swr_inputs import mix_inputs, swr_inputs

pytestmark = pytest.mark.gpu

CASES = [("tc", torch.bfloat16, 128, 16), ("ffma", torch.float32, 64, 5), ("ffma", torch.bfloat16, 16, 33)]


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from conftest import build_lib
    build_lib()
    import paper_2512_13921_b200 as P
    return P


def _step(P, op, t):
    if op == "swr":
        x = P.swr_fwd(t["u"], t["a"])
        du, da, _ = P.swr_bwd(t["u"], t["a"], t["G"])
        return (x, du, da)
    y = P.phalanx_mix(t["q"], t["k"], t["v"], t["a"])
    dq, dk, dv, da, _ = P.phalanx_mix_bwd(t["q"], t["k"], t["v"], t["a"], t["dy"])
    return (y, dq, dk, dv, da)


@pytest.mark.parametrize("op", ["swr", "mix"])
@pytest.mark.parametrize("path,dtype,D,H", CASES)
def test_graph_replay_matches_eager(P, op, path, dtype, D, H):
    want = P.SWR_PATH_TC if path == "tc" else P.SWR_PATH_FFMA
    prev = P.set_path(want)
    try:
        B, L = 2, 1000  # ragged: 62.5 blocks per line
        gen = swr_inputs if op == "swr" else mix_inputs
        static = {k: v.cuda() for k, v in gen(B, L, H, D, dtype=dtype, seed=1).items()}
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up outside the capture (torch's recipe)
            for _ in range(3):
                _step(P, op, static)
        torch.cuda.current_stream().wait_stream(side)
        assert P.last_path() == want
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            outs = _step(P, op, static)
        for seed in (11, 12, 13):
            for k, v in gen(B, L, H, D, dtype=dtype, seed=seed).items():
                static[k].copy_(v)
            g.replay()
            torch.cuda.synchronize()
            got = [o.clone() for o in outs]
            ref = _step(P, op, static)
            torch.cuda.synchronize()
            for i, (x, r) in enumerate(zip(got, ref)):
                assert torch.equal(x, r), f"output {i} differs after replay (seed {seed})"
    finally:
        P.set_path(prev)
