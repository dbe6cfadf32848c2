"""Bit-exact properties of the CUDA path (SURVEY.md pin P6, P8, P9): gate and
decay special cases, locality, shifting by a zero block, run-to-run
determinism, invariance to the kernel's internal chunking, and sequence-parallel
stitching through carry_out -> carry_in / mu_out -> mu_in."""
import pytest
import torch

from swr_inputs import mix_inputs, swr_inputs

pytestmark = pytest.mark.gpu
ELL = 16


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


def cuda(d):
    return {k: v.cuda() for k, v in d.items()}


DT = [torch.float32, torch.bfloat16]


@pytest.mark.parametrize("dtype", DT)
def test_zero_decay_is_identity(P, dtype):
    g = cuda(swr_inputs(2, 100, 3, 64, dtype=dtype, seed=1, decay="zero"))
    assert torch.equal(P.swr_fwd(g["u"], g["a"]), g["u"])


@pytest.mark.parametrize("dtype", DT)
def test_gate_identities(P, dtype):
    g = cuda(mix_inputs(2, 100, 3, 128, dtype=dtype, seed=2))
    assert torch.equal(P.phalanx_mix(torch.zeros_like(g["q"]), g["k"], g["v"], g["a"]), g["v"])
    assert torch.equal(P.phalanx_mix(g["q"], torch.zeros_like(g["k"]), g["v"], g["a"]), g["v"])


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("D", [16, 128])
def test_locality(P, dtype, D):
    L, t = 160, 4
    g = cuda(swr_inputs(1, L, 2, D, dtype=dtype, seed=3))
    x0 = P.swr_fwd(g["u"], g["a"])
    du0, da0, _ = P.swr_bwd(g["u"], g["a"], g["G"])
    sl = slice(t * ELL, (t + 1) * ELL)

    def changed(p, q):
        d = (p.float() - q.float()).abs().reshape(1, L // ELL, -1).amax(dim=(0, 2))
        return set(torch.nonzero(d).flatten().tolist())

    u1 = g["u"].clone(); u1[:, sl] += 1
    assert changed(P.swr_fwd(u1, g["a"]), x0) <= {t, t + 1}
    G1 = g["G"].clone(); G1[:, sl] += 1
    du1, da1, _ = P.swr_bwd(g["u"], g["a"], G1)
    assert changed(du1, du0) <= {t - 1, t}
    assert changed(da1, da0) <= {t - 1, t}
    a1 = g["a"].clone(); a1[:, sl] *= 0.5
    du1, da1, _ = P.swr_bwd(g["u"], a1, g["G"])
    assert changed(P.swr_fwd(g["u"], a1), x0) <= {t, t + 1}
    assert changed(du1, du0) <= {t - 1, t}
    assert changed(da1, da0) <= {t - 1, t, t + 1}


@pytest.mark.parametrize("dtype", DT)
def test_prepending_a_zero_block_shifts_output(P, dtype):
    g = cuda(swr_inputs(2, 96, 3, 32, dtype=dtype, seed=4))
    x = P.swr_fwd(g["u"], g["a"])
    u2 = torch.cat([torch.zeros_like(g["u"][:, :ELL]), g["u"]], dim=1)
    a2 = torch.cat([torch.full_like(g["a"][:, :ELL], 0.5), g["a"]], dim=1)
    assert torch.equal(P.swr_fwd(u2, a2)[:, ELL:], x)


@pytest.mark.parametrize("dtype", DT)
def test_run_to_run_determinism(P, dtype):
    g = cuda(mix_inputs(4, 512, 16, 128, dtype=dtype, seed=5))
    r1 = P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"])
    r2 = P.phalanx_mix_bwd(g["q"], g["k"], g["v"], g["a"], g["dy"])
    for p, q in zip(r1, r2):
        assert torch.equal(p, q)


@pytest.mark.parametrize("dtype", DT)
def test_batch_slice_invariance(P, dtype):
    """The kernels pick their chunk size from B*H; a batch row computed alone
    (different chunking) must match the same row of the batched call bitwise."""
    g = cuda(swr_inputs(8, 1024, 16, 128, dtype=dtype, seed=6))
    x = P.swr_fwd(g["u"], g["a"])
    du, da, _ = P.swr_bwd(g["u"], g["a"], g["G"])
    for b in (0, 5):
        xb = P.swr_fwd(g["u"][b:b + 1].contiguous(), g["a"][b:b + 1].contiguous())
        dub, dab, _ = P.swr_bwd(g["u"][b:b + 1].contiguous(), g["a"][b:b + 1].contiguous(),
                                g["G"][b:b + 1].contiguous())
        assert torch.equal(xb, x[b:b + 1])
        assert torch.equal(dub, du[b:b + 1])
        assert torch.equal(dab, da[b:b + 1])


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("nshard", [2, 4])
def test_sequence_shards_stitch_bitwise(P, dtype, nshard):
    """carry_out -> carry_in forward and mu_out -> mu_in backward reproduce the
    single-device result bit for bit (the SP halo contract)."""
    B, L, H, D = 2, 1024, 4, 128
    g = cuda(swr_inputs(B, L, H, D, dtype=dtype, seed=7))
    x = P.swr_fwd(g["u"], g["a"])
    du, da, _ = P.swr_bwd(g["u"], g["a"], g["G"])
    S = L // nshard
    sh = [slice(p * S, (p + 1) * S) for p in range(nshard)]
    parts = {k: [g[k][:, s].contiguous() for s in sh] for k in ("u", "a", "G")}
    carries, xs = [None], []
    for p in range(nshard):
        xp, co = P.swr_fwd(parts["u"][p], parts["a"][p], carry_in=carries[-1], return_carry=True)
        xs.append(xp)
        carries.append(co)
    assert torch.equal(torch.cat(xs, dim=1), x)
    mu = None
    dus, das = [None] * nshard, [None] * nshard
    for p in reversed(range(nshard)):
        dus[p], das[p], mu = P.swr_bwd(parts["u"][p], parts["a"][p], parts["G"][p],
                                       carry_in=carries[p], mu_in=mu)
    assert torch.equal(torch.cat(dus, dim=1), du)
    assert torch.equal(torch.cat(das, dim=1), da)


def test_weighted_split_is_bitwise_invariant(P):
    """Large enough for one CTA per SM: the tensor-core kernels then size each SM's
    range from the per-SM rates measured on earlier launches, so the split changes
    from launch to launch while the table converges.  Every launch must produce the
    same bits (blocks are computed identically whichever CTA owns them)."""
    g = cuda(swr_inputs(4, 2048, 16, 128, dtype=torch.bfloat16, seed=11))
    m = cuda(mix_inputs(2, 2048, 16, 128, dtype=torch.bfloat16, seed=12))
    ref = None
    for _ in range(8):
        out = (P.swr_fwd(g["u"], g["a"]),) + tuple(P.swr_bwd(g["u"], g["a"], g["G"])[:2]) + \
              (P.phalanx_mix(m["q"], m["k"], m["v"], m["a"]),) + \
              tuple(P.phalanx_mix_bwd(m["q"], m["k"], m["v"], m["a"], m["dy"])[:4])
        if ref is None:
            ref = out
        else:
            for p_, q_ in zip(ref, out):
                assert torch.equal(p_, q_)
