"""Seeded synthetic inputs for the SWR / Phalanx-mixer hot path.

The ONE module shared by tests, bench.py, the oracle comparisons and the CUDA
path.  It holds none of the method's arithmetic: it only draws random tensors
with the distributions of the paper's layer:

* decays  a = sigmoid(N(0,1))            -- a_i = sigma(W u_i)
* key gate k = sigmoid(N(0,1))           -- k = sigma(K u)
* q, v, u, upstream gradients ~ N(0,1)   -- linear projections

Everything is generated on the CPU with a ``torch.Generator`` so both sides of a
parity check see bit-identical values, then rounded to the storage dtype.
"""
from __future__ import annotations

import torch

DECAY_KINDS = ("sigmoid", "uniform", "zero", "one", "tiny", "near_one", "sigmoid3", "bounded")


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def decays(shape, kind: str, g: torch.Generator) -> torch.Tensor:
    """Decay tensor of the requested family, fp32 on CPU."""
    if kind == "sigmoid":            # sigma(N(0,1)), the layer's parametrisation
        return torch.sigmoid(torch.randn(shape, generator=g))
    if kind == "sigmoid3":           # sigma(N(0,1)+3): long memory, most a near 1
        return torch.sigmoid(torch.randn(shape, generator=g) + 3.0)
    if kind == "uniform":            # U(0,1) with 0 excluded
        return torch.rand(shape, generator=g).clamp_min(1e-7)
    if kind == "bounded":            # (0, 0.8): the bounded-decay ablation
        return 0.8 * torch.rand(shape, generator=g).clamp_min(1e-7)
    if kind == "zero":
        return torch.zeros(shape)
    if kind == "one":
        return torch.ones(shape)
    if kind == "tiny":
        return torch.full(shape, 1e-3)
    if kind == "near_one":
        return torch.full(shape, 1.0 - 2.0 ** -8)
    raise ValueError(kind)


def swr_inputs(B, L, H, D, dtype=torch.bfloat16, seed=0, decay="sigmoid", carry=False):
    """u, a, G (and carry_in, mu_in in fp32 if carry=True) on the CPU in `dtype`."""
    g = _gen(seed)
    out = {
        "u": torch.randn((B, L, H, D), generator=g).to(dtype),
        "a": decays((B, L, H), decay, g).to(dtype),
        "G": torch.randn((B, L, H, D), generator=g).to(dtype),
    }
    if carry:
        out["carry_in"] = torch.randn((B, H, D), generator=g)
        out["mu_in"] = torch.randn((B, H, D), generator=g)
    return out


def mix_inputs(B, L, H, D, dtype=torch.bfloat16, seed=0, decay="sigmoid", carry=False):
    """q, k, v, a, dy (and carry_in, mu_in in fp32 if carry=True) on the CPU in `dtype`."""
    g = _gen(seed)
    out = {
        "q": torch.randn((B, L, H, D), generator=g).to(dtype),
        "k": torch.sigmoid(torch.randn((B, L, H, D), generator=g)).to(dtype),
        "v": torch.randn((B, L, H, D), generator=g).to(dtype),
        "a": decays((B, L, H), decay, g).to(dtype),
        "dy": torch.randn((B, L, H, D), generator=g).to(dtype),
    }
    if carry:
        out["carry_in"] = torch.randn((B, H, D), generator=g)
        out["mu_in"] = torch.randn((B, H, D), generator=g)
    return out


def layer_inputs(B, L, H, D, Gq=None, Gk=None, dtype=torch.bfloat16, seed=0, carry=False, za_shift=0.0):
    """Inputs of the Phalanx layer mixer (NEXT-1), as the featurization produces them:
    logits za ~ N(0,1) + za_shift [B, L, H] (a = sigma(za)) and zk ~ N(0,1)
    [B, L, Gk, D] (k = sigma(zk)); q ~ N(0,1) [B, L, Gq, D], v, dy ~
    N(0,1) [B, L, H, D].  Gq = Gk = H (no sharing) by default."""
    Gq = H if Gq is None else Gq
    Gk = H if Gk is None else Gk
    g = _gen(seed)
    out = {
        "q": torch.randn((B, L, Gq, D), generator=g).to(dtype),
        "zk": torch.randn((B, L, Gk, D), generator=g).to(dtype),
        "v": torch.randn((B, L, H, D), generator=g).to(dtype),
        "za": (torch.randn((B, L, H), generator=g) + za_shift).to(dtype),
        "dy": torch.randn((B, L, H, D), generator=g).to(dtype),
    }
    if carry:
        out["carry_in"] = torch.randn((B, H, D), generator=g)
        out["mu_in"] = torch.randn((B, H, D), generator=g)
    return out


def to64(t):
    """Upcast an (already rounded) tensor to a float64 numpy array for the oracle."""
    return None if t is None else t.detach().to("cpu", torch.float64).numpy()
