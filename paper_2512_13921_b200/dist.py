"""Multi-GPU partitioning of the SWR hot path (one process per GPU).

Two modes:

* batch x head sharding -- ``shard_range``: every (b, h) line is independent
  (heads never mix inside the recurrence; batch rows are independent), so
  each rank takes a contiguous slice and runs the single-GPU kernels unchanged.
  No collective on the data path.

* sequence parallel (SP) -- ``swr_sp_fwd`` / ``swr_sp_bwd``: the sequence is cut
  into contiguous per-rank shards whose lengths are multiples of 16 (blocks stay
  aligned to token 0, R1).  Because each block sees only its own and
  its predecessor's inputs, the only exchange is one carrier vector per
  (b, h) and direction -- the segment checkpoint of P:1526:
      forward : rank p -> p+1  carry_out (local end state of p's last block, v_b)
      backward: rank p+1 -> p  mu_out    (a[first] * lambda[block 0][0])
  Each halo value is computed by a one-block prologue call on the rank's own
  inputs, sent with point-to-point send/recv (NCCL over NVLink on GPUs), and the
  main call then runs with carry_in / mu_in.  Results are bitwise identical to
  the single-GPU run (tests/test_props.py, tests/test_dist_cpu.py).

``ops`` defaults to the CUDA binding (paper_2512_13921_b200.ops), whose carriers
are fp32; tests may pass another implementation with the same signatures
(swr_fwd, swr_bwd) and its carrier dtype to exercise the exchange logic on CPU
processes with the gloo backend.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

ELL = 16


def shard_range(n: int, world: int, rank: int):
    """Contiguous [lo, hi) slice of n units for `rank` (balanced, deterministic)."""
    return (n * rank) // world, (n * (rank + 1)) // world


def sp_shard_lengths(L: int, world: int):
    """Per-rank token counts for SP: multiples of 16 except possibly the last."""
    nb = (L + ELL - 1) // ELL
    lens = []
    for r in range(world):
        b0, b1 = shard_range(nb, world, r)
        lens.append(min(b1 * ELL, L) - min(b0 * ELL, L))
    return lens


def _default_ops():
    from . import ops
    return ops


def _exchange(send_t, to_rank, recv_like, from_rank, group):
    """Point-to-point halo exchange; returns the received tensor (or None)."""
    backend = dist.get_backend(group)
    cpu = backend == "gloo"
    reqs, recv = [], None
    if recv_like is not None:
        recv = torch.empty_like(recv_like, device="cpu" if cpu else recv_like.device)
    ops = []
    if send_t is not None:
        s = send_t.contiguous().cpu() if cpu else send_t.contiguous()
        ops.append(dist.P2POp(dist.isend, s, to_rank, group))
    if recv is not None:
        ops.append(dist.P2POp(dist.irecv, recv, from_rank, group))
    if ops:
        reqs = dist.batch_isend_irecv(ops)
        for r in reqs:
            r.wait()
    if recv is not None and recv_like is not None and recv.device != recv_like.device:
        recv = recv.to(recv_like.device)
    return recv


def swr_sp_fwd(u, a, group=None, carry_in=None, ops=None, carry_dtype=torch.float32):
    """Forward SWR of this rank's sequence shard.

    u: [B, Ls, H, D] shard, a: [B, Ls, H]; every shard but the last has Ls % 16 == 0.
    carry_in: only used on rank 0 (the sequence's initial carrier).
    Returns (x, carry_in_used) -- keep carry_in_used for swr_sp_bwd.
    """
    ops = ops or _default_ops()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if rank < world - 1 and u.shape[1] % ELL:
        raise ValueError("every SP shard except the last must be a multiple of 16 tokens")
    # prologue: carrier of this shard's last block (one block of local inputs)
    send = None
    if rank < world - 1:
        nb = u.shape[1] // ELL
        lo = (nb - 1) * ELL
        _, send = ops.swr_fwd(u[:, lo:], a[:, lo:], return_carry=True)
    B, _, H, D = u.shape
    like = torch.empty((B, H, D), dtype=carry_dtype, device=u.device) if rank > 0 else None
    recv = _exchange(send, rank + 1, like, rank - 1, group)
    cin = recv if rank > 0 else carry_in
    x = ops.swr_fwd(u, a, carry_in=cin)
    return x, cin


def swr_sp_bwd(u, a, dx, carry_in=None, group=None, ops=None, carry_dtype=torch.float32):
    """Backward SWR of this rank's shard; carry_in as returned by swr_sp_fwd.

    Returns (du, da, mu_out) where mu_out is the gradient of the sequence's
    initial carrier (meaningful on rank 0)."""
    ops = ops or _default_ops()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    # prologue: mu_out of this shard's first block = a[0] * lambda_0[0] (local)
    send = None
    if rank > 0:
        n0 = min(ELL, u.shape[1])
        _, _, send = ops.swr_bwd(u[:, :n0], a[:, :n0], dx[:, :n0], carry_in=None)
    B, _, H, D = u.shape
    like = torch.empty((B, H, D), dtype=carry_dtype, device=u.device) if rank < world - 1 else None
    mu_in = _exchange(send, rank - 1, like, rank + 1, group)
    du, da, mu_out = ops.swr_bwd(u, a, dx, carry_in=carry_in, mu_in=mu_in)
    return du, da, mu_out
