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
  inputs and sent with point-to-point send/recv (NCCL over NVLink on GPUs).  The
  exchange overlaps the interior: the main call runs without the incoming halo
  while the send/recv is in flight (NCCL's own stream), then only the block that
  needs it is recomputed with it -- the shard's first block (forward, with
  carry_in) or its last block (backward, with mu_in, from a two-block slice so its
  predecessor's carrier is recomputed too) -- and copied over.  Blocks are computed
  identically whichever call computes them, so results are bitwise identical to
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
    """Per-rank token counts for SP: multiples of 16 except possibly the last.

    Every rank gets at least one block: an empty shard would have no block to
    carry the halo through (its neighbours would receive zeros instead of the
    predecessor's carrier), so world > ceil(L / 16) is rejected."""
    nb = (L + ELL - 1) // ELL
    if world > nb:
        raise ValueError(f"sequence parallelism needs at least one 16-token block per rank: "
                         f"L={L} has {nb} blocks for {world} ranks")
    lens = []
    for r in range(world):
        b0, b1 = shard_range(nb, world, r)
        lens.append(min(b1 * ELL, L) - min(b0 * ELL, L))
    return lens


def _default_ops():
    from . import ops
    return ops


def _global(group, r):
    """Global rank of group rank r (P2POp's `peer` is a rank of the default group)."""
    return r if group is None else dist.get_global_rank(group, r)


def _start_exchange(send_t, to_rank, recv_like, from_rank, group):
    """Post the point-to-point halo exchange; returns (requests, receive buffer).
    to_rank / from_rank are ranks inside `group`."""
    cpu = dist.get_backend(group) == "gloo"
    recv = None
    if recv_like is not None:
        recv = torch.empty_like(recv_like, device="cpu" if cpu else recv_like.device)
    ops = []
    if send_t is not None:
        s = send_t.contiguous().cpu() if cpu else send_t.contiguous()
        ops.append(dist.P2POp(dist.isend, s, _global(group, to_rank), group))
    if recv is not None:
        ops.append(dist.P2POp(dist.irecv, recv, _global(group, from_rank), group))
    reqs = dist.batch_isend_irecv(ops) if ops else []
    return reqs, recv


def _finish_exchange(reqs, recv, recv_like):
    """Complete the exchange (NCCL: the current stream waits for it, no host block)."""
    for r in reqs:
        r.wait()
    if recv is not None and recv.device != recv_like.device:
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
    if u.shape[1] == 0:
        raise ValueError("empty SP shard: every rank needs at least one block (sp_shard_lengths)")
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
    reqs, recv = _start_exchange(send, rank + 1, like, rank - 1, group)
    if rank == 0:
        x = ops.swr_fwd(u, a, carry_in=carry_in)
        _finish_exchange(reqs, recv, like)
        return x, carry_in
    # interior while the halo is in flight (block 0 gets v_{-1} = 0 here) ...
    x = ops.swr_fwd(u, a)
    cin = _finish_exchange(reqs, recv, like)
    # ... then block 0 again with the received carrier
    n0 = min(ELL, u.shape[1])
    x[:, :n0] = ops.swr_fwd(u[:, :n0], a[:, :n0], carry_in=cin)
    return x, cin


def swr_sp_bwd(u, a, dx, carry_in=None, group=None, ops=None, carry_dtype=torch.float32):
    """Backward SWR of this rank's shard; carry_in as returned by swr_sp_fwd.

    Returns (du, da, mu_out) where mu_out is the gradient of the sequence's
    initial carrier (meaningful on rank 0)."""
    ops = ops or _default_ops()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if u.shape[1] == 0:
        raise ValueError("empty SP shard: every rank needs at least one block (sp_shard_lengths)")
    # prologue: mu_out of this shard's first block = a[0] * lambda_0[0] (local)
    send = None
    if rank > 0:
        n0 = min(ELL, u.shape[1])
        _, _, send = ops.swr_bwd(u[:, :n0], a[:, :n0], dx[:, :n0], carry_in=None)
    B, Ls, H, D = u.shape
    like = torch.empty((B, H, D), dtype=carry_dtype, device=u.device) if rank < world - 1 else None
    reqs, recv = _start_exchange(send, rank - 1, like, rank + 1, group)
    # interior while the halo is in flight (the last block gets mu = 0 here) ...
    du, da, mu_out = ops.swr_bwd(u, a, dx, carry_in=carry_in)
    mu_in = _finish_exchange(reqs, recv, like)
    if mu_in is not None:
        # ... then the last block again with mu_in; its carrier comes from the
        # block before it, so the slice starts one block earlier (or at 0 with
        # carry_in), and only the last block is copied back
        nb = (Ls + ELL - 1) // ELL
        lo = (nb - 1) * ELL
        s0 = max(lo - ELL, 0)
        cin = carry_in if s0 == 0 else None
        dus, das, mos = ops.swr_bwd(u[:, s0:], a[:, s0:], dx[:, s0:], carry_in=cin, mu_in=mu_in)
        du[:, lo:] = dus[:, lo - s0:]
        da[:, lo:] = das[:, lo - s0:]
        if nb == 1:
            mu_out = mos  # a one-block shard: its first block is its last
    return du, da, mu_out
