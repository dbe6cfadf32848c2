"""Multi-process tests of the partitioning logic (paper_2512_13921_b200/dist.py)
on CPU processes with the gloo backend, world_size 2 and 4.

The halo exchange (carry_out -> carry_in forward, mu_out -> mu_in backward) and
the shard bookkeeping are the host logic under test; the per-shard compute is
injected as the fp64 oracle (test infrastructure), so stitched results must
equal the single-run oracle bit for bit (SURVEY pin P8)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleOps:
    """swr_fwd / swr_bwd with the binding's signatures, computed by the fp64 oracle."""

    @staticmethod
    def swr_fwd(u, a, carry_in=None, return_carry=False):
        import oracle
        ci = None if carry_in is None else carry_in.double().numpy()
        r = oracle.swr_fwd(u.numpy(), a.numpy(), carry_in=ci, carry_out=return_carry)
        if return_carry:
            return torch.from_numpy(r[0]), torch.from_numpy(r[1])
        return torch.from_numpy(r)

    @staticmethod
    def swr_bwd(u, a, dx, carry_in=None, mu_in=None):
        import oracle
        ci = None if carry_in is None else carry_in.double().numpy()
        mi = None if mu_in is None else mu_in.double().numpy()
        du, da, mo = oracle.swr_bwd(u.numpy(), a.numpy(), dx.numpy(), carry_in=ci, mu_in=mi)
        return torch.from_numpy(du), torch.from_numpy(da), torch.from_numpy(mo)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(B, L, H, D, seed):
    g = torch.Generator().manual_seed(seed)
    u = torch.randn(B, L, H, D, generator=g, dtype=torch.float64)
    a = torch.rand(B, L, H, generator=g, dtype=torch.float64)
    G = torch.randn(B, L, H, D, generator=g, dtype=torch.float64)
    return u, a, G


def _sp_worker(rank, world, port, L, outdir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_13921_b200 import dist as sdist
    B, H, D = 2, 3, 4
    u, a, G = _problem(B, L, H, D, seed=5)
    lens = sdist.sp_shard_lengths(L, world)
    lo = sum(lens[:rank])
    hi = lo + lens[rank]
    us, as_, Gs = u[:, lo:hi].contiguous(), a[:, lo:hi].contiguous(), G[:, lo:hi].contiguous()
    x, cin = sdist.swr_sp_fwd(us, as_, ops=OracleOps, carry_dtype=torch.float64)
    du, da, mo = sdist.swr_sp_bwd(us, as_, Gs, carry_in=cin, ops=OracleOps, carry_dtype=torch.float64)
    torch.save({"x": x, "du": du, "da": da, "mo": mo, "lo": lo, "hi": hi,
                "cin": cin}, os.path.join(outdir, f"r{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,L", [(2, 64), (2, 70), (4, 160), (4, 77), (3, 40)])
def test_sequence_parallel_stitching_gloo(tmp_path, world, L):
    import oracle
    mp.spawn(_sp_worker, args=(world, _free_port(), L, str(tmp_path)), nprocs=world, join=True)
    u, a, G = _problem(2, L, 3, 4, seed=5)
    rx = oracle.swr_fwd(u.numpy(), a.numpy())
    rdu, rda, rmo = oracle.swr_bwd(u.numpy(), a.numpy(), G.numpy())
    parts = [torch.load(tmp_path / f"r{r}.pt") for r in range(world)]
    x = torch.cat([p["x"] for p in parts], dim=1).numpy()
    du = torch.cat([p["du"] for p in parts], dim=1).numpy()
    da = torch.cat([p["da"] for p in parts], dim=1).numpy()
    assert np.array_equal(x, rx)
    assert np.array_equal(du, rdu)
    assert np.array_equal(da, rda)
    assert np.array_equal(parts[0]["mo"].numpy(), rmo)
    # the halo really travelled: rank r>0 received rank r-1's carrier
    for r in range(1, world):
        assert parts[r]["cin"] is not None and torch.count_nonzero(parts[r]["cin"]) > 0
    assert parts[0]["cin"] is None


def _shard_worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_13921_b200 import dist as sdist
    B, L, H, D = 5, 48, 2, 4
    u, a, G = _problem(B, L, H, D, seed=9)
    b0, b1 = sdist.shard_range(B, world, rank)
    x = OracleOps.swr_fwd(u[b0:b1].contiguous(), a[b0:b1].contiguous())
    du, da, _ = OracleOps.swr_bwd(u[b0:b1].contiguous(), a[b0:b1].contiguous(), G[b0:b1].contiguous())
    torch.save({"x": x, "du": du, "da": da, "b0": b0, "b1": b1}, os.path.join(outdir, f"s{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def test_batch_sharding_gloo(tmp_path):
    """Batch x head sharding: no collective on the data path; the union of the
    rank slices equals the single run bit for bit and covers every row once."""
    import oracle
    world = 2
    mp.spawn(_shard_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    u, a, G = _problem(5, 48, 2, 4, seed=9)
    parts = [torch.load(tmp_path / f"s{r}.pt") for r in range(world)]
    assert [(p["b0"], p["b1"]) for p in parts] == [(0, 2), (2, 5)]
    x = torch.cat([p["x"] for p in parts]).numpy()
    du = torch.cat([p["du"] for p in parts]).numpy()
    assert np.array_equal(x, oracle.swr_fwd(u.numpy(), a.numpy()))
    assert np.array_equal(du, oracle.swr_bwd(u.numpy(), a.numpy(), G.numpy())[0])


def test_sp_shard_lengths():
    from paper_2512_13921_b200 import dist as sdist
    assert sdist.sp_shard_lengths(131072, 8) == [16384] * 8
    assert sdist.sp_shard_lengths(77, 4) == [16, 16, 16, 29]
    assert sum(sdist.sp_shard_lengths(1000, 3)) == 1000
    for lens in (sdist.sp_shard_lengths(1000, 3), sdist.sp_shard_lengths(70, 2)):
        assert all(n % 16 == 0 for n in lens[:-1])


def _subgroup_worker(rank, world, port, L, outdir):
    """SP inside sub-groups {0,1} and {2,3} of a world-4 job (sequence parallel
    inside data parallel): halo peers are group ranks, P2POp needs global ones."""
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_13921_b200 import dist as sdist
    groups = [dist.new_group([0, 1]), dist.new_group([2, 3])]
    grp = groups[rank // 2]
    grank = dist.get_rank(grp)
    u, a, G = _problem(2, L, 3, 4, seed=40 + rank // 2)  # one problem per sub-group
    lens = sdist.sp_shard_lengths(L, 2)
    lo = sum(lens[:grank])
    hi = lo + lens[grank]
    us, as_, Gs = u[:, lo:hi].contiguous(), a[:, lo:hi].contiguous(), G[:, lo:hi].contiguous()
    x, cin = sdist.swr_sp_fwd(us, as_, group=grp, ops=OracleOps, carry_dtype=torch.float64)
    du, da, mo = sdist.swr_sp_bwd(us, as_, Gs, carry_in=cin, group=grp, ops=OracleOps,
                                  carry_dtype=torch.float64)
    torch.save({"x": x, "du": du, "da": da, "mo": mo}, os.path.join(outdir, f"g{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def test_sequence_parallel_in_subgroups_gloo(tmp_path):
    import oracle
    L = 80
    mp.spawn(_subgroup_worker, args=(4, _free_port(), L, str(tmp_path)), nprocs=4, join=True)
    parts = [torch.load(tmp_path / f"g{r}.pt") for r in range(4)]
    for gi in range(2):
        u, a, G = _problem(2, L, 3, 4, seed=40 + gi)
        p0, p1 = parts[2 * gi], parts[2 * gi + 1]
        rx = oracle.swr_fwd(u.numpy(), a.numpy())
        rdu, rda, rmo = oracle.swr_bwd(u.numpy(), a.numpy(), G.numpy())
        assert np.array_equal(torch.cat([p0["x"], p1["x"]], dim=1).numpy(), rx)
        assert np.array_equal(torch.cat([p0["du"], p1["du"]], dim=1).numpy(), rdu)
        assert np.array_equal(torch.cat([p0["da"], p1["da"]], dim=1).numpy(), rda)
        assert np.array_equal(p0["mo"].numpy(), rmo)


def test_sp_rejects_empty_shards():
    from paper_2512_13921_b200 import dist as sdist
    with pytest.raises(ValueError):
        sdist.sp_shard_lengths(40, 4)  # 3 blocks for 4 ranks
    assert sdist.sp_shard_lengths(48, 3) == [16, 16, 16]
