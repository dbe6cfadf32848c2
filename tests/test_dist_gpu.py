"""Sequence-parallel halo path (paper_2512_13921_b200/dist.py) on the GPU kernels.

* gloo on one GPU: 2-4 ranks share cuda:0 (a gpurun box has one GPU) and the
  carrier halos go through gloo.  The stitched shard outputs are compared with the
  fp64 oracle on the whole sequence (the jagged operator; the carrier
  checkpoint between segments) and with the single-GPU call bit for bit
  (SURVEY pin P8).
* NCCL: one rank per GPU when the box has >= 2 GPUs (skipped otherwise) -- the
  exchange bench.py --config sp131k uses under torchrun.
* overlap: the interior call is issued before the halo wait and runs while the
  halo is in flight (a delayed sender; the interior's CUDA event has completed
  by the time the receive returns).
"""
import os
import socket
import sys
import time

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 2e-2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port, backend):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if backend == "nccl":
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", rank))
    else:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker(rank, world, port, L, outdir, backend):
    _init(rank, world, port, backend)
    from paper_2512_13921_b200 import dist as sdist
    from swr_inputs import swr_inputs
    inp = swr_inputs(2, L, 16, 128, dtype=torch.bfloat16, seed=21)
    lens = sdist.sp_shard_lengths(L, world)
    lo = sum(lens[:rank])
    hi = lo + lens[rank]
    dev = torch.device("cuda", torch.cuda.current_device())
    u, a, G = (inp[k][:, lo:hi].contiguous().to(dev) for k in ("u", "a", "G"))
    x, cin = sdist.swr_sp_fwd(u, a)
    du, da, mo = sdist.swr_sp_bwd(u, a, G, carry_in=cin)
    torch.cuda.synchronize()
    torch.save({"x": x.cpu(), "du": du.cpu(), "da": da.cpu(), "mo": mo.cpu()},
               os.path.join(outdir, f"g{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def _check_stitched(tmp_path, world, L):
    import oracle
    import paper_2512_13921_b200 as P
    from swr_inputs import swr_inputs, to64
    inp = swr_inputs(2, L, 16, 128, dtype=torch.bfloat16, seed=21)
    parts = [torch.load(tmp_path / f"g{r}.pt") for r in range(world)]
    x = torch.cat([p["x"] for p in parts], dim=1)
    du = torch.cat([p["du"] for p in parts], dim=1)
    da = torch.cat([p["da"] for p in parts], dim=1)
    mo = parts[0]["mo"]
    # against the oracle on the whole sequence
    u, a, G = to64(inp["u"]), to64(inp["a"]), to64(inp["G"])
    rx = oracle.swr_fwd(u, a)
    rdu, rda, rmo = oracle.swr_bwd(u, a, G)
    for name, t, ref in (("x", x, rx), ("du", du, rdu), ("da", da, rda), ("mu_out", mo, rmo)):
        t64 = t.double().numpy()
        e = np.max(np.abs(t64 - ref)) / np.max(np.abs(ref))
        assert e <= TOL, f"{name}: normwise {e:.3e}"
    # and bit for bit against one call on the whole sequence (pin P8)
    g = {k: v.cuda() for k, v in inp.items()}
    assert torch.equal(x, P.swr_fwd(g["u"], g["a"]).cpu())
    sdu, sda, smo = (t.cpu() for t in P.swr_bwd(g["u"], g["a"], g["G"]))
    assert torch.equal(du, sdu)
    assert torch.equal(da, sda)
    assert torch.equal(mo, smo)


@pytest.mark.parametrize("world,L", [(2, 512), (4, 1024), (3, 100), (2, 33)])
def test_sp_gloo_on_gpu_kernels(tmp_path, world, L):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from conftest import build_lib
    build_lib()
    mp.spawn(_worker, args=(world, _free_port(), L, str(tmp_path), "gloo"), nprocs=world, join=True)
    _check_stitched(tmp_path, world, L)


@pytest.mark.parametrize("L", [1024, 1000])
def test_sp_nccl(tmp_path, L):
    """NCCL send/recv between GPUs (needs >= 2 GPUs; gpurun boxes have one)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs for the NCCL halo")
    from conftest import build_lib
    build_lib()
    world = min(torch.cuda.device_count(), 4)
    mp.spawn(_worker, args=(world, _free_port(), L, str(tmp_path), "nccl"), nprocs=world, join=True)
    _check_stitched(tmp_path, world, L)


def _overlap_worker(rank, world, port, outdir):
    _init(rank, world, port, "gloo")
    from paper_2512_13921_b200 import dist as sdist
    from paper_2512_13921_b200 import ops
    from swr_inputs import swr_inputs
    inp = swr_inputs(2, 2048, 16, 128, dtype=torch.bfloat16, seed=5)
    lens = sdist.sp_shard_lengths(2048, world)
    lo = sum(lens[:rank])
    u, a = (inp[k][:, lo:lo + lens[rank]].contiguous().cuda() for k in ("u", "a"))
    calls, halo = [], {}

    class Ops:  # the CUDA ops, with a CUDA event recorded after every call
        @staticmethod
        def swr_fwd(uu, *args, **kw):
            r = ops.swr_fwd(uu, *args, **kw)
            ev = torch.cuda.Event()
            ev.record()
            calls.append((uu.shape[1], ev))
            return r

    start, finish = sdist._start_exchange, sdist._finish_exchange

    def slow_start(*args):
        if rank == 0:
            time.sleep(0.3)  # the halo leaves rank 0 late
        return start(*args)

    def watched_finish(*args):
        r = finish(*args)
        halo["issued_before"] = [n for n, _ in calls]
        halo["done"] = [ev.query() for _, ev in calls]
        return r

    sdist._start_exchange, sdist._finish_exchange = slow_start, watched_finish
    dist.barrier()
    torch.cuda.synchronize()
    sdist.swr_sp_fwd(u, a, ops=Ops)
    torch.cuda.synchronize()
    torch.save({"shard": u.shape[1], **halo}, os.path.join(outdir, f"o{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def test_sp_halo_overlaps_interior(tmp_path):
    """Rank 1's interior call (its whole shard) is issued before the halo wait and
    has finished on the GPU by the time the (delayed) halo arrives: the exchange
    overlaps the interior instead of preceding it (SURVEY 8(e) schedule)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from conftest import build_lib
    build_lib()
    mp.spawn(_overlap_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    r1 = torch.load(tmp_path / "o1.pt")
    # rank 1: the interior (its whole shard) was issued before the halo wait and had
    # completed on the GPU when the delayed halo arrived
    assert r1["issued_before"] == [r1["shard"]]
    assert r1["done"] == [True]
