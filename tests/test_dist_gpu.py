"""Sequence-parallel halo path on the GPU kernels: 2 and 4 ranks share cuda:0 (the
gpurun box has one GPU), the tiny carrier halos go through gloo; the stitched
outputs must equal the single-GPU call bit for bit (SURVEY pin P8)."""
import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, L, outdir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_13921_b200 import dist as sdist
    from swr_inputs import swr_inputs
    inp = swr_inputs(2, L, 16, 128, dtype=torch.bfloat16, seed=21)
    lens = sdist.sp_shard_lengths(L, world)
    lo = sum(lens[:rank])
    hi = lo + lens[rank]
    u, a, G = (inp[k][:, lo:hi].contiguous().cuda() for k in ("u", "a", "G"))
    x, cin = sdist.swr_sp_fwd(u, a)
    du, da, mo = sdist.swr_sp_bwd(u, a, G, carry_in=cin)
    torch.cuda.synchronize()
    torch.save({"x": x.cpu(), "du": du.cpu(), "da": da.cpu(), "mo": mo.cpu()},
               os.path.join(outdir, f"g{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,L", [(2, 512), (4, 1024), (3, 100), (2, 33)])
def test_sp_on_gpu_kernels_is_bitwise(tmp_path, world, L):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from conftest import build_lib
    build_lib()
    import paper_2512_13921_b200 as P
    from swr_inputs import swr_inputs
    mp.spawn(_worker, args=(world, _free_port(), L, str(tmp_path)), nprocs=world, join=True)
    inp = swr_inputs(2, L, 16, 128, dtype=torch.bfloat16, seed=21)
    g = {k: v.cuda() for k, v in inp.items()}
    x = P.swr_fwd(g["u"], g["a"]).cpu()
    du, da, mo = (t.cpu() for t in P.swr_bwd(g["u"], g["a"], g["G"]))
    parts = [torch.load(tmp_path / f"g{r}.pt") for r in range(world)]
    assert torch.equal(torch.cat([p["x"] for p in parts], dim=1), x)
    assert torch.equal(torch.cat([p["du"] for p in parts], dim=1), du)
    assert torch.equal(torch.cat([p["da"] for p in parts], dim=1), da)
    assert torch.equal(parts[0]["mo"], mo)
