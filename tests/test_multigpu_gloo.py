"""CPU (gloo, world_size 2) tests of the multi-GPU launcher's host logic: head sharding covers every (b, h)
exactly once with balanced shards, and the final gather reassembles O in order.  The per-shard compute is a
host stub here (a per-head function of the inputs); the CUDA path is exercised by the GPU tests and bench."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_11594_b200.multigpu import forward_sharded, local_heads, shard_ranges


def test_shard_ranges_cover_and_balance():
    for n in (0, 1, 7, 60, 256):
        for w in (1, 2, 3, 8):
            rs = shard_ranges(n, w)
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [e - s for s, e in rs]
            assert max(sizes) - min(sizes) <= 1
    # C3 (CogVideoX-shaped): 60 heads over 8 GPUs -> 8,8,8,8,7,7,7,7
    assert [e - s for s, e in shard_ranges(60, 8)] == [8, 8, 8, 8, 7, 7, 7, 7]
    assert list(local_heads(2, 30, 8, 7)) == list(range(53, 60))


def stub(q, k, v, causal, scale):
    # a per-head deterministic function standing in for the attention kernel
    return v * 2.0 + q.sum(-1, keepdim=True) * (0.5 if causal else 1.0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, H, causal, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(0)
    q = torch.randn(B, H, 16, 8, generator=g)
    k = torch.randn(B, H, 16, 8, generator=g)
    v = torch.randn(B, H, 16, 8, generator=g)
    out = forward_sharded(q, k, v, causal=causal, compute=stub)
    if rank == 0:
        ret["ok"] = bool(torch.equal(out, stub(q, k, v, causal, 0.0)))
        ret["shape"] = tuple(out.shape)
    else:
        ret[f"local{rank}"] = tuple(out.shape)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B,H", [(1, 4), (1, 3), (2, 3)])
def test_forward_sharded_gather_world2(B, H):
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), B, H, True, ret), nprocs=2, join=True)
    assert ret["ok"] and ret["shape"] == (B, H, 16, 8)
    assert ret["local1"][0] == len(local_heads(B, H, 2, 1))
