"""CPU (gloo, world_size 2) tests of the multi-GPU launcher's host logic: the (b·h, query-tile) unit split
covers every unit exactly once with balanced KV-tile cost, and the final gather reassembles O in order.  The
per-shard compute is a host stub here (a per-head function of the inputs); the CUDA path is exercised by the
GPU tests and bench."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_11594_b200.multigpu import (forward_sharded, local_heads, shard_ranges, shard_units, tiles_per_head,
                                            unit_cost, unit_rows)


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


@pytest.mark.parametrize("B,H,N,causal,world", [(2, 30, 17776, False, 8), (1, 24, 118800, False, 8),
                                                 (8, 32, 32768, True, 8), (1, 3, 300, True, 2), (2, 30, 17776, True, 8),
                                                 (1, 1, 128, True, 4), (1, 5, 1000, True, 3)])
def test_shard_units_cover_and_balance(B, H, N, causal, world):
    T = tiles_per_head(N)
    rs = shard_units(B, H, N, causal, world)
    assert rs[0][0] == 0 and rs[-1][1] == B * H * T and all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    costs = [sum(unit_cost(u, T, causal) for u in range(s, e)) for s, e in rs]
    # a contiguous split is within one unit's cost (<= T KV tiles) of the ideal share
    assert max(costs) - sum(costs) / world <= T
    if not causal:
        assert max(e - s for s, e in rs) - min(e - s for s, e in rs) <= 1
    # C3 on 8 GPUs: 60 heads x 139 tiles -> 1043/1042 units (vs 8/7 whole heads)
    if (B, H, N, causal, world) == (2, 30, 17776, False, 8):
        assert [e - s for s, e in rs] == [1043] * 4 + [1042] * 4


def test_unit_rows_numbering():
    # unit u of a head is query tile T-1-u%T (longest first under causal masking); the last tile is ragged
    T = tiles_per_head(300)
    assert T == 3
    assert unit_rows(0, T, 300) == (0, 256, 300) and unit_rows(2, T, 300) == (0, 0, 128)
    assert unit_rows(4, T, 300) == (1, 128, 256)


def stub(q, k, v, causal, scale, unit_lo=None, unit_hi=None):
    # a per-head deterministic function standing in for the attention kernel (valid on every row)
    return v * 2.0 + q.sum(-1, keepdim=True) * (0.5 if causal else 1.0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, H, N, causal, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(0)
    q = torch.randn(B, H, N, 8, generator=g)
    k = torch.randn(B, H, N, 8, generator=g)
    v = torch.randn(B, H, N, 8, generator=g)
    out = forward_sharded(q, k, v, causal=causal, compute=stub)
    if rank == 0:
        ret["ok"] = bool(torch.equal(out, stub(q, k, v, causal, 0.0)))
        ret["shape"] = tuple(out.shape)
    else:
        ret[f"local{rank}"] = tuple(out.shape)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B,H,N,causal", [(1, 4, 16, True), (1, 3, 300, True), (2, 3, 200, False), (1, 1, 384, True)])
def test_forward_sharded_gather_world2(B, H, N, causal):
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), B, H, N, causal, ret), nprocs=2, join=True)
    assert ret["ok"] and ret["shape"] == (B, H, N, 8)
    s, e = shard_units(B, H, N, causal, 2)[1]
    assert ret["local1"][0] == e - s


@pytest.mark.parametrize("nprocs,shape,causal,mu", [(2, "1,5,300,16", False, 0), (3, "2,3,700,8", True, 7),
                                                    (2, "1,1,128,8", True, 0)])
def test_self_launch_pipelined_gather_gloo(nprocs, shape, causal, mu):
    """The launcher end to end on CPU: self_launch re-executes under torch.distributed.run (127.0.0.1, gloo),
    every rank computes its ShardPlan units head by head (host stub for the kernel) and sends each finished
    head's rows to rank 0 (isend/irecv pipelined gather), which reassembles O exactly."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, os.path.join(root, "tools", "mg_selftest.py"), "--nprocs", str(nprocs), "--stub",
           "--shape", shape, "--min-units", str(mu)] + (["--causal"] if causal else [])
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=dict(os.environ, OMP_NUM_THREADS="1"))
    line = [x for x in p.stdout.splitlines() if x.startswith("MG_SELFTEST")]
    assert line and line[0].startswith(f"MG_SELFTEST OK world={nprocs}"), p.stdout[-2000:] + p.stderr[-2000:]


def test_shard_plan_head_chunks():
    from paper_2505_11594_b200.multigpu import ShardPlan

    # C4 strong scaling: 24 heads over 8 GPUs -> 3 whole heads per rank
    p = ShardPlan(1, 24, 118800, False, 8, 3)
    assert (p.h0, p.h1) == (9, 12) and [c[0] for c in p.head_chunks()] == [9, 10, 11]
    assert all(n == 1 and lo == 0 and hi == 929 for _, n, lo, hi in p.head_chunks())
    assert list(p.head_chunks(1500)) == [(9, 2, 0, 1858), (11, 1, 0, 929)]
    # C3 on 8 GPUs: a rank's range can start and end inside heads
    T = tiles_per_head(17776)
    for r in range(8):
        p = ShardPlan(2, 30, 17776, False, 8, r)
        for mu in (0, 200, 10 ** 9):
            ch = list(p.head_chunks(mu))
            assert sum(hi - lo for _, _, lo, hi in ch) == p.u1 - p.u0
            assert all(0 <= lo < hi <= n * T for _, n, lo, hi in ch)
            assert ch[0][0] == p.h0 and sum(n for _, n, _, _ in ch) == p.h1 - p.h0
