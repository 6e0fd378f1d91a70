"""Multi-GPU launcher for the SageAttention3 forward: one process per GPU (torch.distributed), the flattened
(b, h) heads split into contiguous balanced shards, no data exchange on the hot path, one final gather.

Why no collective: smoothing K (Alg1 L2), φ and the whole Algorithm 1 loop are per
(b, h) head — every head is an independent problem — so each rank quantizes and attends its own heads
and the only communication is collecting O at the end (off the hot path; NCCL gather over NVLink).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_ranges(n_units: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced [start, end) split of n_units over world ranks (sizes differ by at most 1)."""
    if world < 1 or n_units < 0:
        raise ValueError("world must be >= 1 and n_units >= 0")
    base, extra = divmod(n_units, world)
    out, s = [], 0
    for r in range(world):
        e = s + base + (1 if r < extra else 0)
        out.append((s, e))
        s = e
    return out


def local_heads(B: int, H: int, world: int, rank: int) -> range:
    """Flattened head ids (b*H + h) owned by `rank`."""
    s, e = shard_ranges(B * H, world)[rank]
    return range(s, e)


def _default_compute(q, k, v, causal, softmax_scale):
    import paper_2505_11594_b200 as s3

    return s3.attention(q, k, v, causal=causal, softmax_scale=softmax_scale)


def forward_sharded(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, causal: bool = False,
                    softmax_scale: float = 0.0, group=None, gather_to: int = 0, compute=None):
    """Run the FP4 attention forward on this rank's heads and gather O on rank `gather_to`.

    q, k, v: the full [B, H, N, d] inputs (as every rank sees them; only this rank's heads are read).
    Returns the full O on `gather_to` and this rank's [n_local, N, d] slice of O elsewhere.
    `compute(q, k, v, causal, softmax_scale)` maps [1, n_local, N, d] inputs to O; it defaults to the CUDA
    path (quantize + attention through the C ABI).  Tests substitute a host stub to exercise the sharding
    and gather logic without a GPU.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    B, H, N, d = q.shape
    heads = local_heads(B, H, world, rank)
    fn = compute or _default_compute
    flat = lambda x: x.reshape(B * H, N, d)
    sl = slice(heads.start, heads.stop)
    if len(heads):
        o_local = fn(flat(q)[sl].unsqueeze(0), flat(k)[sl].unsqueeze(0), flat(v)[sl].unsqueeze(0), causal,
                     softmax_scale)[0]
    else:
        o_local = q.new_empty(0, N, d)
    if world == 1:
        return o_local.reshape(B, H, N, d)
    # equal-size gather: pad every shard to the largest one
    ranges = shard_ranges(B * H, world)
    cap = max(e - s for s, e in ranges)
    buf = o_local.new_zeros(cap, N, d)
    buf[: o_local.shape[0]] = o_local
    if rank == gather_to:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, parts, dst=gather_to, group=group)
        out = torch.cat([p[: e - s] for p, (s, e) in zip(parts, ranges)])
        return out.reshape(B, H, N, d)
    dist.gather(buf, None, dst=gather_to, group=group)
    return o_local
