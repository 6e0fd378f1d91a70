"""Multi-GPU launcher for the SageAttention3 forward: one process per GPU (torch.distributed), the work split
into contiguous cost-balanced ranges of (b·h, 128-row query tile) units, no data exchange on the hot path,
one final gather.

Why no collective: smoothing K (Alg1 L2), φ and the whole Algorithm 1 loop are per
(b, h) head — every head is an independent problem, and within a head every 128-row query tile is an
independent problem given the head's quantized K and V — so each rank quantizes the heads its units touch,
runs `sage3_attn_fwd_units` on its units, and the only communication is collecting O at the end (off the
hot path; NCCL gather over NVLink).  Unit granularity (not whole heads) keeps head counts that do not
divide the GPU count balanced (C3: 60 heads on 8 GPUs), at the price of a rank re-quantizing the K/V of at
most two heads it shares with its neighbours (memory-bound work, a few % of a head's attention time).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

TILE = 128  # query rows per unit (the kernel's B_q)


def shard_ranges(n_units: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced [start, end) split of n_units equal-cost units over world ranks (sizes differ by at
    most 1)."""
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
    """Flattened head ids (b*H + h) of a whole-head split (kept for reference; the launcher splits units)."""
    s, e = shard_ranges(B * H, world)[rank]
    return range(s, e)


def tiles_per_head(N: int) -> int:
    return (N + TILE - 1) // TILE


def unit_cost(u: int, T: int, causal: bool) -> int:
    """KV tiles a unit processes: unit u is query tile T-1-u%T of its head (the kernel's numbering)."""
    return T - (u % T) if causal else T


def shard_units(B: int, H: int, N: int, causal: bool, world: int) -> list[tuple[int, int]]:
    """Contiguous [start, end) ranges of the B·H·T unit space whose KV-tile costs are as equal as a contiguous
    split allows (boundary r is placed where the cost prefix is closest to r/world of the total)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    T = tiles_per_head(N)
    n = B * H * T
    if not causal:
        return shard_ranges(n, world)
    # prefix cost of whole heads is closed-form; within a head the costs are T, T-1, ..., 1
    head_cost = T * (T + 1) // 2
    total = B * H * head_cost

    def prefix(u: int) -> int:  # cost of units [0, u)
        h, r = divmod(u, T)
        return h * head_cost + r * T - r * (r - 1) // 2

    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        lo, hi = bounds[-1], n
        while lo < hi:  # smallest u with prefix(u) >= target
            mid = (lo + hi) // 2
            if prefix(mid) < target:
                lo = mid + 1
            else:
                hi = mid
        u = lo
        if u > bounds[-1] and abs(prefix(u - 1) - target) < abs(prefix(u) - target):
            u -= 1
        bounds.append(max(u, bounds[-1]))
    bounds.append(n)
    return [(bounds[i], bounds[i + 1]) for i in range(world)]


def unit_rows(u: int, T: int, N: int) -> tuple[int, int, int]:
    """(flattened head, first row, end row) of unit u."""
    bh, r = divmod(u, T)
    qt = T - 1 - r
    return bh, qt * TILE, min(N, qt * TILE + TILE)


def _default_compute(q, k, v, causal, softmax_scale, unit_lo, unit_hi):
    import paper_2505_11594_b200 as s3

    qkv = s3.sage3_quantize_qkv(q, k, v)
    o = torch.empty_like(q)
    return s3.sage3_attn_fwd_units(qkv, o, unit_lo, unit_hi, causal=causal, softmax_scale=softmax_scale)


def forward_sharded(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, causal: bool = False,
                    softmax_scale: float = 0.0, group=None, gather_to: int = 0, compute=None):
    """Run the FP4 attention forward on this rank's work units and gather O on rank `gather_to`.

    q, k, v: the full [B, H, N, d] inputs (as every rank sees them; only the heads of this rank's units are
    read).  Returns the full O on `gather_to`; elsewhere this rank's packed [n_local_units, 128, d] rows.
    `compute(q, k, v, causal, softmax_scale, unit_lo, unit_hi)` maps the [1, n_heads, N, d] inputs of the
    touched heads to O for them, valid at least on the rows of units [unit_lo, unit_hi) (numbered within those
    heads).  It defaults to the CUDA path (sage3_quantize_qkv + sage3_attn_fwd_units through the C ABI);
    tests substitute a host stub to exercise the sharding and gather logic without a GPU.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    B, H, N, d = q.shape
    T = tiles_per_head(N)
    ranges = shard_units(B, H, N, causal, world)
    u0, u1 = ranges[rank]
    fn = compute or _default_compute
    flat = lambda x: x.reshape(B * H, N, d)
    packed = q.new_zeros(max(u1 - u0, 0), TILE, d)
    if u1 > u0:
        h0, h1 = u0 // T, (u1 - 1) // T + 1
        sl = slice(h0, h1)
        o_heads = fn(flat(q)[sl].unsqueeze(0), flat(k)[sl].unsqueeze(0), flat(v)[sl].unsqueeze(0), causal,
                     softmax_scale, u0 - h0 * T, u1 - h0 * T)[0]
        idx, valid = _row_index(u0, u1, T, N, h0, q.device)
        packed.view(-1, d)[valid] = o_heads.reshape(-1, d)[idx[valid]]
    if world == 1:
        out = q.new_empty(B * H, N, d)
        _unpack(out, packed, 0, u1, T, N)
        return out.reshape(B, H, N, d)
    # equal-size gather: pad every rank's packed rows to the largest range
    cap = max(e - s for s, e in ranges)
    buf = q.new_zeros(cap, TILE, d)
    buf[: packed.shape[0]] = packed
    if rank == gather_to:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, parts, dst=gather_to, group=group)
        out = q.new_empty(B * H, N, d)
        for p, (s, e) in zip(parts, ranges):
            _unpack(out, p, s, e, T, N)
        return out.reshape(B, H, N, d)
    dist.gather(buf, None, dst=gather_to, group=group)
    return packed


def _row_index(u0: int, u1: int, T: int, N: int, h0: int, device) -> tuple[torch.Tensor, torch.Tensor]:
    """For the packed rows of units [u0, u1) (TILE rows each): the flat row index into a [heads from h0][N]
    array, and whether the row exists (the last query tile of a head may be ragged)."""
    u = torch.arange(u0, u1, device=device, dtype=torch.int64)
    bh, r = u // T, u % T
    row0 = (T - 1 - r) * TILE
    rows = row0[:, None] + torch.arange(TILE, device=device, dtype=torch.int64)[None, :]
    valid = (rows < N).reshape(-1)
    idx = ((bh - h0)[:, None] * N + rows).reshape(-1)
    return idx, valid


def _unpack(out: torch.Tensor, packed: torch.Tensor, u0: int, u1: int, T: int, N: int):
    if u1 <= u0:
        return
    d = out.shape[-1]
    idx, valid = _row_index(u0, u1, T, N, 0, out.device)
    out.view(-1, d)[idx[valid]] = packed[: u1 - u0].reshape(-1, d)[valid]


# ------------------------------------------------------------------------------------------------ launcher
def self_launch(nprocs: int, argv: list[str], script: str) -> None:
    """One process per GPU: when `nprocs` > 1 and this process was not started by torch.distributed.run (no
    WORLD_SIZE in the environment), re-execute `script argv` under torch.distributed.run with nprocs ranks on
    127.0.0.1 (this call then does not return).  Otherwise a no-op."""
    import os
    import socket
    import sys

    if nprocs <= 1 or "WORLD_SIZE" in os.environ:
        return
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nprocs}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), script, *argv]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def init_from_env(backend: str):
    """(rank, world, local_rank) of a torchrun-launched process; initialises the default process group when
    world > 1 (NCCL on GPUs, gloo for the CPU tests)."""
    import os

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        kw = {}
        if backend == "nccl":
            kw["device_id"] = torch.device("cuda", local)
        dist.init_process_group(backend, **kw)
    return rank, world, local


class ShardPlan:
    """This rank's share of a B x H x N (x d) problem: its contiguous unit range [u0, u1) of the flattened
    (b·h, query-tile) space (shard_units) and the heads [h0, h1) those units touch."""

    def __init__(self, B: int, H: int, N: int, causal: bool, world: int, rank: int):
        self.B, self.H, self.N, self.causal, self.world, self.rank = B, H, N, causal, world, rank
        self.T = tiles_per_head(N)
        self.ranges = shard_units(B, H, N, causal, world)
        self.u0, self.u1 = self.ranges[rank]
        self.h0 = self.u0 // self.T
        self.h1 = (self.u1 - 1) // self.T + 1 if self.u1 > self.u0 else self.h0

    def head_chunks(self, min_units: int = 0):
        """(first head, head count, unit range numbered within those heads) of this rank's work, in order: the
        pieces the pipelined gather sends as soon as each is computed.  Consecutive heads are merged until a piece
        has at least `min_units` units (each piece is one quantize + one attention launch; a launch of a few
        hundred 128-row tiles leaves the 148 SMs a partial last wave)."""
        h = self.h0
        while h < self.h1:
            e = h + 1
            while e < self.h1 and (min(self.u1, e * self.T) - max(self.u0, h * self.T)) < min_units:
                e += 1
            lo, hi = max(self.u0, h * self.T), min(self.u1, e * self.T)
            yield h, e - h, lo - h * self.T, hi - h * self.T
            h = e


def pipelined_forward_gather(plan: ShardPlan, d: int, head_inputs, compute, *, dtype=None, device=None,
                             gather_to: int = 0, group=None, min_units: int = 1024):
    """Strong-scaling form of the launcher: this rank computes its units head by head and, for every finished
    head, starts the transfer of that head's rows to rank `gather_to` (non-blocking point-to-point sends, so the
    NCCL transfer of head h overlaps the compute of head h+1); rank `gather_to` posts all receives up front and
    assembles O.  Returns O [B, H, N, d] on `gather_to` (None elsewhere).

    head_inputs(h0, n) -> (q, k, v) [1, n, N, d] of flattened heads h0 .. h0+n-1 (each rank generates or loads only
    its own); pieces of at least `min_units` units (one piece for the whole range when there is nothing to send);
    compute(q, k, v, causal, scale, unit_lo, unit_hi) -> O [1, 1, N, d] valid on those units' rows (the CUDA path
    by default: _default_compute)."""
    rank, world, N, T = plan.rank, plan.world, plan.N, plan.T
    fn = compute or _default_compute
    out = None
    recvs = []
    if rank == gather_to:
        out = torch.empty(plan.B * plan.H, N, d, dtype=dtype, device=device)
        if world > 1:
            for src in range(world):
                if src == gather_to:
                    continue
                sp = ShardPlan(plan.B, plan.H, N, plan.causal, world, src)
                for h, _, lo, hi in sp.head_chunks(min_units):
                    buf = torch.empty((hi - lo) * TILE, d, dtype=dtype, device=device)
                    recvs.append((dist.irecv(buf, src=src, group=group), buf, h, lo, hi))
    sends = []
    mu = min_units if world > 1 else plan.u1 - plan.u0  # nothing to overlap on one GPU: one piece
    for h, nh, lo, hi in plan.head_chunks(mu):
        q, k, v = head_inputs(h, nh)
        o = fn(q, k, v, plan.causal, 0.0, lo, hi)[0]  # [nh, N, d]
        idx, valid = _row_index(h * T + lo, h * T + hi, T, N, h, o.device)
        rows = o.new_zeros((hi - lo) * TILE, d)
        rows[valid] = o.reshape(-1, d)[idx[valid]]
        if rank == gather_to:
            _unpack(out, rows.view(-1, TILE, d), h * T + lo, h * T + hi, T, N)
        else:
            sends.append((dist.isend(rows, dst=gather_to, group=group), rows))
    for w, _ in sends:
        w.wait()
    for w, buf, h, lo, hi in recvs:
        w.wait()
        _unpack(out, buf.view(-1, TILE, d), h * T + lo, h * T + hi, T, N)
    if out is not None:
        return out.view(plan.B, plan.H, N, d)
    return None
