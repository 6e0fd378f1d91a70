"""Seeded synthetic Q, K, V for the SageAttention3 hot path — shared by tests, bench and smoke.

This module holds NO arithmetic of the method: it only draws random tensors.  Both the CUDA path and
the CPU oracle consume its output (the oracle via a host copy), and neither imports the other.

Recipe (SURVEY §8(d) "concrete synthetic inputs", SPEC S:446-453 GaussianOutlierChannels):
  * one torch.Generator per (b, h), seeded seed*1000003 + b*H + h, so a head's values do not depend on
    how heads are sharded over GPUs;
  * Q, K, V ~ N(0, 1) drawn in fp32, then cast to the input dtype (bf16 or fp16);
  * K gets a per-channel offset mu_c ~ N(0, 1) plus 4 outlier channels with mu = +-20 (what smoothing K,
    Alg1 L2 / P:144, removes); Q gets 2 outlier channels scaled x10 (the channel outliers that motivate
    microscaling).
"""
from __future__ import annotations

import torch


def head_seed(seed: int, b: int, h: int, H: int) -> int:
    return seed * 1000003 + b * H + h


def make_head(N: int, d: int, *, seed: int = 0, b: int = 0, h: int = 0, H: int = 1, dtype=torch.bfloat16,
              device="cpu", outliers: bool = True):
    """One head: returns (Q, K, V), each [N, d] of `dtype` on `device`."""
    g = torch.Generator(device=device)
    g.manual_seed(head_seed(seed, b, h, H))
    q = torch.randn(N, d, generator=g, device=device, dtype=torch.float32)
    k = torch.randn(N, d, generator=g, device=device, dtype=torch.float32)
    v = torch.randn(N, d, generator=g, device=device, dtype=torch.float32)
    if outliers:
        mu = torch.randn(d, generator=g, device=device, dtype=torch.float32)
        perm = torch.randperm(d, generator=g, device=device)
        sign = torch.randint(0, 2, (4,), generator=g, device=device).to(torch.float32) * 2 - 1
        mu[perm[2:6]] = 20.0 * sign
        k += mu
        q[:, perm[:2]] *= 10.0
    return q.to(dtype), k.to(dtype), v.to(dtype)


def make_qkv(B: int, H: int, N: int, d: int, *, seed: int = 0, dtype=torch.bfloat16, device="cpu",
             heads=None, outliers: bool = True):
    """[B, H, N, d] tensors.  `heads` (iterable of flat b*H+h indices) restricts generation to a shard;
    the other heads are left zero (callers pass the shard's own buffers)."""
    Q = torch.empty(B, H, N, d, dtype=dtype, device=device)
    K = torch.empty_like(Q)
    V = torch.empty_like(Q)
    idx = range(B * H) if heads is None else heads
    for f in idx:
        b, h = divmod(f, H)
        q, k, v = make_head(N, d, seed=seed, b=b, h=h, H=H, dtype=dtype, device=device, outliers=outliers)
        Q[b, h], K[b, h], V[b, h] = q, k, v
    return Q, K, V
