#!/usr/bin/env python3
"""The other BASELINE.json configurations (C3 CogVideoX-shaped, C4 HunyuanVideo-shaped, C5 Llama-prefill
causal) as STRONG-scaling runs: the whole configuration is split over the ranks with the launcher's
cost-balanced (b·h, query-tile) unit split (paper_2505_11594_b200.multigpu.shard_units); each rank
quantizes the heads its units touch and runs sage3_attn_fwd_units on its range.  One JSON line per config
(rank 0), device-timed with CUDA events, max over ranks.  bench.py remains the driver's contract (C2).

  python tools/bench_configs.py [--configs C3,C4,C5] [--steps K] [--warmup W]
  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/bench_configs.py ...
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2505_11594_b200 as s3  # noqa: E402
import synth  # noqa: E402
from paper_2505_11594_b200.multigpu import shard_units, tiles_per_head, unit_cost  # noqa: E402

CONFIGS = {  # BASELINE.json configs[2..4]
    "C3": dict(B=2, H=30, N=17776, d=64, causal=False, name="CogVideoX-2B-shaped B=2,H=30,N=17776,d=64"),
    "C4": dict(B=1, H=24, N=118800, d=128, causal=False, name="HunyuanVideo-shaped B=1,H=24,N=118800,d=128"),
    "C5": dict(B=8, H=32, N=32768, d=128, causal=True, name="Llama prefill B=8,H=32,N=32768,d=128,causal"),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C3,C4,C5")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream(dev)
    for key in args.configs.split(","):
        c = CONFIGS[key]
        B, H, N, d, causal = c["B"], c["H"], c["N"], c["d"], c["causal"]
        T = tiles_per_head(N)
        u0, u1 = shard_units(B, H, N, causal, world)[rank]
        h0, h1 = u0 // T, (u1 - 1) // T + 1
        nh = h1 - h0
        Q = torch.empty(1, nh, N, d, dtype=torch.bfloat16, device=dev)
        K, V = torch.empty_like(Q), torch.empty_like(Q)
        for i, f in enumerate(range(h0, h1)):
            b, h = divmod(f, H)
            Q[0, i], K[0, i], V[0, i] = synth.make_head(N, d, seed=0, b=b, h=h, H=H, dtype=torch.bfloat16,
                                                        device=dev)
        qkv = s3.FP4QKV(1, nh, N, d, dev)
        O = torch.empty_like(Q)
        lo, hi = u0 - h0 * T, u1 - h0 * T

        def step():
            s3.sage3_quantize_qkv(Q, K, V, out=qkv, stream=stream)
            s3.sage3_attn_fwd_units(qkv, O, lo, hi, causal=causal, stream=stream)

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        if dist:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        ops = 4.0 * B * H * N * N * d * (0.5 if causal else 1.0)
        local_cost = sum(unit_cost(u, T, causal) for u in range(u0, u1))
        if rank == 0:
            print(json.dumps({
                "config": key, "workload": c["name"], "n_gpus": world, "scaling": "strong",
                "metric": "FP4 attention fwd TOPS (quantize + attention, whole job)", "unit": "TOPS",
                "value": ops / (ms * 1e-3) / 1e12, "ms_per_step": ms, "steps": args.steps,
                "units_rank0": u1 - u0, "heads_touched_rank0": nh, "kv_tiles_rank0": local_cost,
            }), flush=True)
        del Q, K, V, qkv, O
        torch.cuda.empty_cache()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
