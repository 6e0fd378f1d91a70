"""Self-test of the multi-GPU launcher path on CPU (gloo) or GPU (nccl): self_launch -> torchrun ranks ->
init_from_env -> ShardPlan -> pipelined_forward_gather, with a host stub standing in for the attention kernel
(--stub) or the CUDA path.  Rank 0 checks the gathered O against the unsharded computation and prints one line
"MG_SELFTEST OK world=<n> ..." (used by tests/test_multigpu_gloo.py).

    python tools/mg_selftest.py --nprocs 2 --stub            # CPU, gloo
    python tools/mg_selftest.py --nprocs 1                   # GPU, the product path on one device
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_11594_b200 import multigpu  # noqa: E402


def stub(q, k, v, causal, scale, unit_lo=None, unit_hi=None):
    # a per-head deterministic function standing in for the attention kernel (valid on every row)
    return v * 2.0 + q.sum(-1, keepdim=True) * (0.5 if causal else 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nprocs", type=int, default=2)
    ap.add_argument("--stub", action="store_true")
    ap.add_argument("--shape", default="1,5,300,16")
    ap.add_argument("--causal", action="store_true")
    ap.add_argument("--min-units", type=int, default=0)
    a = ap.parse_args()
    multigpu.self_launch(a.nprocs, sys.argv[1:], os.path.abspath(__file__))
    rank, world, local = multigpu.init_from_env("gloo" if a.stub else "nccl")
    B, H, N, d = (int(x) for x in a.shape.split(","))
    dev = torch.device("cpu") if a.stub else torch.device("cuda", local)
    if not a.stub:
        torch.cuda.set_device(dev)
    dtype = torch.float32 if a.stub else torch.bfloat16
    import synth

    def head_inputs(h0, n=1):
        parts = [synth.make_head(N, d, seed=3, b=h // H, h=h % H, H=H, dtype=dtype, device=dev)
                 for h in range(h0, h0 + n)]
        return tuple(torch.stack([p[i] for p in parts])[None] for i in range(3))

    plan = multigpu.ShardPlan(B, H, N, a.causal, world, rank)
    out = multigpu.pipelined_forward_gather(plan, d, head_inputs, stub if a.stub else None, dtype=dtype,
                                            device=dev, min_units=a.min_units)
    if rank == 0:
        ok = True
        for h in range(B * H):
            q, k, v = head_inputs(h)
            if a.stub:
                want = stub(q, k, v, a.causal, 0.0)[0, 0]
            else:
                import paper_2505_11594_b200 as s3

                want = s3.attention(q, k, v, causal=a.causal)[0, 0]
            ok &= bool(torch.equal(out.view(B * H, N, d)[h], want))
        print(f"MG_SELFTEST {'OK' if ok else 'FAIL'} world={world} units={plan.ranges}", flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
