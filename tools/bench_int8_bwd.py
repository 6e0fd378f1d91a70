#!/usr/bin/env python3
"""Device-timed throughput of SageBwd's backward (NEXT #3, Alg3): sage3_int8_attn_bwd at B=1, H=32, d=128 over N
(one JSON line per (N, causal)); TOPS = 10·B·H·N²·d (five N x N x d matmuls: S, dP, dV, dK, dQ; x0.5 causal) /
time of the whole call (memset + prep + main + dQ finalize), with the forward (quantize + attention) that produces
its O and lse timed alongside."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_11594_b200 as s3  # noqa: E402
import synth  # noqa: E402


def main():
    H, d = 32, int(os.environ.get("SAGE3_D", "128"))
    Ns = [int(x) for x in sys.argv[1:]] or [4096, 16384, 32768]
    for N in Ns:
        Q, K, V = synth.make_qkv(1, H, N, d, seed=0, dtype=torch.bfloat16, device="cuda")
        dO = torch.randn_like(Q)
        qkv = s3.sage3_int8_quantize_qkv(Q, K, V)
        O = torch.empty_like(Q)
        lse = torch.empty(1, H, N, dtype=torch.float32, device="cuda")
        ws = torch.empty(s3.sage3_int8_bwd_workspace_bytes(1, H, N, d), dtype=torch.uint8, device="cuda")
        grads = [torch.empty(1, H, N, d, dtype=torch.bfloat16, device="cuda") for _ in range(3)]
        for causal in (False, True):
            s3.sage3_int8_attn_fwd(qkv, O, causal=causal, lse=lse)
            ops = 10.0 * H * N * N * d * (0.5 if causal else 1.0)
            reps = max(3, int(3e13 / ops))
            run = lambda: s3.sage3_int8_attn_bwd(qkv, V, O, dO, lse, causal=causal, dq=grads[0], dk=grads[1],  # noqa
                                                 dv=grads[2], workspace=ws)
            for _ in range(2):
                run()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            e[0].record()
            for _ in range(reps):
                run()
            e[1].record()
            torch.cuda.synchronize()
            ms = e[0].elapsed_time(e[1]) / reps
            print(json.dumps({"workload": f"SageBwd bwd B=1,H={H},N={N},d={d},{'causal' if causal else 'non-causal'}",
                              "bwd_ms": round(ms, 4), "bwd_TOPS": round(ops / ms / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
