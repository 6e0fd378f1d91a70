#!/usr/bin/env python3
"""Device-timed throughput of SageBwd's 8-bit forward (NEXT #3): sage3_int8_quantize_qkv + sage3_int8_attn_fwd at
B=1, H=32, d=128 over N (one JSON line per (N, causal)); TOPS = 4·B·H·N²·d (x0.5 causal) / time."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_11594_b200 as s3  # noqa: E402
import synth  # noqa: E402


def main():
    H, d = 32, 128
    for N in (4096, 16384, 32768):
        Q, K, V = synth.make_qkv(1, H, N, d, seed=0, dtype=torch.bfloat16, device="cuda")
        qkv = s3.sage3_int8_quantize_qkv(Q, K, V)
        O = torch.empty_like(Q)
        for causal in (False, True):
            ops = 4.0 * H * N * N * d * (0.5 if causal else 1.0)
            reps = max(3, int(3e13 / ops))
            for _ in range(2):
                s3.sage3_int8_quantize_qkv(Q, K, V, out=qkv)
                s3.sage3_int8_attn_fwd(qkv, O, causal=causal)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            for _ in range(reps):
                s3.sage3_int8_quantize_qkv(Q, K, V, out=qkv)
            e[1].record()
            for _ in range(reps):
                s3.sage3_int8_attn_fwd(qkv, O, causal=causal)
            e[2].record()
            torch.cuda.synchronize()
            qm, am = e[0].elapsed_time(e[1]) / reps, e[1].elapsed_time(e[2]) / reps
            print(json.dumps({"workload": f"SageBwd fwd B=1,H={H},N={N},d={d},{'causal' if causal else 'non-causal'}",
                              "quantize_ms": round(qm, 4), "attn_ms": round(am, 4),
                              "attn_TOPS": round(ops / am / 1e9, 1), "step_TOPS": round(ops / (qm + am) / 1e9, 1)}),
                  flush=True)


if __name__ == "__main__":
    main()
