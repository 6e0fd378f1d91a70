"""Small probe of the attention path (whichever SAGE3_ATTN_KERNEL selects) against the oracle: one head per shape."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import torch

import oracle
import paper_2505_11594_b200 as s3
import synth
from layout import decode_head
from parity import check, oracle_attention

dev = torch.device("cuda", 0)
for (N, d, causal) in [(128, 128, False), (300, 128, True), (1000, 128, False), (700, 64, True), (1, 128, False)]:
    Q, K, V = synth.make_qkv(1, 2, N, d, seed=5, dtype=torch.bfloat16, device=dev)
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    O = s3.sage3_attn_fwd(qkv, causal=causal, out_dtype=torch.float32)
    torch.cuda.synchronize()
    for bh in range(2):
        h = oracle.quantize_head(*(x[0, bh].float().cpu().numpy() for x in (Q, K, V)))
        ref, _, amb, vmax = oracle_attention([h], causal=causal, scale=1 / math.sqrt(d))
        m = check(O[0, bh].cpu().numpy(), ref[0], torch.float32, f"N={N} d={d} c={causal} h{bh}", amb=amb[0], vmax=vmax[0])
    print("ok", N, d, causal, {k: (round(v, 8) if isinstance(v, float) else v) for k, v in m.items()}, flush=True)
