"""Calibrate the element-wise parity bound (tests/parity.py) on the GPU: for several shapes, the GPU output vs the
oracle on the same codes, and for each decision window delta: elements outside ulp + TIGHT*vmax + amb(delta), the
fraction of rows with an allowance, and the worst error/tight ratio on rows without one.

    python tools/parity_diag.py [--p-quant two_level]
"""
import argparse
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import paper_2505_11594_b200 as s3  # noqa: E402
import synth  # noqa: E402
from parity import TIGHT, dtype_spacing, round_to, vmax_of  # noqa: E402
from test_gpu_attn import oracle_heads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p-quant", default="two_level")
a = ap.parse_args()
pm = {"two_level": oracle.PMODE_TWO_LEVEL, "direct": oracle.PMODE_DIRECT, "lazy": oracle.PMODE_LAZY}[a.p_quant]
deltas = [0.0, 1e-6, 4e-6, 1.6e-5, 3e-5, 6.4e-5, 2.56e-4]
for (N, d, causal, odt, rows_n) in [(15, 128, False, torch.float32, None), (64, 64, True, torch.float32, None),
                                    (300, 128, True, torch.float32, None), (1024, 128, False, torch.float32, None),
                                    (1024, 64, True, torch.bfloat16, None), (4096, 128, False, torch.float32, 256),
                                    (32768, 128, False, torch.bfloat16, 64)]:
    H = 2
    Q, K, V = synth.make_qkv(1, H, N, d, seed=7 * N + d, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    O = s3.sage3_attn_fwd(qkv, causal=causal, out_dtype=odt, p_quant=a.p_quant)
    torch.cuda.synchronize()
    heads = oracle_heads(qkv, range(H))
    rows = None if rows_n is None else np.unique(np.linspace(0, N - 1, rows_n).astype(np.int32))
    g_all = O.float().cpu().numpy().reshape(H, N, d)
    line = [f"N={N} d={d} {'c' if causal else 'n'} {str(odt)[6:]}:"]
    for dl in deltas:
        ref, _, amb = oracle.attn_fwd(heads, causal=causal, scale=1 / math.sqrt(d), rows=rows, p_mode=pm,
                                      amb_delta=dl)
        out, fr, worst = 0, 0.0, 0.0
        for h in range(H):
            g = g_all[h] if rows is None else g_all[h][rows]
            r = round_to(ref[h], odt)
            vm = vmax_of(heads[h])
            tight = dtype_spacing(np.maximum(np.abs(g), np.abs(r)), odt) + TIGHT * vm
            err = np.abs(g - r)
            out += int((err > tight + 1.01 * amb[h]).sum())
            fr += float(np.mean(amb[h].max(axis=1) > 0)) / H
            clean = amb[h].max(axis=1) == 0
            if clean.any():
                worst = max(worst, float((err[clean] / tight[clean]).max()))
        line.append(f"d{dl:g}: out={out} rows%={100 * fr:.1f} worst_clean={worst:.2f}")
    print(" | ".join(line), flush=True)
