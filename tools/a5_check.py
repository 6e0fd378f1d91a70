"""attn5.cu (B_kv = 64) against the oracle run with bkv = 64 (non-causal), both gates of tests/parity.py on every
element; run with SAGE3_ATTN_KERNEL=5."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2505_11594_b200 as s3  # noqa: E402
import synth  # noqa: E402
from parity import check, oracle_attention  # noqa: E402

dev = torch.device("cuda", 0)
for i, (N, d) in enumerate([(1, 128), (64, 128), (100, 64), (128, 128), (300, 128), (1000, 64), (1000, 128),
                            (2100, 128), (2100, 64)]):
    Q, K, V = synth.make_qkv(1, 2, N, d, seed=70 + i, dtype=torch.bfloat16, device=dev)
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    big = torch.full((1, 2, N + 256, d + 16), float("nan"), dtype=torch.float32, device=dev)
    O = big[:, :, 128:128 + N, :d]
    s3.sage3_attn_fwd(qkv, O, causal=False)
    torch.cuda.synchronize()
    canary = big.clone()
    canary[:, :, 128:128 + N, :d] = float("nan")
    assert torch.isnan(canary).all(), "write outside O"
    for bh in range(2):
        h = oracle.quantize_head(*(x[0, bh].float().cpu().numpy() for x in (Q, K, V)))
        ref, _, amb, vmax = oracle_attention([h], causal=False, scale=1 / math.sqrt(d), bkv=64)
        m = check(O[0, bh].cpu().numpy(), ref[0], torch.float32, f"N={N} d={d} head {bh}", amb=amb[0], vmax=vmax[0])
    print("ok", N, d, {k: (round(v, 8) if isinstance(v, float) else v) for k, v in m.items()}, flush=True)
print("ALL OK")
