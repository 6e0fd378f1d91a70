"""Parity of one attention kernel selection against the oracle (run in a subprocess by test_gpu_attn_kernels.py with
SAGE3_ATTN_KERNEL=2 (attn.cu) or =3 (attn3.cu) fixed for the process): every case through the C ABI, both gates of
tests/parity.py on every element, and canary bands around O (rows and columns) and the LSE that every write must
leave untouched (an out-of-bounds check that does not need compute-sanitizer)."""
import math
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), HERE]
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2505_11594_b200 as s3  # noqa: E402
import synth  # noqa: E402
from parity import check, oracle_attention  # noqa: E402

CASES = [(1, 128, False), (15, 64, True), (127, 128, True), (128, 64, False), (300, 128, True), (1000, 64, False),
         (1000, 128, False), (2100, 128, True), (2100, 64, False), (700, 64, True)]


def main():
    dev = torch.device("cuda", 0)
    for i, (N, d, causal) in enumerate(CASES):
        for dt in (torch.bfloat16, torch.float16):
            Q, K, V = synth.make_qkv(1, 2, N, d, seed=40 + i, dtype=dt, device=dev)
            qkv = s3.sage3_quantize_qkv(Q, K, V)
            # O and the LSE are views into canary-filled buffers (128 rows before and after each head's rows, 16 extra
            # columns per row, 32 floats around the LSE): every write outside them is caught
            big = torch.full((1, 2, N + 256, d + 16), float("nan"), dtype=torch.float32, device=dev)
            O = big[:, :, 128:128 + N, :d]
            lse_big = torch.full((2 * N + 64,), float("nan"), dtype=torch.float32, device=dev)
            lse = lse_big[32:32 + 2 * N]
            s3.sage3_attn_fwd(qkv, O, causal=causal, lse=lse)
            torch.cuda.synchronize()
            canary = big.clone()
            canary[:, :, 128:128 + N, :d] = float("nan")
            assert torch.isnan(canary).all(), f"N={N} d={d} causal={causal}: write outside O"
            assert torch.isnan(lse_big[:32]).all() and torch.isnan(lse_big[32 + 2 * N:]).all(), "write outside lse"
            assert torch.isfinite(lse).all() and torch.isfinite(O).all(), "unwritten O / lse element"
            for bh in range(2):
                h = oracle.quantize_head(*(x[0, bh].float().cpu().numpy() for x in (Q, K, V)))
                ref, _, amb, vmax = oracle_attention([h], causal=causal, scale=1 / math.sqrt(d))
                check(O[0, bh].cpu().numpy(), ref[0], torch.float32, f"N={N} d={d} causal={causal} {dt} head {bh}",
                      amb=amb[0], vmax=vmax[0])
        print("ok", N, d, causal, flush=True)
    print("ALL OK")


if __name__ == "__main__":
    main()
