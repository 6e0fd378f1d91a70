"""Small end-to-end cases for compute-sanitizer (SURVEY §4 layer 7): quantize + attention (d 64/128, causal
and not, ragged N, smoothing Q, MXFP4, direct, lazy and qsum P, SageBwd INT8 forward and backward) through the C ABI,
plus the host-buffer path.  With SAGE3_QUANT_FUSED_K=1 in the environment the quantizer runs its fused K-mean path.
  compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_case.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_11594_b200 as s3  # noqa: E402
import synth  # noqa: E402

for d in (64, 128):
    for causal in (False, True):
        for N in (256, 200):
            Q, K, V = synth.make_qkv(1, 1, N, d, seed=N, dtype=torch.bfloat16, device="cuda")
            s3.attention(Q, K, V, causal=causal)
            s3.attention(Q, K, V, causal=causal, smooth_q=True)
            s3.attention(Q, K, V, causal=causal, fmt="mxfp4")
            s3.attention(Q, K, V, causal=causal, p_quant="direct")
            s3.attention(Q, K, V, causal=causal, p_quant="lazy")
            s3.attention(Q, K, V, causal=causal, fmt="mxfp4", p_quant="lazy")
            s3.attention(Q, K, V, causal=causal, p_quant="qsum")  # round 2: the row-sum variant
            qkv8 = s3.sage3_int8_quantize_qkv(Q, K, V)
            lse = torch.empty(1, 1, N, dtype=torch.float32, device="cuda")
            O8 = s3.sage3_int8_attn_fwd(qkv8, causal=causal, lse=lse)
            s3.sage3_int8_attn_bwd(qkv8, V, O8, torch.randn_like(Q), lse, causal=causal)
            torch.cuda.synchronize()
Q, K, V = synth.make_qkv(1, 2, 300, 128, seed=1, dtype=torch.bfloat16, device="cpu")
qh, kh, vh = (x.pin_memory() for x in (Q, K, V))
oh = torch.empty_like(qh).pin_memory()
scratch = torch.empty(s3.sage3_forward_host_scratch_bytes(1, 2, 300, 128), dtype=torch.uint8, device="cuda")
s3.sage3_forward_host(qh, kh, vh, oh, scratch)
torch.cuda.synchronize()
print("sanitize cases done")
