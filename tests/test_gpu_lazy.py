"""GPU parity of the NEXT #2 throughput variant (p_quant = "lazy", attn_lazy.cu; reading n1) against
the oracle's PMODE_LAZY on the same codes: north_star tolerance on O, LSE, both FP4 formats, causal and not,
ragged N, unit sub-ranges bitwise; the Q = 0 closed form; and the accuracy the variant is meant to keep."""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_2505_11594_b200 as s3
import synth
from parity import check, oracle_attention
from test_gpu_attn import oracle_heads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fmt", ["nvfp4", "mxfp4"])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("N,d", [(1, 64), (15, 128), (127, 64), (128, 128), (300, 64), (1024, 128), (2500, 64)])
def test_lazy_parity(N, d, causal, fmt):
    B, H = 1, 2
    Q, K, V = synth.make_qkv(B, H, N, d, seed=17 * N + d, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V, fmt=fmt)
    lse = torch.empty(B, H, N, dtype=torch.float32, device="cuda")
    O = s3.sage3_attn_fwd(qkv, causal=causal, out_dtype=torch.float32, lse=lse, p_quant="lazy")
    torch.cuda.synchronize()
    rows = np.arange(N, dtype=np.int32) if N <= 1024 else np.arange(0, N, 7, dtype=np.int32)
    ref, ref_lse, amb, vmax = oracle_attention(oracle_heads(qkv, range(B * H)), causal=causal,
                                               scale=1 / math.sqrt(d), p_mode=oracle.PMODE_LAZY, rows=rows)
    for bh in range(B * H):
        check(O[0, bh].cpu().numpy()[rows], ref[bh], torch.float32, f"head {bh}", amb=amb[bh], vmax=vmax[bh])
    np.testing.assert_allclose(lse.cpu().numpy().reshape(B * H, N)[:, rows], ref_lse, rtol=1e-5, atol=1e-4)
    O2 = torch.zeros_like(O)
    n = s3.n_units(qkv)
    s3.sage3_attn_fwd_ex(qkv, O2, causal=causal, p_quant="lazy", unit_begin=0, unit_end=n // 3)
    s3.sage3_attn_fwd_ex(qkv, O2, causal=causal, p_quant="lazy", unit_begin=n // 3)
    torch.cuda.synchronize()
    assert torch.equal(O, O2)


@pytest.mark.parametrize("out_dtype", [torch.bfloat16, torch.float16])
def test_lazy_bf16_fp16_outputs_and_strided(out_dtype):
    B, H, N, d = 2, 3, 700, 128
    Q, K, V = synth.make_qkv(B, H, N, d, seed=5, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    want = s3.sage3_attn_fwd(qkv, causal=True, out_dtype=torch.float32, p_quant="lazy")
    big = torch.zeros(B, N, H, 2 * d, dtype=out_dtype, device="cuda")
    view = big[..., :d].permute(0, 2, 1, 3)
    s3.sage3_attn_fwd(qkv, view, causal=True, p_quant="lazy")
    torch.cuda.synchronize()
    assert torch.equal(view, want.to(out_dtype))
    assert not big[..., d:].any()


@pytest.mark.parametrize("causal", [False, True])
def test_lazy_zero_query_closed_form(causal):
    """Q = 0: r = 0, P̃2 = 10.5 = 6·1.75 exactly -> O = (causal) running mean of deq(V̂), lse = ln(#keys)."""
    N, d = 384, 128
    _, K, V = synth.make_qkv(1, 1, N, d, seed=3, device="cuda")
    qkv = s3.sage3_quantize_qkv(torch.zeros_like(K), K, V)
    lse = torch.empty(1, 1, N, dtype=torch.float32, device="cuda")
    O = s3.sage3_attn_fwd(qkv, causal=causal, out_dtype=torch.float32, lse=lse, p_quant="lazy")
    torch.cuda.synchronize()
    h = oracle_heads(qkv, [0])[0]
    Vd = oracle.dequant(h.v_codes, h.v_sf)[:, :N].T
    cnt = np.arange(1, N + 1) if causal else np.full(N, N)
    ref = (np.cumsum(Vd, axis=0) / cnt[:, None]) if causal else np.broadcast_to(Vd.mean(0), (N, d))
    np.testing.assert_allclose(O[0, 0].cpu().numpy(), ref, rtol=2e-5, atol=2e-6)
    np.testing.assert_allclose(lse[0, 0].cpu().numpy(), np.log(cnt), rtol=1e-5, atol=1e-5)


def test_lazy_accuracy_close_to_two_level_on_gpu():
    """vs fp64 attention, the variant stays within 20% of the paper's two-level rel-L1 (reading n1's claim)."""
    N, d = 4096, 128
    Q, K, V = synth.make_qkv(1, 1, N, d, seed=51, dtype=torch.bfloat16, device="cuda")
    Q = (Q.float() * 3).to(torch.bfloat16)  # sharper attention: many P̃ far below the row max
    rows = np.arange(0, N, 16, dtype=np.int32)
    ref = oracle.reference_attention(Q[0, 0].float().cpu().numpy(), K[0, 0].float().cpu().numpy(),
                                     V[0, 0].float().cpu().numpy(), causal=False, scale=1 / math.sqrt(d), rows=rows)
    m = {p: oracle.accuracy_metrics(ref, s3.attention(Q, K, V, p_quant=p, out_dtype=torch.float32)[0, 0].cpu().numpy()[rows])
         for p in ("two_level", "lazy", "direct")}
    print("GPU two-level / lazy / direct:", m)
    assert m["lazy"]["l1"] <= 1.2 * m["two_level"]["l1"]
