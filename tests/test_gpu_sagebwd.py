"""GPU parity of SageBwd's 8-bit forward (NEXT #3, Algorithm 2): the INT8 quantizer (smooth-K mean, per-block
ψ codes and scales) BIT-EXACT against oracle.sb_quantize_head, and the kind::i8 attention against
oracle.sb_attn_fwd on the same codes (north_star tolerance, LSE), plus the Q = 0 closed form."""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_2505_11594_b200 as s3
import parity
import synth

pytestmark = pytest.mark.gpu


def decode(qkv, bh):
    Np, d, T = qkv.N_pad, qkv.d, qkv.N_pad // 128
    h = oracle.SbHead(qkv.N, d)
    h.q = qkv.q.view(torch.int8).view(-1, Np, d)[bh].cpu().numpy()
    h.k = qkv.k.view(torch.int8).view(-1, Np, d)[bh].cpu().numpy()
    h.v = np.ascontiguousarray(qkv.v_t.view(torch.int8).view(-1, d, Np)[bh].cpu().numpy().T)
    h.sq, h.sk, h.sv = (getattr(qkv, n).view(torch.float32).view(-1, T)[bh].cpu().numpy() for n in ("s_q", "s_k", "s_v"))
    h.km = qkv.k_mean.view(torch.float32).view(-1, d)[bh].cpu().numpy()
    return h


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("N", [1, 127, 128, 300, 1000])
def test_int8_quantize_bit_exact(dtype, d, N):
    Q, K, V = synth.make_qkv(1, 2, N, d, seed=N + 3 * d, dtype=dtype, device="cuda")
    qkv = s3.sage3_int8_quantize_qkv(Q, K, V)
    torch.cuda.synchronize()
    for bh in range(2):
        got = decode(qkv, bh)
        want = oracle.sb_quantize_head(*(x[0, bh].float().cpu().numpy() for x in (Q, K, V)))
        for name in ("km", "sq", "sk", "sv", "q", "k", "v"):
            g, w = getattr(got, name), getattr(want, name)
            bad = np.argwhere(g != w)
            assert bad.size == 0, f"{name}: {len(bad)} mismatches, first {bad[:3].tolist()}"


def check(gpu, ref, what="", amb=None, vmax=None):
    """north_star per-head gate + the element-wise bound of tests/parity.py (fp32 output)."""
    return parity.check(gpu, ref, torch.float32, what, amb=amb, vmax=vmax)


def sb_vmax(h) -> float:
    """max |deq(V̂)| of a SageBwd head: |int8 code| x its block scale."""
    T = h.Np // 128
    return float((np.abs(h.v.astype(np.float64)).reshape(T, 128, -1).max(axis=(1, 2)) * h.sv).max())


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("N,d", [(1, 64), (15, 128), (127, 64), (128, 128), (300, 64), (1000, 128), (2000, 64)])
def test_int8_attention_parity(N, d, causal):
    B, H = 1, 2
    Q, K, V = synth.make_qkv(B, H, N, d, seed=N + d, dtype=torch.bfloat16, device="cuda", outliers=False)
    qkv = s3.sage3_int8_quantize_qkv(Q, K, V)
    lse = torch.empty(B, H, N, dtype=torch.float32, device="cuda")
    O = s3.sage3_int8_attn_fwd(qkv, causal=causal, lse=lse, out_dtype=torch.float32)
    torch.cuda.synchronize()
    rows = np.arange(N, dtype=np.int32) if N <= 1000 else np.arange(0, N, 3, dtype=np.int32)
    heads = [decode(qkv, bh) for bh in range(B * H)]
    ref, ref_lse, amb = oracle.sb_attn_fwd(heads, causal=causal, scale=1 / math.sqrt(d), rows=rows,
                                           amb_delta=parity.AMB_DELTA)
    for bh in range(B * H):
        check(O[0, bh].cpu().numpy()[rows], ref[bh], f"head {bh}", amb=amb[bh], vmax=sb_vmax(heads[bh]))
    np.testing.assert_allclose(lse.cpu().numpy().reshape(B * H, N)[:, rows], ref_lse, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("out_dtype", [torch.bfloat16, torch.float16])
def test_int8_attention_16bit_outputs(out_dtype):
    Q, K, V = synth.make_qkv(2, 2, 500, 128, seed=7, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_int8_quantize_qkv(Q, K, V)
    O32 = s3.sage3_int8_attn_fwd(qkv, causal=True, out_dtype=torch.float32)
    O16 = s3.sage3_int8_attn_fwd(qkv, causal=True, out_dtype=out_dtype)
    torch.cuda.synchronize()
    assert torch.equal(O16, O32.to(out_dtype))


@pytest.mark.parametrize("causal", [False, True])
def test_int8_zero_query_closed_form(causal):
    """Q = 0: P̂ = 127, s_P = 1/127 -> O = (running) mean of deq(V̂) (x 127·fl32(1/127) in the oracle; the
    kernel's fp32 weight 2^0/127 differs from it by < 1 ulp)."""
    N, d = 384, 64
    _, K, V = synth.make_qkv(1, 1, N, d, seed=3, device="cuda")
    qkv = s3.sage3_int8_quantize_qkv(torch.zeros_like(K), K, V)
    O = s3.sage3_int8_attn_fwd(qkv, causal=causal, out_dtype=torch.float32)
    torch.cuda.synchronize()
    h = decode(qkv, 0)
    Vd = h.v[:N].astype(np.float64) * np.repeat(h.sv, 128)[:N, None]
    cnt = np.arange(1, N + 1) if causal else np.full(N, N)
    ref = (np.cumsum(Vd, axis=0) / cnt[:, None]) if causal else np.broadcast_to(Vd.mean(0), (N, d))
    np.testing.assert_allclose(O[0, 0].cpu().numpy(), ref, rtol=1e-5, atol=1e-6)


def test_int8_accuracy_vs_fp64():
    """Alg 2 vs full-precision attention on the GPU path (the paper's 8-bit forward is near lossless)."""
    N, d = 2048, 128
    Q, K, V = synth.make_qkv(1, 1, N, d, seed=13, dtype=torch.bfloat16, device="cuda", outliers=False)
    rows = np.arange(0, N, 8, dtype=np.int32)
    ref = oracle.reference_attention(Q[0, 0].float().cpu().numpy(), K[0, 0].float().cpu().numpy(),
                                     V[0, 0].float().cpu().numpy(), causal=False, scale=1 / math.sqrt(d), rows=rows)
    qkv = s3.sage3_int8_quantize_qkv(Q, K, V)
    O = s3.sage3_int8_attn_fwd(qkv, out_dtype=torch.float32)[0, 0].cpu().numpy()[rows]
    m = oracle.accuracy_metrics(ref, O)
    print("GPU SageBwd forward vs fp64:", m)
    assert m["cos_sim"] > 0.9995
