"""Pins for the oracle's Algorithm 1: the online-softmax recurrence against plain softmax
attention (the definition), shift invariance behind smoothing K, and closed forms where
the quantized pipeline is exact (S = 0 everywhere; causal row 0; N = 1)."""
import numpy as np
import pytest
import torch
from scipy.special import softmax

import oracle
import synth


def numpy_attention(Q, K, V, scale, causal):
    """Plain softmax attention written directly from P:71 with scipy's softmax (independent of the oracle)."""
    Q, K, V = (np.asarray(x, np.float64) for x in (Q, K, V))
    S = scale * (Q @ K.T)
    if causal:
        S = np.where(np.tril(np.ones_like(S, dtype=bool)), S, -np.inf)
    return softmax(S, axis=1) @ V


def head(N, d, seed=0, dtype=torch.float16):
    q, k, v = synth.make_head(N, d, seed=seed, dtype=dtype)
    return q.float().numpy(), k.float().numpy(), v.float().numpy()


@pytest.mark.parametrize("bkv", [16, 64, 128])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("N,d", [(200, 64), (130, 128)])
def test_tiled_recurrence_equals_plain_attention(N, d, bkv, causal):
    """With P quantization off (p_mode NONE) Alg1's tiled recurrence is FlashAttention and must equal
    softmax(QK^T)V for every B_kv — pins m, alpha, l and the final diag(l)^-1."""
    Q, K, V = head(N, d, seed=N + d)
    scale = 1.0 / np.sqrt(d)
    O = oracle.attn_fwd_float(Q, K, V, causal=causal, scale=scale, bkv=bkv)
    ref = numpy_attention(Q, K, V, scale, causal)
    np.testing.assert_allclose(O, ref, rtol=1e-11, atol=1e-12)
    O2 = oracle.reference_attention(Q, K, V, causal=causal, scale=scale)
    np.testing.assert_allclose(O2, ref, rtol=1e-11, atol=1e-12)


def test_shift_invariance_of_keys():
    """Adding a constant row vector to every key leaves softmax(QK^T) unchanged (basis of Alg1 L2)."""
    N, d = 160, 64
    Q, K, V = head(N, d, seed=1)
    c = np.random.default_rng(0).integers(-8, 9, d).astype(np.float32)  # exact in fp32
    a = oracle.attn_fwd_float(Q, K, V, causal=False, scale=0.125, bkv=64)
    b = oracle.attn_fwd_float(Q, (K + c).astype(np.float32), V, causal=False, scale=0.125, bkv=64)
    np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-10)


def _deqV(h):
    return oracle.dequant(h.v_codes, h.v_sf)  # [d][Np]


C2688 = 2688.0 * float(np.float32(1.0) / np.float32(2688.0))  # deq(P̂2) * s_P1 when P̃ == 1


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("N,d", [(128, 64), (300, 128), (1, 64)])
def test_zero_scores_closed_form(N, d, causal):
    """Q = 0 => S = 0 => P̃ = 1, s_P1 = fl32(1/2688), P̃2 = 2688 -> s_P2 = 448, codes 6 (Alg1 L9-L11).
    O_i = mean_{j visible} deq(V̂)_j * 2688 * fl32(1/2688) exactly (up to fp64 summation)."""
    _, K, V = head(N, d, seed=2)
    Q = np.zeros((N, d), np.float32)
    h = oracle.quantize_head(Q, K, V)
    O = oracle.attn_fwd([h], causal=causal, scale=1 / np.sqrt(d))[0]
    Vd = _deqV(h)[:, :N].T  # [N][d]
    if causal:
        ref = np.cumsum(Vd, axis=0) / np.arange(1, N + 1)[:, None]
    else:
        ref = np.broadcast_to(Vd.mean(axis=0), (N, d))
    np.testing.assert_allclose(O, ref * C2688, rtol=1e-12, atol=1e-12)


def test_identical_keys_smoothed_to_zero():
    """Smoothing K (Alg1 L2): identical key rows become exactly 0 after K - mean(K), so S = 0 for any Q
    and the output is the same closed form as Q = 0.  Without smoothing it is not."""
    N, d = 256, 64
    Q, K, V = head(N, d, seed=3)
    K = np.tile(K[7], (N, 1))
    h = oracle.quantize_head(Q, K, V)
    assert not h.k_codes.any() and not h.k_sf.any()
    O = oracle.attn_fwd([h], causal=False, scale=0.125)[0]
    ref = _deqV(h)[:, :N].T.mean(axis=0)
    np.testing.assert_allclose(O, np.broadcast_to(ref, O.shape) * C2688, rtol=1e-12, atol=1e-12)
    h2 = oracle.quantize_head(Q, K, V, smooth_k=False)
    assert h2.k_codes.any()


def test_causal_first_row_is_first_value():
    N, d = 300, 128
    Q, K, V = head(N, d, seed=4)
    h = oracle.quantize_head(Q, K, V)
    O = oracle.attn_fwd([h], causal=True, scale=1 / np.sqrt(d), rows=[0])[0, 0]
    np.testing.assert_allclose(O, _deqV(h)[:, 0] * C2688, rtol=1e-13, atol=0)


def test_padding_rows_and_keys():
    """N not a multiple of 128: pad codes/scales are zero (reading c13) and padded keys are masked, so
    appending junk beyond N changes nothing."""
    N, d = 137, 64
    Q, K, V = head(N + 50, d, seed=5)
    h = oracle.quantize_head(Q[:N], K[:N], V[:N])
    assert not h.q_codes[N:].any() and not h.k_sf[N:].any() and not h.v_codes[:, N:].any()
    O = oracle.attn_fwd([h], causal=False, scale=0.125)[0]
    assert np.all(np.isfinite(O)) and O.shape == (N, d)


def test_row_sample_is_exact_subset():
    N, d = 384, 64
    Q, K, V = head(N, d, seed=6)
    h = oracle.quantize_head(Q, K, V)
    full = oracle.attn_fwd([h], causal=True, scale=0.125)[0]
    rows = np.array([0, 5, 127, 128, 300, 383])
    part = oracle.attn_fwd([h], causal=True, scale=0.125, rows=rows)[0]
    assert np.array_equal(full[rows], part)


def test_lse_matches_plain_logsumexp_without_quantization():
    N, d = 256, 64
    Q, K, V = head(N, d, seed=7)
    _, lse = oracle.attn_fwd_float(Q, K, V, causal=True, scale=0.125, bkv=128, want_lse=True)
    S = 0.125 * (Q.astype(np.float64) @ K.astype(np.float64).T)
    S = np.where(np.tril(np.ones_like(S, dtype=bool)), S, -np.inf)
    ref = np.log(np.exp(S - S.max(1, keepdims=True)).sum(1)) + S.max(1)
    np.testing.assert_allclose(lse, ref, rtol=1e-12, atol=1e-12)


def test_quantized_pipeline_accuracy_and_orderings():
    """Reported properties (not exact pins): the quantized output tracks full-precision attention, and the
    paper's orderings hold on this synthetic draw: two-level > direct (Tab1b), smoothing K > none
    (P:1225-1229)."""
    N, d = 512, 128
    Q, K, V = head(N, d, seed=8, dtype=torch.bfloat16)
    scale = 1 / np.sqrt(d)
    rows = np.arange(0, N, 4)
    ref = oracle.reference_attention(Q, K, V, causal=False, scale=scale, rows=rows)
    h = oracle.quantize_head(Q, K, V)
    m2 = oracle.accuracy_metrics(ref, oracle.attn_fwd([h], causal=False, scale=scale, rows=rows)[0])
    m1 = oracle.accuracy_metrics(ref, oracle.attn_fwd([h], causal=False, scale=scale, rows=rows,
                                                      p_mode=oracle.PMODE_DIRECT)[0])
    h0 = oracle.quantize_head(Q, K, V, smooth_k=False)
    m0 = oracle.accuracy_metrics(ref, oracle.attn_fwd([h0], causal=False, scale=scale, rows=rows)[0])
    assert m2["cos_sim"] > 0.9
    assert m2["l1"] <= m1["l1"] * 1.05
    assert m2["cos_sim"] > m0["cos_sim"]


def test_metrics_definitions():
    x = np.random.default_rng(0).standard_normal(100)
    assert oracle.accuracy_metrics(x, x) == {"cos_sim": pytest.approx(1.0), "l1": 0.0, "rmse": 0.0}
    m = oracle.accuracy_metrics(x, 2 * x)
    assert m["cos_sim"] == pytest.approx(1.0) and m["l1"] == pytest.approx(1.0)
