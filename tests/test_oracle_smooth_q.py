"""Pins for the oracle's smoothing Q (Alg1 L5 + the GEMV of L8; SageAttention2): q̄ of a 128-row
query tile against exact rational means, the closed form where Q - q̄ vanishes (S is then exactly the GEMV
q̄·K^T with the full-precision smoothed K), bitwise identity when q̄ = 0, and the accuracy gain the paper
attributes to smoothing Q on queries with a large shared component."""
from fractions import Fraction

import ml_dtypes
import numpy as np
import pytest
import torch
from scipy.special import softmax

import oracle
import synth


def _bf16_exact(x):
    return torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16).float().numpy()


@pytest.mark.parametrize("N", [128, 300, 5])
def test_qmean_is_the_exact_mean_of_the_tile_rows(N):
    """Integer-valued Q: q̄_i = fl32(exact mean over the tile's real rows) (reading c10 order, one rounding)."""
    d = 32
    rng = np.random.default_rng(N)
    Q = rng.integers(-1000, 1000, (N, d)).astype(np.float32)
    for tile in range((N + 127) // 128):
        r0, r1 = tile * 128, min(N, tile * 128 + 128)
        qm = oracle.qmean_tile(Q, tile)
        for c in range(d):
            exact = Fraction(int(Q[r0:r1, c].astype(np.int64).sum()), r1 - r0)
            assert qm[c] == np.float32(float(exact)), (tile, c)


def _deq(codes, sf):
    """Independent dequantization with ml_dtypes (E2M1 codes 0..15, E4M3 scale bytes), 16-blocks along cols."""
    vals = codes.astype(np.uint8).view(ml_dtypes.float4_e2m1fn).astype(np.float64)
    scales = sf.view(ml_dtypes.float8_e4m3fn).astype(np.float64)
    return vals * np.repeat(scales, 16, axis=1)


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("N,d", [(256, 64), (300, 128)])
def test_tile_constant_queries_reduce_to_the_gemv(N, d, causal):
    """Rows of Q equal inside each 128-row tile => Q - q̄ = 0 exactly => Q̂ = 0 and S = q̄_i·K_s^T, with K_s the
    full-precision smoothed K.  With P quantization off (p_mode NONE) O must be softmax(scale·S)·deq(V̂)."""
    _, K, V = (x.float().numpy() for x in synth.make_head(N, d, seed=3, dtype=torch.bfloat16))
    rng = np.random.default_rng(1)
    Q = np.zeros((N, d), np.float32)
    for t in range((N + 127) // 128):
        Q[t * 128:(t + 1) * 128] = _bf16_exact(rng.standard_normal(d) * 2)
    h = oracle.quantize_head(Q, K, V, smooth_q=True)
    assert not h.q_codes.any() and not h.q_sf.any()
    Ks = (K - oracle.kmean(K)).astype(np.float32)  # fl32(K - km), the K_j of Alg1 L8
    np.testing.assert_array_equal(h.ks[:N], Ks)
    scale = 1 / np.sqrt(d)
    O = oracle.attn_fwd([h], causal=causal, scale=scale, p_mode=oracle.PMODE_NONE)[0]
    S = scale * (Q.astype(np.float64) @ Ks.T.astype(np.float64))
    if causal:
        S = np.where(np.tril(np.ones_like(S, dtype=bool)), S, -np.inf)
    Vd = _deq(h.v_codes, h.v_sf)[:, :N].T  # [N][d]
    np.testing.assert_allclose(O, softmax(S, axis=1) @ Vd, rtol=1e-10, atol=1e-12)


def test_zero_mean_tiles_give_identical_results():
    """q̄ = 0 exactly (rows come in ± pairs inside every tile) => same codes, GEMV term 0 => bitwise equal O."""
    N, d = 256, 64
    q, K, V = (x.float().numpy() for x in synth.make_head(N, d, seed=4, dtype=torch.bfloat16))
    Q = np.concatenate([q[:64], -q[:64], q[64:128], -q[64:128]]).astype(np.float32)
    a = oracle.quantize_head(Q, K, V)
    b = oracle.quantize_head(Q, K, V, smooth_q=True)
    assert not b.q_mean.any()
    np.testing.assert_array_equal(a.q_codes, b.q_codes)
    np.testing.assert_array_equal(a.q_sf, b.q_sf)
    for causal in (False, True):
        oa = oracle.attn_fwd([a], causal=causal, scale=0.125)
        ob = oracle.attn_fwd([b], causal=causal, scale=0.125)
        np.testing.assert_array_equal(oa, ob)


def test_smoothing_q_improves_accuracy_on_offset_queries():
    """SageAttention2's motivation: a large component shared by the queries of a tile dominates the
    per-block scales and drowns the informative part in FP4 noise; subtracting q̄ removes it.  With such
    queries the smoothed pipeline must be closer to fp64 attention (paper metrics)."""
    N, d = 1024, 128
    q, K, V = (x.float().numpy() for x in synth.make_head(N, d, seed=6, dtype=torch.bfloat16))
    offset = np.random.default_rng(2).standard_normal(d).astype(np.float32) * 6
    Q = _bf16_exact(q + offset)
    rows = np.arange(0, N, 8, dtype=np.int32)
    scale = 1 / np.sqrt(d)
    ref = oracle.reference_attention(Q, K, V, causal=False, scale=scale, rows=rows)
    m0 = oracle.accuracy_metrics(ref, oracle.attn_fwd([oracle.quantize_head(Q, K, V)], causal=False, scale=scale,
                                                      rows=rows)[0])
    m1 = oracle.accuracy_metrics(ref, oracle.attn_fwd([oracle.quantize_head(Q, K, V, smooth_q=True)], causal=False,
                                                      scale=scale, rows=rows)[0])
    print("without / with smoothing Q:", m0, m1)
    assert m1["cos_sim"] > m0["cos_sim"] and m1["l1"] < m0["l1"]
