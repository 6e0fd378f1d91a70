"""Pins for the oracle's MXFP4 ablation (P:129 / Tab1a: 1x32 blocks, E8M0 scales; reading: the scale is the
smallest power of two >= amax/6): φ against its definition with an independent E2M1 decode, the
closed form of the quantized pipeline at S = 0, and the paper's data-type ordering NVFP4 > MXFP4."""
import math

import ml_dtypes
import numpy as np
import pytest
import torch

import oracle
import synth


def _e2m1(codes):
    return np.asarray(codes, np.uint8).view(ml_dtypes.float4_e2m1fn).astype(np.float64)


def test_phi_mxfp4_examples():
    codes, sc = oracle.phi_mxfp4(np.full(32, 6.0, np.float32))
    assert sc == 127 and (codes == 7).all()  # s = 1, E2M1 code 7 = 6.0
    x = np.zeros(32, np.float32)
    x[0] = 3.0
    codes, sc = oracle.phi_mxfp4(x)
    assert sc == 126 and codes[0] == 7 and not codes[1:].any()  # s = 0.5, 3 / 0.5 = 6
    codes, sc = oracle.phi_mxfp4(np.zeros(32, np.float32))
    assert sc == 0 and not codes.any()


def test_phi_mxfp4_against_its_definition():
    rng = np.random.default_rng(0)
    for trial in range(2000):
        x = (rng.standard_normal(32) * 10.0 ** rng.uniform(-3, 3)).astype(np.float32)
        codes, sc = oracle.phi_mxfp4(x)
        p = int(sc) - 127
        s32 = np.float32(np.abs(x).max()) * np.float32(1.0 / 6.0)
        assert 2.0 ** p >= s32 > 2.0 ** (p - 1)  # smallest power of two >= amax/6
        y = (x.astype(np.float64) / 2.0 ** p).astype(np.float32)  # exact: power-of-two scale
        want = y.astype(ml_dtypes.float4_e2m1fn).astype(np.float64)  # RNE, satfinite (library routine)
        np.testing.assert_array_equal(_e2m1(codes), want)


@pytest.mark.parametrize("causal", [False, True])
def test_zero_scores_closed_form_mxfp4(causal):
    """Q = 0 => S = 0 => P̃ = 1, s_P1 = fl32(1/2688), P̃2 = 2688 -> E8M0 scale 512 (smallest 2^p >= 448),
    E2M1(5.25) = 6.0 (code 7) -> deq 3072: O_i = mean_{j visible} deq(V̂)_j * 3072 * fl32(1/2688)."""
    N, d = 300, 64
    _, K, V = (x.float().numpy() for x in synth.make_head(N, d, seed=2, dtype=torch.bfloat16))
    Q = np.zeros((N, d), np.float32)
    h = oracle.quantize_head(Q, K, V, fmt=oracle.FMT_MXFP4)
    O = oracle.attn_fwd([h], causal=causal, scale=1 / math.sqrt(d))[0]
    Vd = oracle.dequant_fmt(h.v_codes, h.v_sf, oracle.FMT_MXFP4)[:, :N].T
    c = 3072.0 * float(np.float32(1.0) / np.float32(2688.0))
    ref = (np.cumsum(Vd, axis=0) / np.arange(1, N + 1)[:, None]) if causal else np.broadcast_to(Vd.mean(0), (N, d))
    np.testing.assert_allclose(O, ref * c, rtol=1e-12, atol=1e-12)


def test_nvfp4_is_more_accurate_than_mxfp4():
    """Tab1a: NVFP4 (E4M3 scales per 16) beats MXFP4 (E8M0 per 32) in CosSim / L1 vs fp64."""
    N, d = 1024, 128
    Q, K, V = (x.float().numpy() for x in synth.make_head(N, d, seed=9, dtype=torch.bfloat16))
    rows = np.arange(0, N, 4, dtype=np.int32)
    ref = oracle.reference_attention(Q, K, V, causal=False, scale=1 / math.sqrt(d), rows=rows)
    m = {}
    for fmt in (oracle.FMT_NVFP4, oracle.FMT_MXFP4):
        o = oracle.attn_fwd([oracle.quantize_head(Q, K, V, fmt=fmt)], causal=False, scale=1 / math.sqrt(d), rows=rows)
        m[fmt] = oracle.accuracy_metrics(ref, o[0])
    print("NVFP4 / MXFP4:", m)
    assert m[oracle.FMT_NVFP4]["cos_sim"] > m[oracle.FMT_MXFP4]["cos_sim"]
    assert m[oracle.FMT_NVFP4]["l1"] < m[oracle.FMT_MXFP4]["l1"]
