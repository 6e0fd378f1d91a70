"""Pins for the oracle's decision-sensitivity bound (oracle_phi_sensitivity / attn_fwd(amb_delta=...)), the
test-infrastructure quantity the GPU parity tests use as the per-element allowance for P codes that sit
within the GPU's exp/accumulation error of a rounding midpoint.  It is pinned against brute
force: every perturbation of a block within the relative window must land inside the bound, the bound is
attained, and it vanishes when no decision is near a boundary."""
import ctypes
import math

import ml_dtypes
import numpy as np
import pytest

import oracle

MID = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0])  # E2M1 rounding midpoints (between 0, .5, 1, ..., 6)


def sens(x, fmt, delta):
    x = np.ascontiguousarray(x, np.float32)
    dq = np.zeros(x.shape[0], np.float64)
    oracle.lib().oracle_phi_sensitivity(x.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), x.shape[0], fmt,
                                        ctypes.c_double(delta), dq.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return dq


def deq(x, fmt):
    """φ then dequantize through an independent decode (ml_dtypes)."""
    codes, sc = (oracle.phi_mxfp4 if fmt else oracle.phi_nvfp4)(np.asarray(x, np.float32))
    vals = np.asarray(codes, np.uint8).view(ml_dtypes.float4_e2m1fn).astype(np.float64)
    s = 2.0 ** (int(sc) - 127) if fmt else np.asarray([sc], np.uint8).view(ml_dtypes.float8_e4m3fn).astype(np.float64)[0]
    if fmt and sc == 0 and not np.any(codes):
        s = 0.0
    return vals * s


def blocks(rng, G, n):
    out = []
    for i in range(n):
        x = rng.exponential(1.0, G).astype(np.float32) * np.float32(2.0 ** rng.integers(-6, 12))
        if i % 3 == 0:  # put some elements exactly on (or a hair off) a midpoint of the block's own scale
            s = float(oracle.e4m3_decode(oracle.phi_nvfp4(x)[1])) if G == 16 else 2.0 ** (int(oracle.phi_mxfp4(x)[1]) - 127)
            k = rng.integers(0, G, 4)
            x[k] = (MID[rng.integers(0, 7, 4)] * s * (1 + rng.choice([0.0, 3e-6, -3e-6], 4))).astype(np.float32)
            x[int(np.argmax(x))] = max(x.max(), np.float32(5.9 * s))  # keep the block scale in place
        out.append(x)
    return out


@pytest.mark.parametrize("fmt,G", [(0, 16), (1, 32)])
def test_sensitivity_covers_brute_force_perturbations(fmt, G):
    rng = np.random.default_rng(11 + fmt)
    delta = 1e-5
    hit = 0
    for x in blocks(rng, G, 120):
        dq = sens(x, fmt, delta)
        base = deq(x, fmt)
        spread = np.zeros(G)
        for _ in range(60):
            eps = rng.uniform(-delta, delta, G) * rng.choice([0.0, 1.0], G, p=[0.3, 0.7])
            xp = (x.astype(np.float64) * (1 + eps)).astype(np.float32)
            dv = np.abs(deq(xp, fmt) - base)
            assert np.all(dv <= dq * (1 + 1e-12) + 1e-300), (x, xp, dq)
            spread = np.maximum(spread, dv)
        hit += int(np.any(spread > 0))
    assert hit > 10  # the constructed near-midpoint blocks really do flip, and the bound covered them


@pytest.mark.parametrize("fmt,G", [(0, 16), (1, 32)])
def test_sensitivity_zero_away_from_boundaries_and_at_delta_zero(fmt, G):
    rng = np.random.default_rng(5)
    for x in blocks(rng, G, 60):
        assert not sens(x, fmt, 0.0).any()
    # values at exactly representable points y·s (NVFP4: amax = 6s; MXFP4: amax = 4s, because amax/6 = s would
    # itself sit on the power-of-two boundary of the round-up scale rule)
    top = 6 if fmt == 0 else 4
    x = np.array([top, 4, 3, 2, 1, 0.5, 0, 1.5] * (G // 8), np.float32) * np.float32(2.0 ** -3)
    assert not sens(x, fmt, 1e-5).any()


def test_sensitivity_attained_at_a_midpoint():
    s = 2.0 ** -2
    x = np.full(16, 0.0, np.float32)
    x[0] = 6 * s  # amax -> scale exactly s (E4M3 exact)
    x[1] = 2.5 * s  # midpoint between 2 and 3: RNE gives 2, a relative +delta gives 3
    dq = sens(x, 0, 1e-6)
    assert dq[1] == pytest.approx(1.0 * s) and dq[2:].sum() == 0.0


def test_attention_amb_is_zero_at_delta_zero_monotone_and_leaves_o_unchanged():
    rng = np.random.default_rng(3)
    N, d = 260, 64
    Q, K, V = (rng.standard_normal((N, d)).astype(np.float32) for _ in range(3))
    h = oracle.quantize_head(Q, K, V)
    sc = 1 / math.sqrt(d)
    for p_mode in (oracle.PMODE_TWO_LEVEL, oracle.PMODE_DIRECT, oracle.PMODE_LAZY):
        O = oracle.attn_fwd([h], causal=True, scale=sc, p_mode=p_mode)
        O0, _, a0 = oracle.attn_fwd([h], causal=True, scale=sc, p_mode=p_mode, amb_delta=0.0)
        assert np.array_equal(O, O0) and not a0.any()
        prev = a0
        for dl in (1e-6, 1e-5, 1e-4, 1e-3):
            O1, _, a1 = oracle.attn_fwd([h], causal=True, scale=sc, p_mode=p_mode, amb_delta=dl)
            assert np.array_equal(O, O1)
            assert np.all(a1 >= prev - 1e-15)
            prev = a1
        assert prev.any()
