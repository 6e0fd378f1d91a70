"""Pins for the oracle's PMODE_QSUM (SURVEY §8(f) NEXT #2 throughput variant, reading n2): the paper's
two-level P quantization (Alg1 L10) unchanged, but l accumulates the quantized P (s_P1·Σ deq(P̂2)) — the value the
GPU reads from the tensor core (P̂2 times a ones column) — instead of the unquantized P̃ (reading c9).  Pinned by
closed forms independent of the oracle's own arithmetic: the weights of every row then sum to exactly one, so a
constant V row comes back exactly and Q = 0 gives the plain running mean of deq(V̂) (no 2688·fl32(1/2688) factor);
the codes and scales it quantizes are the two-level mode's; and the accuracy sits with the paper's mode."""
import math

import ml_dtypes
import numpy as np
import pytest
import torch

import oracle
import synth


def _deq(codes, sf, G=16):
    vals = codes.astype(np.uint8).view(ml_dtypes.float4_e2m1fn).astype(np.float64)
    return vals * np.repeat(sf.view(ml_dtypes.float8_e4m3fn).astype(np.float64), G, axis=1)


def _head(N, d, seed):
    return [x.float().numpy() for x in synth.make_head(N, d, seed=seed, dtype=torch.bfloat16)]


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("N,d", [(1, 64), (200, 64), (300, 128)])
def test_constant_values_come_back_exactly(N, d, causal):
    """V rows all equal to one vector c: O_i = Σ_k p̂_k c / Σ_k p̂_k = deq(c) for every query, exactly — the weights
    are normalised by their own sum.  (The paper's mode divides by Σ P̃ instead and misses by the quantization
    error of the row sum.)"""
    Q, K, _ = _head(N, d, seed=N + d)
    c = np.random.default_rng(1).standard_normal(d).astype(np.float32)
    V = np.tile(c, (N, 1))
    h = oracle.quantize_head(Q, K, V)
    cdeq = _deq(h.v_codes, h.v_sf)[:, 0]  # every token of a channel has the same code and block scale
    O = oracle.attn_fwd([h], causal=causal, scale=1 / math.sqrt(d), p_mode=oracle.PMODE_QSUM)[0]
    np.testing.assert_allclose(O, np.broadcast_to(cdeq, O.shape), rtol=1e-12, atol=1e-12)
    if N > 1:
        O2 = oracle.attn_fwd([h], causal=causal, scale=1 / math.sqrt(d))[0]
        assert np.abs(O2 - cdeq).max() > 1e-6  # the two modes really differ


@pytest.mark.parametrize("causal", [False, True])
def test_zero_scores_plain_running_mean(causal):
    """Q = 0: P̃2 = 2688 -> code 6, scale 448, deq(P̂2) = 2688 = P̃2, so O is exactly the (causal) running mean of
    deq(V̂) (the two-level mode has the extra factor 2688·fl32(1/2688) there)."""
    N, d = 300, 64
    _, K, V = _head(N, d, seed=2)
    h = oracle.quantize_head(np.zeros((N, d), np.float32), K, V)
    O = oracle.attn_fwd([h], causal=causal, scale=0.125, p_mode=oracle.PMODE_QSUM)[0]
    Vd = _deq(h.v_codes, h.v_sf)[:, :N].T
    ref = (np.cumsum(Vd, 0) / np.arange(1, N + 1)[:, None]) if causal else np.broadcast_to(Vd.mean(0), (N, d))
    np.testing.assert_allclose(O, ref, rtol=1e-12, atol=1e-13)


def test_same_numerator_as_two_level():
    """Only l changes: O_qsum · l_qsum = O_two · l_two row by row (the same P̂2 codes, scales and s_P1 reach the PV
    product), checked through the LSE: l = exp(lse - scale·m), and m is the same in both modes."""
    N, d = 400, 128
    Q, K, V = _head(N, d, seed=9)
    h = oracle.quantize_head(Q, K, V)
    sc = 1 / math.sqrt(d)
    O2, lse2 = oracle.attn_fwd([h], causal=True, scale=sc, want_lse=True)
    Oq, lseq = oracle.attn_fwd([h], causal=True, scale=sc, p_mode=oracle.PMODE_QSUM, want_lse=True)
    num2 = O2[0] * np.exp(lse2[0])[:, None]
    numq = Oq[0] * np.exp(lseq[0])[:, None]
    np.testing.assert_allclose(numq, num2, rtol=1e-9, atol=1e-9 * np.abs(num2).max())
    # the two row sums differ by the quantization of P: Σ deq(P̂2) < Σ P̃2 on average (values far below their
    # block's max round to 0 on the E2M1 grid), a few percent on this data, more on the first causal rows
    dl = (lse2 - lseq)[0]
    print("lse(two-level) - lse(qsum): median %.4f max %.4f" % (np.median(dl), np.abs(dl).max()))
    assert np.median(dl) > 0 and np.abs(dl).max() < 0.25


def test_accuracy_against_fp64_with_the_paper_mode():
    """Reported: CosSim / rel-L1 against plain fp64 attention, next to the paper's two-level mode (the variant is
    meant to keep the paper's accuracy)."""
    N, d = 1024, 128
    Q, K, V = _head(N, d, seed=5)
    rows = np.arange(0, N, 4, dtype=np.int32)
    ref = oracle.reference_attention(Q, K, V, causal=False, scale=1 / math.sqrt(d), rows=rows)
    h = oracle.quantize_head(Q, K, V)
    m = {pm: oracle.accuracy_metrics(ref, oracle.attn_fwd([h], causal=False, scale=1 / math.sqrt(d), rows=rows,
                                                            p_mode=pm)[0])
         for pm in (oracle.PMODE_TWO_LEVEL, oracle.PMODE_QSUM)}
    print("two-level / qsum vs fp64:", m)
    a, b = m[oracle.PMODE_TWO_LEVEL], m[oracle.PMODE_QSUM]
    assert b["cos_sim"] > a["cos_sim"] - 2e-3 and b["l1"] < a["l1"] * 1.1
