"""Pins for the SageBwd oracle (NEXT #3; §4, Algorithm 2 forward P:241-277, Algorithm 3 backward
P:283-331, ψ P:279-282): ψ's invariants, the Q = 0 closed form of the forward, forward accuracy against fp64
attention, the zero-gradient case, and the backward against fp64 autograd of plain softmax attention (the
gradients Alg 3 approximates)."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth


def test_psi_examples():
    q, s = oracle.sb_psi(np.array([1.0, -2.0, 127.0, 0.4], np.float32))
    assert s == 1.0 and q.tolist() == [1, -2, 127, 0]
    q, s = oracle.sb_psi(np.zeros(8, np.float32))
    assert s == 0.0 and not q.any()
    q, s = oracle.sb_psi(np.array([0.5, -0.25], np.float32))  # s = fl32(0.5/127): codes 127, -64 (63.5 -> 64, RNE)
    assert q.tolist() == [127, -64]


def test_psi_invariants():
    """|code| <= 127, the block max maps to ±127, every element within half a step (+1 ulp of the product) of
    its code, sign kept, s = fl32(amax·fl32(1/127))."""
    rng = np.random.default_rng(0)
    for _ in range(300):
        x = (rng.standard_normal(rng.integers(1, 600)) * 10.0 ** rng.uniform(-6, 6)).astype(np.float32)
        q, s = oracle.sb_psi(x)
        amax = np.abs(x).max()
        assert s == np.float32(amax) * np.float32(1.0 / 127.0)
        assert np.abs(q.astype(np.int32)).max() == 127
        assert np.abs(q[np.argmax(np.abs(x))]) == 127
        err = np.abs(x.astype(np.float64) / s - q)
        assert err.max() <= 0.5 + 1e-5
        assert np.all((q == 0) | (np.sign(q) == np.sign(x)))


@pytest.mark.parametrize("causal", [False, True])
def test_forward_zero_query_closed_form(causal):
    """Q = 0 -> S = 0, P̃ = 1, s_P = fl32(1/127), P̂ = 127: O = 127·fl32(1/127)·(running) mean of deq(V̂)."""
    N, d = 300, 64
    _, K, V = (x.float().numpy() for x in synth.make_head(N, d, seed=2, dtype=torch.bfloat16))
    h = oracle.sb_quantize_head(np.zeros((N, d), np.float32), K, V)
    O, lse = oracle.sb_attn_fwd([h], causal=causal, scale=0.125, want_lse=True)
    Vd = h.v[:N].astype(np.float64) * np.repeat(h.sv, 128)[:N, None]
    c = 127.0 * float(np.float32(1.0) / np.float32(127.0))
    cnt = np.arange(1, N + 1) if causal else np.full(N, N)
    ref = (np.cumsum(Vd, axis=0) / cnt[:, None]) if causal else np.broadcast_to(Vd.mean(0), (N, d))
    np.testing.assert_allclose(O[0], c * ref, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(lse[0], np.log(cnt), rtol=1e-12)


@pytest.mark.parametrize("causal", [False, True])
def test_forward_accuracy_vs_fp64(causal):
    """The paper's claim for 8-bit attention: close to full precision (paper metrics).  Inputs
    without the outlier channels (one INT8 scale per 128 x d block is what Alg 2 specifies; a few x10 channels
    would dominate it)."""
    N, d = 512, 128
    Q, K, V = (x.float().numpy() for x in synth.make_head(N, d, seed=5, dtype=torch.bfloat16, outliers=False))
    scale = 1 / math.sqrt(d)
    h = oracle.sb_quantize_head(Q, K, V)
    O = oracle.sb_attn_fwd([h], causal=causal, scale=scale)[0]
    ref = oracle.reference_attention(Q, K, V, causal=causal, scale=scale)
    m = oracle.accuracy_metrics(ref, O)
    print(m)
    assert m["cos_sim"] > 0.9995 and m["l1"] < 0.03


def _fwd_bwd_fp64(Q, K, V, dO, causal, scale):
    q, k, v = (torch.tensor(x, dtype=torch.float64, requires_grad=True) for x in (Q, K, V))
    S = scale * q @ k.T
    if causal:
        S = S.masked_fill(torch.triu(torch.ones_like(S, dtype=torch.bool), 1), float("-inf"))
    O = torch.softmax(S, dim=1) @ v
    O.backward(torch.tensor(dO, dtype=torch.float64))
    return O.detach().numpy(), q.grad.numpy(), k.grad.numpy(), v.grad.numpy()


@pytest.mark.parametrize("causal", [False, True])
def test_backward_against_fp64_autograd(causal):
    """Alg 3's gradients vs the exact gradients of softmax attention (torch autograd, fp64) on the same
    16-bit inputs: the INT8 quantization of four of the five matmuls only adds noise (the paper's Tab1c
    reports dQ CosSim ~0.997 with dO·Vᵀ in FP16).  A transposed operand, a wrong sign, a missing softmax scale
    or dropping the D_i term fails this by a wide margin."""
    N, d = 384, 64
    Q, K, V = (x.float().numpy() for x in synth.make_head(N, d, seed=8, dtype=torch.bfloat16, outliers=False))
    dO = torch.randn(N, d, generator=torch.Generator().manual_seed(3)).to(torch.bfloat16).float().numpy()
    scale = 1 / math.sqrt(d)
    h = oracle.sb_quantize_head(Q, K, V)
    O, lse = oracle.sb_attn_fwd([h], causal=causal, scale=scale, want_lse=True)
    O32 = O[0].astype(np.float32)
    dQ, dK, dV = oracle.sb_attn_bwd(h, V, O32, dO, lse[0].astype(np.float32), causal=causal, scale=scale)
    _, gQ, gK, gV = _fwd_bwd_fp64(Q, K, V, dO, causal, scale)
    for name, got, want in (("dQ", dQ, gQ), ("dK", dK, gK), ("dV", dV, gV)):
        m = oracle.accuracy_metrics(want, got)
        print(name, m)
        assert m["cos_sim"] > 0.995 and m["l1"] < 0.1, (name, m)


def test_backward_zero_upstream_gradient():
    N, d = 200, 64
    Q, K, V = (x.float().numpy() for x in synth.make_head(N, d, seed=1, dtype=torch.bfloat16))
    h = oracle.sb_quantize_head(Q, K, V)
    O, lse = oracle.sb_attn_fwd([h], causal=True, scale=0.125, want_lse=True)
    g = oracle.sb_attn_bwd(h, V, O[0].astype(np.float32), np.zeros((N, d), np.float32),
                           lse[0].astype(np.float32), causal=True, scale=0.125)
    for x in g:
        assert not x.any()


def test_smooth_k_correction_term_of_dq():
    """Alg3 L10's '+ rowsum(dS)·K_m' (the backward of smooth-K): with O = 0 given, D_i = 0 so rowsum(dS) =
    Σ_j P_ij·dP_ij ≠ 0, and shifting K by a constant row vector c (which only moves K_m, not the quantized
    smoothed K) must move dQ by exactly scale·rowsum(dS)·c while dK, dV stay put."""
    N, d = 256, 64
    Q, K, V = (x.float().numpy() for x in synth.make_head(N, d, seed=4, dtype=torch.bfloat16, outliers=False))
    K = np.clip(np.rint(K * 8) / 8, -8, 8).astype(np.float32)  # N = 256, K on a 1/8 grid: K - K_m is exact
    dO = torch.randn(N, d, generator=torch.Generator().manual_seed(9)).to(torch.bfloat16).float().numpy()
    h0 = oracle.sb_quantize_head(Q, K, V)
    h1 = oracle.sb_quantize_head(Q, K + np.float32(1.0), V)
    np.testing.assert_array_equal(h0.k, h1.k)
    np.testing.assert_array_equal(h0.sk, h1.sk)
    assert np.allclose(h1.km - h0.km, 1.0)
    Z = np.zeros((N, d), np.float32)
    O, lse = oracle.sb_attn_fwd([h0], causal=False, scale=0.125, want_lse=True)
    L = lse[0].astype(np.float32)
    g0 = oracle.sb_attn_bwd(h0, V, Z, dO, L, causal=False, scale=0.125)
    g1 = oracle.sb_attn_bwd(h1, V, Z, dO, L, causal=False, scale=0.125)
    np.testing.assert_array_equal(g0[1], g1[1])
    np.testing.assert_array_equal(g0[2], g1[2])
    # P and dP from the decoded codes (independent of the oracle's loops): rowsum(dS) = Σ_j P_ij dP_ij
    S = (h0.q[:N].astype(np.float64) * np.repeat(h0.sq, 128)[:N, None]) @ \
        (h0.k[:N].astype(np.float64) * np.repeat(h0.sk, 128)[:N, None]).T
    P = np.exp(0.125 * S - L[:, None].astype(np.float64)).astype(np.float32).astype(np.float64)
    rs = (P * (dO.astype(np.float64) @ V.astype(np.float64).T)).astype(np.float32).astype(np.float64).sum(1)
    diff = g1[0] - g0[0]
    want = 0.125 * rs[:, None] * (h1.km - h0.km)[None, :].astype(np.float64)
    np.testing.assert_allclose(diff, want, rtol=1e-5, atol=1e-6 * np.abs(want).max())
