"""Pins for φ (Eq. 1), the smoothing-K mean (Alg1 L2), FP4MM (Eq. 3) and the
two-level P quantization (§3.2) in the oracle.  References are the paper's printed values,
SPEC's worked examples, exact rational arithmetic, scale invariances and independent library decodes."""
import json
import os
from fractions import Fraction

import ml_dtypes
import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
E2M1 = np.array([0, 0.5, 1, 1.5, 2, 3, 4, 6, -0.0, -0.5, -1, -1.5, -2, -3, -4, -6])


def lib_decode_e2m1(codes):
    """Independent decode through ml_dtypes (library routine)."""
    return np.asarray(codes, np.uint8).view(ml_dtypes.float4_e2m1fn).astype(np.float64)


def lib_decode_e4m3(codes):
    return np.asarray(codes, np.uint8).view(ml_dtypes.float8_e4m3fn).astype(np.float64)


@pytest.mark.parametrize("name", ["all_six", "three_then_zeros"])
def test_phi_spec_examples(name):
    ex = GOLD["phi_examples"][name]
    codes, sc = oracle.phi_nvfp4(ex["x"])
    assert oracle.e4m3_decode(sc) == ex["scale"]
    assert np.array_equal(lib_decode_e2m1(codes) * ex["scale"], np.array(ex["deq"], np.float64))


def test_phi_zero_block_fixed_point():
    codes, sc = oracle.phi_nvfp4(np.zeros(16))
    assert sc == 0 and not codes.any()


def test_phi_invariants_random():
    """|code| <= 6, scale <= 448, scale code never NaN, and every element within half the local E2M1
    gap (times s) of x, except elements whose magnitude exceeds 6 s (saturated), SURVEY c2."""
    rng = np.random.default_rng(3)
    for trial in range(3000):
        x = (rng.standard_normal(16) * 10.0 ** rng.uniform(-4, 3)).astype(np.float32)
        if trial % 7 == 0:
            x[rng.integers(16)] *= 50  # an outlier inside the block
        codes, sc = oracle.phi_nvfp4(x)
        s = lib_decode_e4m3([sc])[0]
        assert 0 < s <= 448 or (s == 0 and np.abs(x).max() * np.float32(1 / 6) <= 2.0 ** -10)
        deq = lib_decode_e2m1(codes) * s
        assert np.all(np.abs(lib_decode_e2m1(codes)) <= 6)
        for xi, di in zip(x.astype(np.float64), deq):
            if abs(xi) >= 6 * s:
                assert abs(di) == 6 * s
                continue
            mags = np.abs(E2M1[:8]) * s
            k = np.searchsorted(mags, abs(xi))
            lo, hi = mags[max(k - 1, 0)], mags[min(k, 7)]
            assert abs(abs(di) - abs(xi)) <= (hi - lo) / 2 * (1 + 1e-6) + 1e-30


def test_phi_power_of_two_scaling_invariance():
    """φ(2^k x): same element codes, scale multiplied by 2^k, while s stays a normal E4M3 value."""
    rng = np.random.default_rng(4)
    for _ in range(500):
        x = rng.standard_normal(16).astype(np.float32)
        c0, s0 = oracle.phi_nvfp4(x)
        for k in (-3, -1, 1, 2, 4):
            c1, s1 = oracle.phi_nvfp4(x * np.float32(2.0**k))
            v0, v1 = lib_decode_e4m3([s0])[0], lib_decode_e4m3([s1])[0]
            if 2.0**-6 <= v0 * 2.0**k <= 240 and v0 >= 2.0**-6:
                assert np.array_equal(c0, c1)
                assert v1 == v0 * 2.0**k


def test_phi_scale_uses_one_sixth_multiply():
    """Reading c3 regression vector: amax = 0x3F63FFFF gives scale code 0x22 via fl32(amax*fl32(1/6))
    (0x21 via true division)."""
    amax = np.array([0x3F63FFFF], np.uint32).view(np.float32)[0]
    x = np.zeros(16, np.float32)
    x[5] = amax
    _, sc = oracle.phi_nvfp4(x)
    assert sc == 0x22
    # by hand: fl32(amax*fl32(1/6)) is exactly the midpoint 0.1484375 between codes 0x21 and 0x22 -> even
    prod = np.float32(amax) * np.float32(1.0 / 6.0)
    assert float(prod) == 0.1484375


def test_kmean_closed_forms():
    rng = np.random.default_rng(5)
    const = rng.standard_normal(64).astype(np.float32)
    K = np.tile(const, (300, 1))
    assert np.array_equal(oracle.kmean(K), const)  # constant columns -> exact mean
    Kint = rng.integers(-1000, 1000, size=(1000, 128)).astype(np.float32)
    exact = np.array([float(Fraction(int(Kint[:, c].sum()), 1000)) for c in range(128)], np.float64)
    assert np.array_equal(oracle.kmean(Kint), exact.astype(np.float32))


def test_fp4mm_spec_example():
    sixes, s6 = oracle.phi_nvfp4(np.full(16, 6.0))
    ones, s1 = oracle.phi_nvfp4(np.full(16, 1.0))
    C = oracle.fp4mm(sixes[None, :], np.array([[s6]]), ones[None, :], np.array([[s1]]))
    deq_ones = lib_decode_e2m1(ones)[0] * lib_decode_e4m3([s1])[0]
    assert C[0, 0] == GOLD["fp4mm_example"]["value"] * deq_ones  # 96 x (deq of 1.0 = 1.03125)
    exact_ones = np.zeros(16, np.uint8) + 0x2  # code of 1.0 with scale 1.0 (0x38)
    C2 = oracle.fp4mm(sixes[None, :], np.array([[s6]]), exact_ones[None, :], np.array([[0x38]]))
    assert C2[0, 0] == GOLD["fp4mm_example"]["value"]


def test_fp4mm_exact_against_rationals_and_library_matmul():
    rng = np.random.default_rng(6)
    M, N, K = 8, 6, 128
    a = rng.integers(0, 16, size=(M, K)).astype(np.uint8)
    b = rng.integers(0, 16, size=(N, K)).astype(np.uint8)
    sa = rng.integers(0, 0x7E, size=(M, K // 16)).astype(np.uint8)
    sb = rng.integers(0, 0x7E, size=(N, K // 16)).astype(np.uint8)
    C = oracle.fp4mm(a, sa, b, sb)
    A = lib_decode_e2m1(a) * np.repeat(lib_decode_e4m3(sa), 16, axis=1)
    B = lib_decode_e2m1(b) * np.repeat(lib_decode_e4m3(sb), 16, axis=1)
    np.testing.assert_allclose(C, A @ B.T, rtol=1e-12, atol=1e-300)
    for m in range(3):
        for n in range(3):
            exact = sum(Fraction(float(A[m, k])) * Fraction(float(B[n, k])) for k in range(K))
            assert Fraction(float(C[m, n])) == exact  # fp64 FP4MM is exact (bit-count argument)


def test_dequant_matches_library_decode():
    rng = np.random.default_rng(7)
    codes = rng.integers(0, 16, size=(5, 64)).astype(np.uint8)
    sf = rng.integers(0, 0x7E, size=(5, 4)).astype(np.uint8)
    ref = lib_decode_e2m1(codes) * np.repeat(lib_decode_e4m3(sf), 16, axis=1)
    assert np.array_equal(oracle.dequant(codes, sf), ref)


def test_two_level_spec_examples():
    g = GOLD["two_level"]
    P = np.zeros(128, np.float32)
    P[3] = 2688.0
    s, codes, sf = oracle.two_level_row(P)
    assert s == g["rowmax_2688_gives_sP1"]
    P = np.random.default_rng(8).uniform(0, 1, 128).astype(np.float32)
    P[17] = 1.0
    s, codes, sf = oracle.two_level_row(P)
    assert s == np.float32(1.0) / np.float32(2688.0)
    assert abs(s * 2688 - g["rowmax_1_gives_sP1_times_2688"]) < 1e-6
    # the max element maps to 2688 -> block scale 448 (0x7E) and code 6 (0x7)
    assert sf[17 // 16] == 0x7E and codes[17] == 0x7


def test_two_level_reconstruction_and_benefit():
    """P̃ ≈ P̂2 s_P2 s_P1 within φ's bound, and two-level beats direct φ(P̃) on softmax-like rows
    (appendix E2 < E1; Tab1b ordering)."""
    rng = np.random.default_rng(9)
    err2 = err1 = 0.0
    for _ in range(200):
        logits = rng.standard_normal(128) * rng.uniform(0.5, 4)
        P = np.exp(logits - logits.max()).astype(np.float32) * np.float32(rng.uniform(0.01, 1))
        s1, c, sf = oracle.two_level_row(P)
        rec = lib_decode_e2m1(c) * np.repeat(lib_decode_e4m3(sf), 16) * s1
        blockmax = np.repeat(P.reshape(8, 16).max(1), 16).astype(np.float64)
        assert np.all(np.abs(rec - P) <= blockmax / 6 * 1.07 + 1e-30)
        err2 += np.abs(rec - P).sum()
        _, cd, sfd = oracle.two_level_row(P, oracle.PMODE_DIRECT)
        rec1 = lib_decode_e2m1(cd) * np.repeat(lib_decode_e4m3(sfd), 16)
        err1 += np.abs(rec1 - P).sum()
    assert err2 < err1
