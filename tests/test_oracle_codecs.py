"""Pins for the oracle's E2M1 / E4M3 codecs (readings c1-c2).

Each check compares the oracle with something other than itself: the value table and counts the
paper prints (tests/golden/paper_values.json), SPEC's worked rounding examples, and the independent
ml_dtypes / torch float8 conversions (library routines implementing IEEE-style RNE on these formats).
"""
import json
import os

import ml_dtypes
import numpy as np
import pytest
import torch

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_e2m1_value_table_matches_paper():
    vals = oracle.e2m1_table()
    assert sorted(set(vals.tolist())) == GOLD["e2m1_values"]["values"]
    assert len(oracle.enumerate_values("e2m1", -6, 6)) == GOLD["e2m1_values"]["distinct_count"]
    assert vals.max() == 6.0


@pytest.mark.parametrize("x,want", GOLD["e2m1_rounding"]["cases"])
def test_e2m1_spec_examples(x, want):
    assert oracle.e2m1_decode(oracle.e2m1_encode(x)) == want


def test_e2m1_midpoints_ties_to_even():
    # midpoints between neighbouring magnitudes resolve to the even mantissa code (reading c1)
    mids = {0.25: 0.0, 0.75: 1.0, 1.25: 1.0, 1.75: 2.0, 2.5: 2.0, 3.5: 4.0, 5.0: 4.0}
    for x, want in mids.items():
        assert oracle.e2m1_decode(oracle.e2m1_encode(x)) == want
        assert oracle.e2m1_decode(oracle.e2m1_encode(-x)) == -want
    assert oracle.e2m1_encode(-0.2) == 0x8  # sign kept on underflow
    assert oracle.e2m1_encode(1e9) == 0x7  # saturation
    assert oracle.e2m1_encode(-1e9) == 0xF


def _probe_floats(rng, n_random=1 << 20):
    """Dense structured sample: every value near each e2m1/e4m3 midpoint +- 64 ulp, plus random bits."""
    pts = []
    tab4 = np.array([0, 0.5, 1, 1.5, 2, 3, 4, 6], np.float64)
    tab8 = np.array([oracle.e4m3_decode(c) for c in range(0x7F)])
    for tab in (tab4, tab8):
        mids = (tab[1:] + tab[:-1]) / 2
        for m in np.concatenate([tab, mids, [6.5, 7.0, 448.0, 456.0, 463.9, 2.0 ** -10]]):
            base = np.float32(m).view(np.uint32).astype(np.int64)
            pts.append((base + np.arange(-64, 65)).clip(0, 0x7F7FFFFF).astype(np.uint32).view(np.float32))
    bits = rng.integers(0, 1 << 32, size=n_random, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    x = x[np.isfinite(x)]
    # also a log-uniform sample over the interesting range
    lg = (2.0 ** rng.uniform(-12, 10, size=n_random)).astype(np.float32)
    allp = np.concatenate(pts + [x, lg, -lg])
    return allp


def test_e2m1_matches_ml_dtypes():
    rng = np.random.default_rng(0)
    x = _probe_floats(rng)
    ours = oracle.e2m1_encode_array(x)
    ref = x.astype(ml_dtypes.float4_e2m1fn).view(np.uint8) & 0xF
    bad = np.nonzero(ours != ref)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first x={x[bad[:5]]} ours={ours[bad[:5]]} ref={ref[bad[:5]]}"


def test_e4m3_table_and_counts_match_paper():
    g = GOLD["e4m3"]
    tab = oracle.e4m3_table()
    assert np.nanmax(tab) == g["max_finite"]
    for v in g["exact"]:
        assert oracle.e4m3_decode(oracle.e4m3_encode(v)) == v
    assert len(oracle.enumerate_values("e4m3", 0.0, 0.167)) == g["count_0_to_0.167"]
    assert len(oracle.enumerate_values("e4m3", 0.0, 448.0)) == g["count_0_to_448"]


def test_e4m3_matches_ml_dtypes_and_torch_in_range():
    rng = np.random.default_rng(1)
    x = _probe_floats(rng)
    x = x[np.abs(x) < 464.0]  # libraries return NaN above the satfinite region; checked separately below
    ours = oracle.e4m3_encode_array(x)
    ref = x.astype(ml_dtypes.float8_e4m3fn).view(np.uint8)
    bad = np.nonzero(ours != ref)[0]
    assert bad.size == 0, f"{bad.size} mismatches vs ml_dtypes, first x={x[bad[:5]]}"
    tref = torch.from_numpy(x).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    assert np.array_equal(ours, tref)


def test_e4m3_satfinite_and_never_nan():
    # cuda_fp8.hpp satfinite semantics: every finite value above 448 clamps to 448 (0x7E)
    for x in [448.0, 450.0, 463.99, 464.0, 465.0, 1e6, 3.0e38]:
        assert oracle.e4m3_encode(x) == 0x7E
        assert oracle.e4m3_encode(-x) == 0xFE
    x = np.float32(2.0) ** -10  # half the smallest subnormal 2^-9: tie -> even (zero)
    assert oracle.e4m3_encode(float(x)) == 0x00
    codes = oracle.e4m3_encode_array(np.linspace(-500, 500, 100001, dtype=np.float32))
    assert not np.any((codes & 0x7F) == 0x7F)


def test_codec_roundtrip_identity():
    for c in range(16):
        v = oracle.e2m1_decode(c)
        if v != 0:
            assert oracle.e2m1_encode(v) == c
    for c in range(256):
        if (c & 0x7F) == 0x7F:
            continue
        v = oracle.e4m3_decode(c)
        if v != 0:
            assert oracle.e4m3_encode(v) == c
