"""GPU parity of the MXFP4 data-type ablation (Tab1a; NEXT #4): the quantizer's E2M1 codes and
UE8M0 scales (1x32 blocks, scale = smallest power of two >= amax/6, reading m1) BIT-EXACT against
oracle.quantize_head(fmt=FMT_MXFP4), and the scale_vec::2X attention path against the oracle's Algorithm 1 in
the MXFP4 format on the same codes (north_star tolerance).  Also the data-type ordering the paper reports:
NVFP4 more accurate than MXFP4, on the GPU path."""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_2505_11594_b200 as s3
import synth
from layout import decode_head
from parity import check, oracle_attention

pytestmark = pytest.mark.gpu

MX = oracle.FMT_MXFP4


def _check_head(qkv, bh, Q, K, V, smooth_q=False):
    want = oracle.quantize_head(Q, K, V, smooth_q=smooth_q, fmt=MX)
    got = decode_head(qkv, bh)
    d = Q.shape[1]
    np.testing.assert_array_equal(got["km"], want.km)
    for name in ("q_codes", "k_codes", "v_codes", "q_sf", "k_sf"):
        g, w = got[name], getattr(want, name)
        bad = np.argwhere(g != w)
        assert bad.size == 0, f"{name}: {len(bad)} mismatches, first at {bad[:4].tolist()} got {g[tuple(bad[0])]} want {w[tuple(bad[0])]}"
    assert not got["sf_pad"].any()  # atom columns >= d/32 (d = 64) stay zero
    np.testing.assert_array_equal(got["v_sf_full"][:d], want.v_sf)
    assert not got["v_sf_full"][d:].any()
    if smooth_q:
        np.testing.assert_array_equal(got["q_mean"], want.q_mean)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("N", [1, 31, 32, 127, 129, 1000])
def test_mxfp4_quantize_bit_exact(dtype, d, N):
    B, H = 1, 2
    Q, K, V = synth.make_qkv(B, H, N, d, seed=N + d + 1, dtype=dtype, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V, fmt="mxfp4")
    torch.cuda.synchronize()
    for bh in range(B * H):
        _check_head(qkv, bh, *(x[0, bh].float().cpu().numpy() for x in (Q, K, V)))


def test_mxfp4_quantize_extreme_magnitudes():
    """Scales across the E8M0 range: rows scaled by powers of two from 2^-120 to 2^120 (bf16 keeps them exact),
    exact powers of two at the block amax (2^p = amax/6 boundary), zero blocks, subnormal bf16 inputs."""
    N, d = 256, 128
    g = torch.Generator().manual_seed(5)
    X = torch.randn(3, N, d, generator=g)
    e = torch.randint(-120, 121, (3, N, 1), generator=g).float()
    X = X * torch.exp2(e)
    X[0, :8] = 0.0                                  # all-zero blocks: scale byte 0, zero codes
    X[1, 8:16, :32] = 6.0 * torch.exp2(torch.arange(8).float() - 4)[:, None]  # amax/6 exactly a power of two
    X[2, 16:24] = torch.randn(8, d, generator=g) * 2.0 ** -133  # bf16 subnormals
    Q, K, V = (X[i].to(torch.bfloat16)[None, None].cuda() for i in range(3))
    qkv = s3.sage3_quantize_qkv(Q, K, V, fmt="mxfp4")
    torch.cuda.synchronize()
    _check_head(qkv, 0, *(x[0, 0].float().cpu().numpy() for x in (Q, K, V)))


@pytest.mark.parametrize("N,d", [(300, 64), (1000, 128)])
def test_mxfp4_quantize_smooth_q_bit_exact(N, d):
    Q, K, V = synth.make_qkv(1, 2, N, d, seed=N, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V, smooth_q=True, fmt="mxfp4")
    torch.cuda.synchronize()
    for bh in range(2):
        _check_head(qkv, bh, *(x[0, bh].float().cpu().numpy() for x in (Q, K, V)), smooth_q=True)


def oracle_heads(qkv, heads):
    out = []
    for bh in heads:
        g = decode_head(qkv, bh)
        h = oracle.QuantizedHead(qkv.N, qkv.d, fmt=MX)
        h.q_codes, h.k_codes, h.v_codes = g["q_codes"], g["k_codes"], g["v_codes"]
        h.q_sf, h.k_sf, h.v_sf = g["q_sf"], g["k_sf"], np.ascontiguousarray(g["v_sf_full"][: qkv.d])
        out.append(h)
    return out




@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("N", [1, 31, 127, 128, 300, 1024])
def test_mxfp4_attention_parity(N, d, causal):
    B, H = 1, 2
    Q, K, V = synth.make_qkv(B, H, N, d, seed=5 * N + d, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V, fmt="mxfp4")
    lse = torch.empty(B, H, N, dtype=torch.float32, device="cuda")
    O = s3.sage3_attn_fwd(qkv, causal=causal, lse=lse, out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref, ref_lse, amb, vmax = oracle_attention(oracle_heads(qkv, range(B * H)), causal=causal,
                                               scale=1 / math.sqrt(d))
    for bh in range(B * H):
        check(O[0, bh].cpu().numpy(), ref[bh], torch.float32, f"head {bh}", amb=amb[bh], vmax=vmax[bh])
    np.testing.assert_allclose(lse.cpu().numpy().reshape(B * H, N), ref_lse, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("causal", [False, True])
def test_mxfp4_zero_query_closed_form(causal):
    """Q = 0: P̃2 = 2688 -> UE8M0 scale 512, E2M1(5.25) = 6.0 -> every deq P̂2 = 3072, so O is the (causal) running
    mean of deq(V̂) times 3072·fl32(1/2688) (test_oracle_mxfp4's closed form, on the GPU)."""
    N, d = 384, 128
    _, K, V = synth.make_qkv(1, 1, N, d, seed=3, device="cuda")
    Q = torch.zeros_like(K)
    qkv = s3.sage3_quantize_qkv(Q, K, V, fmt="mxfp4")
    O = s3.sage3_attn_fwd(qkv, causal=causal, out_dtype=torch.float32)
    torch.cuda.synchronize()
    h = oracle_heads(qkv, [0])[0]
    Vd = oracle.dequant_fmt(h.v_codes, h.v_sf, MX)[:, :N].T
    c = 3072.0 * float(np.float32(1.0) / np.float32(2688.0))
    ref = (np.cumsum(Vd, axis=0) / np.arange(1, N + 1)[:, None]) if causal else np.broadcast_to(Vd.mean(0), (N, d))
    np.testing.assert_allclose(O[0, 0].cpu().numpy(), ref * c, rtol=2e-5, atol=2e-6)


def test_mxfp4_smooth_q_and_units():
    """The format switch composes with smoothing Q and with unit sub-ranges (bitwise equal rows)."""
    N, d = 700, 128
    Q, K, V = synth.make_qkv(1, 3, N, d, seed=21, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V, smooth_q=True, fmt="mxfp4")
    O = s3.sage3_attn_fwd(qkv, causal=True, out_dtype=torch.float32)
    O2 = torch.zeros_like(O)
    n = s3.n_units(qkv)
    for lo, hi in ((0, 5), (5, n)):
        s3.sage3_attn_fwd_units(qkv, O2, lo, hi, causal=True)
    torch.cuda.synchronize()
    assert torch.equal(O, O2)
    heads = [oracle.quantize_head(*(x[0, bh].float().cpu().numpy() for x in (Q, K, V)), smooth_q=True, fmt=MX)
             for bh in range(3)]
    rows = np.arange(0, N, 3, dtype=np.int32)
    ref, _, amb, vmax = oracle_attention(heads, causal=True, scale=1 / math.sqrt(d), rows=rows)
    for bh in range(3):
        check(O[0, bh].cpu().numpy()[rows], ref[bh], torch.float32, f"head {bh}", amb=amb[bh], vmax=vmax[bh])


def test_nvfp4_more_accurate_than_mxfp4_on_gpu():
    """Tab1a's ordering on the GPU path (CosSim up, rel-L1 down vs fp64 attention), paper-like inputs."""
    N, d = 4096, 128
    Q, K, V = synth.make_qkv(1, 1, N, d, seed=31, dtype=torch.bfloat16, device="cuda")
    rows = np.arange(0, N, 16, dtype=np.int32)
    ref = oracle.reference_attention(Q[0, 0].float().cpu().numpy(), K[0, 0].float().cpu().numpy(),
                                     V[0, 0].float().cpu().numpy(), causal=False, scale=1 / math.sqrt(d), rows=rows)
    m = {f: oracle.accuracy_metrics(ref, s3.attention(Q, K, V, fmt=f, out_dtype=torch.float32)[0, 0].cpu().numpy()[rows])
         for f in ("nvfp4", "mxfp4")}
    print("GPU NVFP4 / MXFP4:", m)
    assert m["nvfp4"]["cos_sim"] > m["mxfp4"]["cos_sim"] and m["nvfp4"]["l1"] < m["mxfp4"]["l1"]
