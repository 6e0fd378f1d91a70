"""GPU parity of sage3_quantize_qkv against oracle_quantize_head: codes, E4M3 scales and the smoothing-K
mean must be BIT-EXACT, including padded tails (N not a multiple of 16/128), both input
dtypes, both head dims and non-contiguous inputs.  Also the hardware E2M1/E4M3 converts against the
oracle codecs on a dense sample."""
import numpy as np
import pytest
import torch

import oracle
import paper_2505_11594_b200 as s3
import synth
from layout import decode_head

pytestmark = pytest.mark.gpu


def _check_head(qkv, bh, Q, K, V):
    N = Q.shape[0]
    want = oracle.quantize_head(Q, K, V)
    got = decode_head(qkv, bh)
    d = Q.shape[1]
    np.testing.assert_array_equal(got["km"], want.km)
    for name in ("q_codes", "k_codes", "v_codes", "q_sf", "k_sf"):
        g, w = got[name], getattr(want, name)
        bad = np.argwhere(g != w)
        assert bad.size == 0, f"{name}: {len(bad)} mismatches, first at {bad[:4].tolist()} got {g[tuple(bad[0])]} want {w[tuple(bad[0])]}"
    np.testing.assert_array_equal(got["v_sf_full"][:d], want.v_sf)
    assert not got["v_sf_full"][d:].any()


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("N", [1, 15, 16, 127, 128, 129, 1000])
def test_quantize_bit_exact(dtype, d, N):
    B, H = 1, 2
    Q, K, V = synth.make_qkv(B, H, N, d, seed=N + d, dtype=dtype, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    torch.cuda.synchronize()
    for bh in range(B * H):
        b, h = divmod(bh, H)
        _check_head(qkv, bh, Q[b, h].float().cpu().numpy(), K[b, h].float().cpu().numpy(),
                    V[b, h].float().cpu().numpy())


def test_quantize_strided_inputs_and_nonfinite_flag():
    B, H, N, d = 2, 3, 200, 128
    big = torch.randn(B, N, H, 2 * d, device="cuda").to(torch.bfloat16)  # [B, N, H, 2d] -> strided views
    Q = big[..., :d].permute(0, 2, 1, 3)
    K = (big[..., d:] + 3).permute(0, 2, 1, 3)
    V = big[..., :d].flip(-1).contiguous().permute(0, 2, 1, 3)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V, nonfinite=flag)
    torch.cuda.synchronize()
    assert flag.item() == 0
    for bh in (0, 4):
        b, h = divmod(bh, H)
        _check_head(qkv, bh, Q[b, h].float().cpu().numpy(), K[b, h].float().cpu().numpy(),
                    V[b, h].float().cpu().numpy())
    Q2 = Q.clone()
    Q2[1, 2, 17, 5] = float("nan")
    s3.sage3_quantize_qkv(Q2, K, V, nonfinite=flag)
    torch.cuda.synchronize()
    assert flag.item() == 1


def test_quantize_k_mean_order_with_large_offsets():
    """Smoothed K with |mean| >> |K - mean| stresses the fixed-order fp64 mean (reading c10)."""
    N, d = 4096 + 77, 128
    g = torch.Generator(device="cuda").manual_seed(11)
    K = (torch.randn(1, 1, N, d, device="cuda", generator=g) * 0.01 + 300.0).to(torch.bfloat16)
    Q = torch.randn(1, 1, N, d, device="cuda", generator=g).to(torch.bfloat16)
    qkv = s3.sage3_quantize_qkv(Q, K, Q)
    torch.cuda.synchronize()
    _check_head(qkv, 0, Q[0, 0].float().cpu().numpy(), K[0, 0].float().cpu().numpy(), Q[0, 0].float().cpu().numpy())


def test_hardware_converts_match_oracle_codecs():
    """cvt.rn.satfinite.{e2m1x2,e4m3x2}.f32 (what the kernels use) vs the oracle encoders, through the
    quantizer on crafted blocks: each 16-block is [a, x, x, ..] with amax fixed, sweeping x densely."""
    rng = np.random.default_rng(0)
    vals = np.concatenate([rng.standard_normal(1 << 16) * 4, rng.uniform(-6, 6, 1 << 16),
                           np.linspace(-6, 6, 1 << 15)]).clip(-6, 6).astype(np.float32)
    n_rows = vals.size // 15
    x = np.zeros((n_rows, 16), np.float32)
    x[:, 0] = 6.0  # amax 6 -> s = e4m3(1.0) = 1, so codes are e2m1(x) directly
    x[:, 1:] = vals[: n_rows * 15].reshape(n_rows, 15)
    N = (n_rows // 8 // 128) * 128  # 8 blocks per 128-channel token row
    d = 16 * 8
    Xb = torch.from_numpy(x[:N * 8].reshape(N, d)).to(torch.float16)  # fp16 rounding happens before both sides
    Q = Xb.view(1, 1, N, d).cuda()
    qkv = s3.sage3_quantize_qkv(Q, Q, Q)
    torch.cuda.synchronize()
    got = decode_head(qkv, 0)["q_codes"][:N]
    want = oracle.e2m1_encode_array(Xb.float().numpy().reshape(-1) * np.float32(1.0)).reshape(N, d)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("N", [1, 129, 300, 1000])
def test_quantize_smooth_q_bit_exact(d, N):
    """Smoothing Q (Alg1 L5): q̄ per 128-row tile and the codes/scales of Q - q̄ bit-exact with the oracle; the
    GEMV term ds = q̄_i·K_s^T (fp32 on the GPU) within fp32 accumulation error of the oracle's fp64 value."""
    B, H = 1, 2
    Q, K, V = synth.make_qkv(B, H, N, d, seed=3 * N + d, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V, smooth_q=True)
    torch.cuda.synchronize()
    for bh in range(B * H):
        q, k, v = (x[0, bh].float().cpu().numpy() for x in (Q, K, V))
        want = oracle.quantize_head(q, k, v, smooth_q=True)
        got = decode_head(qkv, bh)
        np.testing.assert_array_equal(got["km"], want.km)
        np.testing.assert_array_equal(got["q_mean"], want.q_mean)
        for name in ("q_codes", "q_sf", "k_codes", "k_sf", "v_codes"):
            np.testing.assert_array_equal(got[name], getattr(want, name), err_msg=name)
        ref = want.q_mean.astype(np.float64) @ want.ks.astype(np.float64).T  # [T][Np]
        bound = np.abs(want.q_mean).astype(np.float64) @ np.abs(want.ks).astype(np.float64).T
        err = np.abs(got["ds"][:, :N] - ref[:, :N])
        assert np.all(err <= 1e-6 * bound[:, :N] + 1e-30), err.max()


def test_fused_k_mean_path_bit_exact():
    """The optional fused K-mean quantizer (SAGE3_QUANT_FUSED_K=1: K read from HBM once, per-head chunk sums -> km ->
    φ(K − km) in one persistent launch) gives the same bits: this file's bit-exact cases rerun under it."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", os.path.join(here, "test_gpu_quant.py"),
                        "-k", "(bit_exact and not fused) or strided or large_offset"],
                       env=dict(os.environ, SAGE3_QUANT_FUSED_K="1"), capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
    assert " passed" in p.stdout
