"""GPU parity of SageBwd's backward (NEXT #3, Algorithm 3): sage3_int8_attn_bwd through the C ABI
against oracle.sb_attn_bwd on the same inputs.  Every oracle input comes from the oracle or the seeded synthetic
generator: Q̂/K̂ codes from oracle.sb_quantize_head (the GPU quantizer is bit-exact with it, asserted here), O and
lse from oracle.sb_attn_fwd, dO from synth.  Tolerance: the north_star's rel-L1 <= 2e-3 and cosine >= 0.9999 per
gradient (the GPU's ex2.approx P and fp32 dP flip a few ψ codes at rounding midpoints)."""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_2505_11594_b200 as s3
import synth

pytestmark = pytest.mark.gpu


def _case(B, H, N, d, causal, seed, dtype=torch.bfloat16, outliers=True):
    Q, K, V = synth.make_qkv(B, H, N, d, seed=seed, dtype=dtype, device="cuda", outliers=outliers)
    g = torch.Generator(device="cpu").manual_seed(seed * 7 + 1)
    dO = torch.randn(B, H, N, d, generator=g).to(dtype).cuda()
    scale = 1 / math.sqrt(d)
    heads, O, L, refs = [], torch.empty(B, H, N, d), torch.empty(B, H, N), []
    for bh in range(B * H):
        b, hh = divmod(bh, H)
        h = oracle.sb_quantize_head(*(x[b, hh].float().cpu().numpy() for x in (Q, K, V)))
        o, lse = oracle.sb_attn_fwd([h], causal=causal, scale=scale, want_lse=True)
        O[b, hh], L[b, hh] = torch.from_numpy(o[0]).float(), torch.from_numpy(lse[0]).float()
        heads.append(h)
    for bh in range(B * H):
        b, hh = divmod(bh, H)
        refs.append(oracle.sb_attn_bwd(heads[bh], V[b, hh].float().cpu().numpy(), O[b, hh].numpy(),
                                       dO[b, hh].float().cpu().numpy(), L[b, hh].numpy(), causal=causal, scale=scale))
    qkv = s3.sage3_int8_quantize_qkv(Q, K, V)
    torch.cuda.synchronize()
    Np = qkv.N_pad
    for bh in range(B * H):  # same Q̂, K̂, s_Q, s_K, K_m on both sides
        assert np.array_equal(qkv.q.view(torch.int8).view(-1, Np, d)[bh].cpu().numpy(), heads[bh].q)
        assert np.array_equal(qkv.k.view(torch.int8).view(-1, Np, d)[bh].cpu().numpy(), heads[bh].k)
    return Q, K, V, dO, O.cuda(), L.cuda().contiguous(), qkv, refs, scale


ROW_L1_MAX = 2e-2


def _check(got, ref, what):
    """north_star per-head gate, plus a per-row bound: every gradient row (a query row of dQ, a key row of dK/dV)
    has an L1 error within ROW_L1_MAX of the head's MEAN row L1 norm, so one wrong row or tile cannot hide inside
    the head average.  (Relative to the row's own norm would not do: ψ(dS) has one INT8 scale per 128 x 128 tile,
    so rows of small dS carry few quantization levels and a single code decided differently at a rounding
    midpoint moves them by percents of their own size.)"""
    m = oracle.accuracy_metrics(ref, got.astype(np.float64))
    assert np.all(np.isfinite(got)), what
    assert m["l1"] <= 2e-3 and m["cos_sim"] >= 0.9999, f"{what}: {m}"
    g = got.astype(np.float64)
    row = np.abs(g - ref).sum(axis=1) / (np.abs(ref).sum(axis=1).mean() + 1e-300)
    bad = np.argwhere(row > ROW_L1_MAX)
    assert bad.size == 0, f"{what}: rows {bad[:5, 0].tolist()} L1 / mean row L1 {row[bad[:5, 0]].tolist()}"
    m["max_row_l1"] = float(row.max())
    return m


@pytest.mark.parametrize("N,d,causal", [(128, 64, False), (128, 128, True), (300, 128, False), (300, 64, True),
                                        (1000, 128, True), (1000, 64, False), (640, 128, False), (2500, 64, True),
                                        (2100, 128, False)])
def test_int8_bwd_parity(N, d, causal):
    B, H = 1, 2
    _, _, V, dO, O, L, qkv, refs, scale = _case(B, H, N, d, causal, seed=N + d + int(causal))
    dq, dk, dv = s3.sage3_int8_attn_bwd(qkv, V, O, dO, L, causal=causal, softmax_scale=scale)
    torch.cuda.synchronize()
    for bh in range(B * H):
        b, hh = divmod(bh, H)
        for name, got, ref in zip(("dQ", "dK", "dV"), (dq, dk, dv), refs[bh]):
            _check(got[b, hh].cpu().numpy(), ref, f"head {bh} {name}")


@pytest.mark.parametrize("grad_dtype", [torch.bfloat16, torch.float16])
def test_int8_bwd_16bit_outputs(grad_dtype):
    _, _, V, dO, O, L, qkv, _, scale = _case(1, 2, 260, 128, True, seed=5)
    g32 = s3.sage3_int8_attn_bwd(qkv, V, O, dO, L, causal=True, softmax_scale=scale)
    g16 = s3.sage3_int8_attn_bwd(qkv, V, O, dO, L, causal=True, softmax_scale=scale, grad_dtype=grad_dtype)
    torch.cuda.synchronize()
    for a, b in zip(g32, g16):
        assert torch.equal(b, a.to(grad_dtype))


def test_int8_bwd_deterministic_dkdv_and_strided():
    """dK, dV are written by one CTA each (bitwise repeatable); outputs may be strided views."""
    _, _, V, dO, O, L, qkv, _, scale = _case(2, 2, 200, 64, False, seed=9)
    a = s3.sage3_int8_attn_bwd(qkv, V, O, dO, L, softmax_scale=scale)
    big = torch.empty(2, 2, 200, 3 * 64, dtype=torch.float32, device="cuda")
    b = s3.sage3_int8_attn_bwd(qkv, V, O, dO, L, softmax_scale=scale, dq=big[..., :64], dk=big[..., 64:128],
                               dv=big[..., 128:])
    torch.cuda.synchronize()
    assert torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    torch.testing.assert_close(a[0], b[0], rtol=1e-5, atol=1e-6)  # dQ: fp32 reduce-add order may differ


def test_int8_bwd_vs_fp64_autograd():
    """The GPU SageBwd gradients against fp64 autograd of plain attention (the paper's Tab1c level, CosSim)."""
    N, d = 512, 128
    Q, K, V = synth.make_qkv(1, 1, N, d, seed=21, dtype=torch.bfloat16, device="cuda", outliers=False)
    dO = torch.randn(1, 1, N, d, generator=torch.Generator().manual_seed(3)).to(torch.bfloat16).cuda()
    qkv = s3.sage3_int8_quantize_qkv(Q, K, V)
    lse = torch.empty(1, 1, N, dtype=torch.float32, device="cuda")
    O = s3.sage3_int8_attn_fwd(qkv, causal=True, lse=lse, out_dtype=torch.float32)
    dq, dk, dv = s3.sage3_int8_attn_bwd(qkv, V, O, dO, lse, causal=True)
    q, k, v = (x[0, 0].double().cpu().requires_grad_() for x in (Q, K, V))
    s = (q @ k.T) / math.sqrt(d)
    s = s.masked_fill(torch.triu(torch.ones(N, N, dtype=torch.bool), 1), float("-inf"))
    (torch.softmax(s, -1) @ v).backward(dO[0, 0].double().cpu())
    for name, got, ref in (("dQ", dq, q.grad), ("dK", dk, k.grad), ("dV", dv, v.grad)):
        m = oracle.accuracy_metrics(ref.numpy(), got[0, 0].double().cpu().numpy())
        print(name, m)
        assert m["cos_sim"] > 0.99, (name, m)
