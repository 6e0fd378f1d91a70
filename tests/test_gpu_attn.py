"""GPU parity of sage3_attn_fwd against the oracle's Algorithm 1 on the SAME quantized codes.

Gates (tests/parity.py): the north_star per-head tolerance (rel-L1 <= 2e-3, cosine >= 0.9999 against the
oracle rounded to the GPU output dtype) AND an element-wise bound on every output element (one output-dtype
ulp + fp32 accumulation slack + the oracle's decision-sensitivity allowance for P codes within the GPU's exp
error of a rounding boundary).  Small/medium shapes use every row; the bench-size configuration uses a
deterministic row sample (rows are independent, so the sampled oracle rows are exact); full-size tests feed
the oracle its own quantize_head output of the original inputs."""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_2505_11594_b200 as s3
import synth
from layout import decode_head
from parity import check, oracle_attention, round_to  # noqa: F401  (round_to: re-exported for other tests)

pytestmark = pytest.mark.gpu


def oracle_heads(qkv, heads):
    out = []
    for bh in heads:
        g = decode_head(qkv, bh)
        h = oracle.QuantizedHead(qkv.N, qkv.d, fmt=qkv.fmt)  # the library's sage3_fp4_format = oracle FMT_*
        h.q_codes, h.k_codes, h.v_codes = g["q_codes"], g["k_codes"], g["v_codes"]
        h.q_sf, h.k_sf, h.v_sf = g["q_sf"], g["k_sf"], np.ascontiguousarray(g["v_sf_full"][: qkv.d])
        out.append(h)
    return out


def own_heads(Q, K, V, heads, **kw):
    """The oracle's OWN quantize_head of the original inputs for the flattened heads `heads` of [B,H,N,d]."""
    B, H, N, d = Q.shape
    f = lambda x, bh: x[bh // H, bh % H].float().cpu().numpy()
    return [oracle.quantize_head(f(Q, bh), f(K, bh), f(V, bh), **kw) for bh in heads]


# N < 128 (one partial tile that is both the first and the last), exact tiles, ragged tails, several tiles
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("N", [1, 15, 64, 127, 128, 300, 1024])
def test_attention_parity_full(N, d, causal, out_dtype):
    B, H = 1, 2
    Q, K, V = synth.make_qkv(B, H, N, d, seed=7 * N + d, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    scale = 1 / math.sqrt(d)
    lse = torch.empty(B, H, N, dtype=torch.float32, device="cuda")
    O = s3.sage3_attn_fwd(qkv, causal=causal, lse=lse, out_dtype=out_dtype)
    torch.cuda.synchronize()
    heads = oracle_heads(qkv, range(B * H))
    assert s3.sage3_kv_tile(d) == 128
    ref, ref_lse, amb, vmax = oracle_attention(heads, causal=causal, scale=scale)
    got = O.float().cpu().numpy().reshape(B * H, N, d)
    for bh in range(B * H):
        check(got[bh], ref[bh], out_dtype, f"head {bh}", amb=amb[bh], vmax=vmax[bh])
    np.testing.assert_allclose(lse.cpu().numpy().reshape(B * H, N), ref_lse, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("d", [64, 128])
def test_single_token_closed_form(d):
    """SPEC's N = 1 special case: one key, P̃ = 1, P̃2 = 2688 -> s_P2 = 448, code 6, so O = deq(V̂_0) times
    2688·fl32(1/2688) (the oracle's form) — on the GPU up to its 2^x evaluation of the row sum (key 0 sits in
    the polynomial exp2 lane, max relative error 2.7e-6, reading c14), hence rtol 5e-6."""
    Q, K, V = synth.make_qkv(2, 3, 1, d, seed=17 + d, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    O = s3.sage3_attn_fwd(qkv, causal=False, out_dtype=torch.float32)
    Oc = s3.sage3_attn_fwd(qkv, causal=True, out_dtype=torch.float32)
    torch.cuda.synchronize()
    c2688 = 2688.0 * float(np.float32(1.0) / np.float32(2688.0))
    for bh in range(6):
        g = decode_head(qkv, bh)
        v0 = oracle.dequant_fmt(g["v_codes"], np.ascontiguousarray(g["v_sf_full"][:d]), 0)[:, 0]
        want = v0 * c2688
        np.testing.assert_allclose(O.reshape(6, d)[bh].cpu().numpy(), want, rtol=5e-6, atol=0)
        np.testing.assert_allclose(Oc.reshape(6, d)[bh].cpu().numpy(), want, rtol=5e-6, atol=0)


@pytest.mark.parametrize("causal", [False, True])
def test_attention_zero_query_closed_form(causal):
    """Q = 0: every P̃2 = 2688 exactly on the GPU too, so O is the (causal) running mean of deq(V̂) times
    2688·fl32(1/2688) up to fp32 accumulation."""
    N, d = 384, 128
    _, K, V = synth.make_qkv(1, 1, N, d, seed=3, device="cuda")
    Q = torch.zeros_like(K)
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    O = s3.sage3_attn_fwd(qkv, causal=causal, out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref = oracle.attn_fwd(oracle_heads(qkv, [0]), causal=causal, scale=1 / math.sqrt(d))[0]
    np.testing.assert_allclose(O[0, 0].cpu().numpy(), ref, rtol=2e-5, atol=2e-6)


def test_attention_ragged_batch_heads_and_fp16():
    B, H, N, d = 2, 3, 777, 64
    Q, K, V = synth.make_qkv(B, H, N, d, seed=5, dtype=torch.float16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    O = s3.sage3_attn_fwd(qkv, causal=True, out_dtype=torch.float16)
    torch.cuda.synchronize()
    rows = np.array(sorted(set([0, 1, 127, 128, 129, 400, 640, 641, 775, 776])), np.int32)
    heads = [0, 4, 5]
    ref, _, amb, vmax = oracle_attention(oracle_heads(qkv, heads), causal=True, scale=1 / math.sqrt(d), rows=rows)
    got = O.float().cpu().numpy().reshape(B * H, N, d)
    for i, bh in enumerate(heads):
        check(got[bh][rows], ref[i], torch.float16, f"head {bh}", amb=amb[i], vmax=vmax[i])


@pytest.mark.parametrize("causal", [False, True])
def test_attention_bench_config_sampled_rows(causal):
    """The bench workload shape (B=1, H=32, N=32768, d=128) in the bench's launch configuration, checked
    on a deterministic sample of rows of two heads against the oracle run on its OWN quantization of the
    original inputs (the GPU codes of those heads are asserted bit-exact with it first)."""
    from test_gpu_quant import _check_head

    B, H, N, d = 1, 32, 32768, 128
    Q, K, V = synth.make_qkv(B, H, N, d, seed=0, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    O = s3.sage3_attn_fwd(qkv, causal=causal, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([[0, 1, 127, 128, N - 1], np.linspace(0, N - 1, 59).astype(np.int32)]))
    heads = [0, 31]
    own = own_heads(Q, K, V, heads)
    for bh in heads:
        _check_head(qkv, bh, *(x[0, bh].float().cpu().numpy() for x in (Q, K, V)))
    ref, _, amb, vmax = oracle_attention(own, causal=causal, scale=1 / math.sqrt(d), rows=rows)
    for i, bh in enumerate(heads):
        check(O[0, bh].float().cpu().numpy()[rows], ref[i], torch.bfloat16, f"head {bh}", amb=amb[i], vmax=vmax[i])


def test_accuracy_vs_full_precision_reported():
    """Paper metrics of the whole pipeline vs fp64 attention on the original inputs: reported, and
    sanity-gated loosely (synthetic outlier inputs; the paper's 99.5% is on real CogVideoX tensors)."""
    N, d = 2048, 128
    Q, K, V = synth.make_qkv(1, 1, N, d, seed=1, dtype=torch.bfloat16, device="cuda")
    O = s3.attention(Q, K, V, causal=False)
    torch.cuda.synchronize()
    rows = np.arange(0, N, 16, dtype=np.int32)
    ref = oracle.reference_attention(Q[0, 0].float().cpu().numpy(), K[0, 0].float().cpu().numpy(),
                                     V[0, 0].float().cpu().numpy(), causal=False, scale=1 / math.sqrt(d), rows=rows)
    m = oracle.accuracy_metrics(ref, O[0, 0].float().cpu().numpy()[rows])
    print("accuracy vs fp64 attention:", m)
    assert m["cos_sim"] > 0.9


def test_head_subset_is_bitwise_identical():
    """Sharding invariant: a head's O does not depend on which other heads share the launch, so
    O gathered from any number of GPUs is bitwise identical to the 1-GPU O."""
    B, H, N, d = 1, 6, 1000, 128
    Q, K, V = synth.make_qkv(B, H, N, d, seed=9, dtype=torch.bfloat16, device="cuda")
    full = s3.attention(Q, K, V, causal=True)
    part = s3.attention(Q[:, 2:5].contiguous(), K[:, 2:5].contiguous(), V[:, 2:5].contiguous(), causal=True)
    torch.cuda.synchronize()
    assert torch.equal(full[:, 2:5], part)


def test_forward_sharded_single_process_matches_direct():
    from paper_2505_11594_b200.multigpu import forward_sharded

    Q, K, V = synth.make_qkv(2, 3, 300, 64, seed=4, dtype=torch.bfloat16, device="cuda")
    a = forward_sharded(Q, K, V, causal=False)
    b = s3.attention(Q, K, V, causal=False)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


@pytest.mark.parametrize("B,H,N,d,causal", [(2, 5, 300, 64, False), (1, 11, 1000, 128, True), (1, 1, 128, 128, False)])
def test_forward_host_pipeline_matches_device_path(B, H, N, d, causal):
    """sage3_forward_host (head groups pipelined over three streams, pinned host buffers) gives bitwise the
    device-path result: every (b,h) is an independent problem, so grouping heads cannot change a bit."""
    Q, K, V = synth.make_qkv(B, H, N, d, seed=99 + H, dtype=torch.bfloat16, device="cuda")
    want = s3.attention(Q, K, V, causal=causal, out_dtype=torch.bfloat16)
    qh, kh, vh = (x.cpu().pin_memory() for x in (Q, K, V))
    oh = torch.empty(B, H, N, d, dtype=torch.bfloat16).pin_memory()
    scratch = torch.empty(s3.sage3_forward_host_scratch_bytes(B, H, N, d), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.Stream()
    s3.sage3_forward_host(qh, kh, vh, oh, scratch, causal=causal, stream=stream)
    stream.synchronize()
    torch.cuda.synchronize()
    assert torch.equal(oh, want.cpu())


@pytest.mark.parametrize("causal", [False, True])
def test_attn_fwd_units_subranges_bitwise(causal):
    """sage3_attn_fwd_units on any unit range writes exactly those rows, bitwise equal to the full launch (the
    invariant the multi-GPU unit split relies on); other rows stay untouched."""
    B, H, N, d = 1, 3, 1000, 128
    Q, K, V = synth.make_qkv(B, H, N, d, seed=21, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    full = s3.sage3_attn_fwd(qkv, causal=causal)
    T = (N + 127) // 128
    from paper_2505_11594_b200.multigpu import unit_rows
    for u0, u1 in [(0, 1), (5, 17), (7, 8), (0, 3 * T)]:
        o = torch.full_like(full, float("nan"))
        s3.sage3_attn_fwd_units(qkv, o, u0, u1, causal=causal)
        torch.cuda.synchronize()
        written = torch.zeros(B * H, N, dtype=torch.bool)
        for u in range(u0, u1):
            bh, r0, r1 = unit_rows(u, T, N)
            written[bh, r0:r1] = True
        of, ff = o.reshape(B * H, N, d).cpu(), full.reshape(B * H, N, d).cpu()
        assert torch.equal(of[written], ff[written])
        assert torch.isnan(of[~written].float()).all()


# The other BASELINE.json configurations at full size, in the bench's launch configuration (one launch over
# all heads): quantizer bit-exact on sampled heads, attention on sampled rows of those heads vs the oracle.
# C5 (B=8, H=32, N=32768, causal, 8 GPUs) runs 32 heads of N=32768 per GPU — the C2 causal case above.
CONFIGS = {
    "C3-cogvideox": (2, 30, 17776, 64, False, [0, 37, 59]),
    "C4-hunyuanvideo": (1, 24, 118800, 128, False, [0, 23]),
}


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_paper_config_full_size_sampled(name):
    from test_gpu_quant import _check_head

    B, H, N, d, causal, heads = CONFIGS[name]
    Q, K, V = synth.make_qkv(B, H, N, d, seed=5, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    O = s3.sage3_attn_fwd(qkv, causal=causal, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    Qf, Kf, Vf = (x.reshape(B * H, N, d) for x in (Q, K, V))
    for bh in heads:
        _check_head(qkv, bh, Qf[bh].float().cpu().numpy(), Kf[bh].float().cpu().numpy(), Vf[bh].float().cpu().numpy())
    rows = np.unique(np.concatenate([[0, 1, 127, 128, N - 129, N - 1], np.linspace(0, N - 1, 26).astype(np.int32)]))
    ref, _, amb, vmax = oracle_attention(own_heads(Q, K, V, heads), causal=causal, scale=1 / math.sqrt(d), rows=rows)
    Of = O.reshape(B * H, N, d)
    for i, bh in enumerate(heads):
        check(Of[bh].float().cpu().numpy()[rows], ref[i], torch.bfloat16, f"{name} head {bh}", amb=amb[i],
              vmax=vmax[i])


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("N,d", [(300, 64), (1000, 128), (128, 128), (15, 128), (1, 64), (2100, 128)])
def test_attention_smooth_q_parity(N, d, causal):
    """Smoothing Q (Alg1 L5 + L8's GEMV, NEXT #1): the GPU path (q̄ tiles, Q - q̄ codes, ds = q̄·K_s^T in fp32,
    S_j += 1·ds_jᵀ by a tf32 MMA on the hi/mid/lo split of ds) against the oracle's fp64 Algorithm 1 with
    smoothing Q, element-wise.  N = 2100: 17 KV tiles, so the ds rings (4 raw, 3 operand slots) wrap."""
    B, H = 1, 2
    Q, K, V = synth.make_qkv(B, H, N, d, seed=11 * N + d, dtype=torch.bfloat16, device="cuda")
    Q = Q + 4.0 * torch.randn(1, H, 1, d, device="cuda", dtype=torch.float32).to(torch.bfloat16)  # shared offset
    qkv = s3.sage3_quantize_qkv(Q, K, V, smooth_q=True)
    O = s3.sage3_attn_fwd(qkv, causal=causal, out_dtype=torch.float32)
    torch.cuda.synchronize()
    heads = [oracle.quantize_head(*(x[0, bh].float().cpu().numpy() for x in (Q, K, V)), smooth_q=True)
             for bh in range(B * H)]
    ref, _, amb, vmax = oracle_attention(heads, causal=causal, scale=1 / math.sqrt(d))
    for bh in range(B * H):
        check(O[0, bh].cpu().numpy(), ref[bh], torch.float32, f"head {bh}", amb=amb[bh], vmax=vmax[bh])


def test_smooth_q_improves_accuracy_on_gpu():
    """The paper's reason for smoothing Q, measured on the GPU path: queries sharing a large offset."""
    N, d = 2048, 128
    Q, K, V = synth.make_qkv(1, 1, N, d, seed=12, dtype=torch.bfloat16, device="cuda")
    Q = (Q.float() + 6.0 * torch.randn(1, 1, 1, d, device="cuda")).to(torch.bfloat16)
    rows = np.arange(0, N, 16, dtype=np.int32)
    ref = oracle.reference_attention(Q[0, 0].float().cpu().numpy(), K[0, 0].float().cpu().numpy(),
                                     V[0, 0].float().cpu().numpy(), causal=False, scale=1 / math.sqrt(d), rows=rows)
    m0 = oracle.accuracy_metrics(ref, s3.attention(Q, K, V)[0, 0].float().cpu().numpy()[rows])
    m1 = oracle.accuracy_metrics(ref, s3.attention(Q, K, V, smooth_q=True)[0, 0].float().cpu().numpy()[rows])
    print("GPU without / with smoothing Q:", m0, m1)
    assert m1["cos_sim"] > m0["cos_sim"]


@pytest.mark.parametrize("o_dtype", [torch.bfloat16, torch.float32])
def test_strided_output_and_lse(o_dtype):
    """O written through arbitrary (16-byte aligned) strides: a [B, H, N, d] view into a wider, head-major
    buffer; the rows and columns outside the view stay untouched; LSE matches the contiguous launch."""
    B, H, N, d = 2, 2, 300, 64
    Q, K, V = synth.make_qkv(B, H, N, d, seed=8, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    want = s3.sage3_attn_fwd(qkv, causal=True, out_dtype=o_dtype)
    big = torch.full((H, B, N + 8, 2 * d), 7.0, dtype=o_dtype, device="cuda")
    view = big[:, :, 4:4 + N, d:].permute(1, 0, 2, 3)  # [B, H, N, d], strides (2d(N+8), B·2d(N+8), 2d, 1)
    lse = torch.empty(B, H, N, dtype=torch.float32, device="cuda")
    lse_c = torch.empty_like(lse)
    s3.sage3_attn_fwd(qkv, view, causal=True, lse=lse)
    s3.sage3_attn_fwd(qkv, want, causal=True, lse=lse_c)
    torch.cuda.synchronize()
    assert torch.equal(view, want)
    assert torch.equal(lse, lse_c)
    mask = torch.ones_like(big, dtype=torch.bool)
    mask[:, :, 4:4 + N, d:] = False
    assert (big[mask] == 7.0).all()


def test_abi_rejects_bad_unit_ranges_and_half_smooth_q():
    Q, K, V = synth.make_qkv(1, 1, 256, 64, seed=2, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    o = torch.empty_like(Q)
    n = s3.n_units(qkv)
    for lo, hi in [(-1, 1), (2, 1), (0, n + 1)]:
        with pytest.raises(s3.Sage3Error):
            s3.sage3_attn_fwd_units(qkv, o, lo, hi)
    s3.sage3_attn_fwd_units(qkv, o, 1, 1)  # empty range: nothing enqueued, OK
    qkv.struct.q_mean = qkv.k_mean.data_ptr()  # q_mean without ds
    with pytest.raises(s3.Sage3Error):
        s3.sage3_attn_fwd(qkv, o)


@pytest.mark.parametrize("fmt", ["nvfp4", "mxfp4"])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("N,d", [(128, 128), (300, 64), (1024, 128)])
def test_direct_p_ablation_parity(N, d, causal, fmt):
    """Tab1b's direct-P ablation on the GPU (sage3_attn_fwd_ex, p_quant = direct): P̂ = φ(P̃) relative to the
    running max, s_P1 = 1, against the oracle's PMODE_DIRECT on the same codes, north_star tolerance."""
    B, H = 1, 2
    Q, K, V = synth.make_qkv(B, H, N, d, seed=13 * N + d, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V, fmt=fmt)
    lse = torch.empty(B, H, N, dtype=torch.float32, device="cuda")
    O = s3.sage3_attn_fwd(qkv, causal=causal, out_dtype=torch.float32, lse=lse, p_quant="direct")
    torch.cuda.synchronize()
    heads = oracle_heads(qkv, range(B * H))
    ref, ref_lse, amb, vmax = oracle_attention(heads, causal=causal, scale=1 / math.sqrt(d),
                                               p_mode=oracle.PMODE_DIRECT)
    for bh in range(B * H):
        check(O[0, bh].cpu().numpy(), ref[bh], torch.float32, f"head {bh}", amb=amb[bh], vmax=vmax[bh])
    np.testing.assert_allclose(lse.cpu().numpy().reshape(B * H, N), ref_lse, rtol=1e-5, atol=1e-4)
    # the unit-range form of the same call is bitwise identical
    O2 = torch.zeros_like(O)
    n = s3.n_units(qkv)
    s3.sage3_attn_fwd_ex(qkv, O2, causal=causal, p_quant="direct", unit_begin=0, unit_end=n // 2)
    s3.sage3_attn_fwd_ex(qkv, O2, causal=causal, p_quant="direct", unit_begin=n // 2)
    torch.cuda.synchronize()
    assert torch.equal(O, O2)


def test_two_level_beats_direct_p_on_gpu():
    """Tab1b: two-level P quantization is more accurate than direct φ(P̃) (the E4M3 scales of
    P̃ <= 1 underflow), measured on the GPU path against fp64 attention."""
    N, d = 4096, 128
    Q, K, V = synth.make_qkv(1, 1, N, d, seed=41, dtype=torch.bfloat16, device="cuda")
    rows = np.arange(0, N, 16, dtype=np.int32)
    ref = oracle.reference_attention(Q[0, 0].float().cpu().numpy(), K[0, 0].float().cpu().numpy(),
                                     V[0, 0].float().cpu().numpy(), causal=False, scale=1 / math.sqrt(d), rows=rows)
    m = {p: oracle.accuracy_metrics(ref, s3.attention(Q, K, V, p_quant=p, out_dtype=torch.float32)[0, 0].cpu().numpy()[rows])
         for p in ("two_level", "direct")}
    print("GPU two-level / direct P:", m)
    assert m["two_level"]["cos_sim"] > m["direct"]["cos_sim"] and m["two_level"]["l1"] < m["direct"]["l1"]


def test_direct_p_rejects_smoothing_q():
    Q, K, V = synth.make_qkv(1, 1, 256, 64, seed=2, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V, smooth_q=True)
    with pytest.raises(s3.Sage3Error):
        s3.sage3_attn_fwd(qkv, p_quant="direct")


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("N,d", [(1, 64), (100, 128), (128, 64), (300, 128), (1024, 128), (2100, 64)])
def test_qsum_variant_parity(N, d, causal):
    """NEXT #2 row-sum variant (p_quant = "qsum", reading n2): l from the tensor core's ones-column product of the
    quantized P̂2, against the oracle's PMODE_QSUM on the same codes (both gates of tests/parity.py), LSE, and the
    unit-range form bitwise."""
    B, H = 1, 2
    Q, K, V = synth.make_qkv(B, H, N, d, seed=23 * N + d, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    lse = torch.empty(B, H, N, dtype=torch.float32, device="cuda")
    O = s3.sage3_attn_fwd(qkv, causal=causal, out_dtype=torch.float32, lse=lse, p_quant="qsum")
    torch.cuda.synchronize()
    rows = np.arange(N, dtype=np.int32) if N <= 1024 else np.arange(0, N, 5, dtype=np.int32)
    ref, ref_lse, amb, vmax = oracle_attention(oracle_heads(qkv, range(B * H)), causal=causal,
                                               scale=1 / math.sqrt(d), p_mode=oracle.PMODE_QSUM, rows=rows)
    for bh in range(B * H):
        check(O[0, bh].cpu().numpy()[rows], ref[bh], torch.float32, f"head {bh}", amb=amb[bh], vmax=vmax[bh])
    # LSE = scale·m + ln l with l from the quantized P: a P code decided the other way at a rounding midpoint (the
    # decisions the element-wise bound allows for) moves l too, so a few rows may differ by up to a few 1e-3
    dl = np.abs(lse.cpu().numpy().reshape(B * H, N)[:, rows] - ref_lse)
    assert np.mean(dl > 1e-4 + 1e-5 * np.abs(ref_lse)) <= 0.01 and dl.max() <= 5e-3, (np.mean(dl > 1e-4), dl.max())
    O2 = torch.zeros_like(O)
    n = s3.n_units(qkv)
    s3.sage3_attn_fwd_ex(qkv, O2, causal=causal, p_quant="qsum", unit_begin=0, unit_end=n // 2)
    s3.sage3_attn_fwd_ex(qkv, O2, causal=causal, p_quant="qsum", unit_begin=n // 2)
    torch.cuda.synchronize()
    assert torch.equal(O, O2)


def test_qsum_constant_values_exact_on_gpu():
    """The variant's defining property on the GPU: with every V row equal, O equals that row (the weights are
    normalised by their own tensor-core sum) up to fp32 accumulation."""
    N, d = 1000, 128
    Q, K, V = synth.make_qkv(1, 1, N, d, seed=5, dtype=torch.bfloat16, device="cuda")
    V = V[:, :, :1].expand(1, 1, N, d).contiguous()
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    O = s3.sage3_attn_fwd(qkv, causal=True, out_dtype=torch.float32, p_quant="qsum")
    torch.cuda.synchronize()
    g = decode_head(qkv, 0)
    cdeq = oracle.dequant_fmt(g["v_codes"], np.ascontiguousarray(g["v_sf_full"][:d]), 0)[:, 0]
    np.testing.assert_allclose(O[0, 0].cpu().numpy(), np.broadcast_to(cdeq, (N, d)), rtol=2e-6, atol=1e-7)


def test_qsum_rejects_mxfp4_and_smoothing_q():
    Q, K, V = synth.make_qkv(1, 1, 256, 64, seed=2, dtype=torch.bfloat16, device="cuda")
    for kw in ({"fmt": "mxfp4"}, {"smooth_q": True}):
        qkv = s3.sage3_quantize_qkv(Q, K, V, **kw)
        with pytest.raises(s3.Sage3Error):
            s3.sage3_attn_fwd(qkv, p_quant="qsum")
