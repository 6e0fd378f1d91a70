"""CPU checks of the C-ABI library: it loads without a GPU, exports every function include/sage3.h
declares, and its host-only logic (size queries, argument validation) behaves as documented."""
import ctypes
import os
import re

import pytest

import paper_2505_11594_b200 as s3
from paper_2505_11594_b200 import build as s3build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    s3build.build()
    return s3.load()


def header_functions():
    txt = open(os.path.join(ROOT, "include", "sage3.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sage3_[a-z0-9_]+)\s*\(", txt)))


def test_header_and_binding_agree():
    assert header_functions() == sorted(s3.ABI_FUNCTIONS)


def test_library_exports_every_declared_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name


def test_version_and_status_strings(lib):
    assert "sm_100a" in s3.version()
    assert lib.sage3_status_str(0) == b"SAGE3_OK"
    assert lib.sage3_status_str(3) == b"SAGE3_ERR_WORKSPACE"


def test_size_queries(lib):
    assert s3.sage3_kv_tile(128) == 128 and s3.sage3_kv_tile(64) == 128 and s3.sage3_kv_tile(96) == 0
    B, H, N, d = 2, 3, 300, 64
    Np = 384
    sizes = s3.sage3_fp4_qkv_sizes(B, H, N, d)
    assert sizes == [B * H * Np * d // 2] * 3 + [B * H * Np * d // 16] * 2 + [B * H * 128 * Np // 16, B * H * d * 4]
    # fp64 chunk sums [BH][d][Np/128] (256-byte aligned) + the fused K-mean control words (16 + 8 per head, aligned)
    al = lambda x: (x + 255) // 256 * 256
    assert s3.sage3_quantize_workspace_bytes(B, H, N, d) == al(B * H * (Np // 128) * d * 8) + al(16 + 8 * B * H)
    with pytest.raises(s3.Sage3Error):
        s3.sage3_fp4_qkv_sizes(1, 1, 0, 64)
    with pytest.raises(s3.Sage3Error):
        s3.sage3_fp4_qkv_sizes(1, 1, 128, 96)
    assert s3.sage3_fp4_qkv_sizes_fmt(B, H, N, d, "nvfp4") == sizes
    # MXFP4: d/32 <= 4 scale columns -> one 512-byte atom per 128 rows for Q/K, 4 token blocks per V atom
    for dd in (64, 128):
        mx = s3.sage3_fp4_qkv_sizes_fmt(B, H, N, dd, "mxfp4")
        assert mx == [B * H * Np * dd // 2] * 3 + [B * H * Np * 4] * 3 + [B * H * dd * 4]
    with pytest.raises(s3.Sage3Error):
        s3.sage3_fp4_qkv_sizes_fmt(B, H, N, d, 2)


def test_invalid_arguments_rejected_before_any_cuda_call(lib):
    """Null pointers / bad shapes return SAGE3_ERR_INVALID_ARG on the host (no device needed)."""
    z = s3.Tensor4(None, 0, 0, 0)
    f = s3.FP4QKVStruct(1, 1, 128, 64, 128)
    st = lib.sage3_quantize_qkv(z, z, z, s3.SAGE3_BF16, 1, 1, 128, 64, ctypes.byref(f), None, 0, None, None)
    assert st == s3.SAGE3_ERR_INVALID_ARG
    st = lib.sage3_attn_fwd(None, z, s3.SAGE3_BF16, 0, 0.0, None, None)
    assert st == s3.SAGE3_ERR_INVALID_ARG
    f.N_pad = 128
    t = s3.Tensor4(16, 0, 0, 64)  # misaligned-free fake pointer, but the qkv buffers are null
    st = lib.sage3_attn_fwd(ctypes.byref(f), t, s3.SAGE3_BF16, 0, 0.0, None, None)
    assert st == s3.SAGE3_ERR_INVALID_ARG
    for opts in (None, s3.AttnOptions(0, 0.0, 2, 0, 0, -1), s3.AttnOptions(0, 0.0, 0, 1, 0, -1)):
        st = lib.sage3_attn_fwd_ex(ctypes.byref(f), t, s3.SAGE3_BF16, ctypes.byref(opts) if opts else None, None,
                                   None)
        assert st == s3.SAGE3_ERR_INVALID_ARG  # null options, unknown p_quant, non-zero reserved
    f.fmt = 7  # not a sage3_fp4_format
    st = lib.sage3_quantize_qkv(t, t, t, s3.SAGE3_BF16, 1, 1, 128, 64, ctypes.byref(f), None, 0, None, None)
    assert st == s3.SAGE3_ERR_INVALID_ARG
    st = lib.sage3_forward_host(None, None, None, s3.SAGE3_BF16, 1, 1, 128, 64, 0, 0.0, None, s3.SAGE3_BF16, None, 0,
                                None)
    assert st == s3.SAGE3_ERR_INVALID_ARG


def test_binding_refuses_missing_library(monkeypatch, tmp_path):
    monkeypatch.setattr(s3, "_lib", None)
    monkeypatch.setattr(s3, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(s3.Sage3Error):
        s3.load()


def test_int8_bwd_host_checks(lib):
    """sage3_int8_attn_bwd: workspace size query and host-side rejections (no device needed)."""
    B, H, N, d = 2, 3, 300, 64
    Np = 384
    al = lambda x: (x + 255) // 256 * 256  # noqa: E731
    want = al(B * H * Np * d) + al(B * H * (Np // 128) * 4) + 2 * al(B * H * Np * 4) + al(B * H * Np * d * 4)
    assert s3.sage3_int8_bwd_workspace_bytes(B, H, N, d) == want
    assert s3.sage3_int8_bwd_workspace_bytes(1, 1, 128, 96) == 0
    t = s3.Tensor4(1 << 20, 0, 0, 64)
    z = s3.Tensor4(None, 0, 0, 0)
    q = s3.INT8QKVStruct(1, 1, 128, 64, 128)
    args = lambda qq, v, lse, gdt, ws, wsb: lib.sage3_int8_attn_bwd(  # noqa: E731
        qq, v, t, s3.SAGE3_FP32, t, s3.SAGE3_BF16, lse, 0, 0.0, t, t, t, gdt, ws, wsb, None)
    assert args(None, t, 16, s3.SAGE3_FP32, 1 << 20, 1 << 30) == s3.SAGE3_ERR_INVALID_ARG  # null qkv
    assert args(ctypes.byref(q), t, 16, s3.SAGE3_FP32, 1 << 20, 1 << 30) == s3.SAGE3_ERR_INVALID_ARG  # null codes
    q.q = q.k = q.s_q = q.s_k = q.k_mean = 1 << 20
    assert args(ctypes.byref(q), z, 16, s3.SAGE3_FP32, 1 << 20, 1 << 30) == s3.SAGE3_ERR_INVALID_ARG  # null v
    assert args(ctypes.byref(q), t, None, s3.SAGE3_FP32, 1 << 20, 1 << 30) == s3.SAGE3_ERR_INVALID_ARG  # null lse
    assert args(ctypes.byref(q), t, 16, 7, 1 << 20, 1 << 30) == s3.SAGE3_ERR_UNSUPPORTED  # gradient dtype
    assert args(ctypes.byref(q), t, 16, s3.SAGE3_FP32, 1 << 20, 16) == s3.SAGE3_ERR_WORKSPACE


class _FakeStream:  # the argument checks below return before anything is enqueued
    cuda_stream = 0


def test_binding_rejects_mismatched_outputs_before_the_call(lib):
    """an output whose shape or device does not match the problem, or a wrong lse, is refused in the
    binding (the C ABI only sees pointers and strides, and would write B*H*N rows)."""
    import torch

    qkv = s3.FP4QKV(1, 2, 200, 64, "cpu")
    st = _FakeStream()
    for bad in (torch.empty(1, 1, 200, 64), torch.empty(1, 2, 199, 64), torch.empty(2, 2, 200, 64)):
        with pytest.raises(s3.Sage3Error):
            s3.sage3_attn_fwd(qkv, bad, stream=st)
        with pytest.raises(s3.Sage3Error):
            s3.sage3_attn_fwd_units(qkv, bad, 0, 1, stream=st)
    o = torch.empty(1, 2, 200, 64, dtype=torch.bfloat16)
    for lse in (torch.empty(1, 2, 199), torch.empty(1, 2, 200, dtype=torch.float16), torch.empty(2, 400)[:, ::2]):
        with pytest.raises(s3.Sage3Error):
            s3.sage3_attn_fwd(qkv, o, lse=lse, stream=st)
    with pytest.raises(s3.Sage3Error):
        s3.sage3_forward_host(torch.empty(1, 2, 8, 64), torch.empty(1, 2, 8, 64), torch.empty(1, 2, 9, 64),
                              torch.empty(1, 2, 8, 64), torch.empty(16, dtype=torch.uint8), stream=st)


def test_abi_rejects_zero_head_stride_outputs(lib):
    """with H > 1 (or B > 1) an output with a zero head (batch) stride would make CTAs write the same
    rows concurrently; the ABI refuses it before any launch (no GPU needed to get the status)."""
    import torch

    qkv = s3.FP4QKV(1, 2, 200, 64, "cpu")
    st = _FakeStream()
    o = torch.empty(1, 1, 200, 64, dtype=torch.bfloat16).expand(1, 2, 200, 64)  # stride_h == 0
    with pytest.raises(s3.Sage3Error, match="INVALID_ARG"):
        s3.sage3_attn_fwd(qkv, o, stream=st)
