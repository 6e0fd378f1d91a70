"""B200-native (sm_100a) SageAttention3 FP4 attention forward — thin ctypes binding over libsage3.so.

The C ABI is ``include/sage3.h``; the functions here carry the same names and only marshal arguments
(torch tensors -> device pointers / strides, the current CUDA stream).  Every step of the method runs in
the CUDA kernels of ``csrc/``; there is no CPU or PyTorch fallback: if the library is missing this
module raises.  PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import math
import os

import torch

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SAGE3_LIB") or os.path.join(PKG, "libsage3.so")  # env override: experiments only

SAGE3_OK, SAGE3_ERR_INVALID_ARG, SAGE3_ERR_UNSUPPORTED, SAGE3_ERR_WORKSPACE, SAGE3_ERR_CUDA = range(5)
SAGE3_FP16, SAGE3_BF16, SAGE3_FP32 = 0, 1, 2
SAGE3_NVFP4, SAGE3_MXFP4 = 0, 1  # sage3_fp4_format: the method / the Tab1a data-type ablation
_FMT = {"nvfp4": SAGE3_NVFP4, "mxfp4": SAGE3_MXFP4, SAGE3_NVFP4: SAGE3_NVFP4, SAGE3_MXFP4: SAGE3_MXFP4}
# sage3_p_quant: the method / the Tab1b ablation / the NEXT #2 lazy-reference throughput variant
SAGE3_P_TWO_LEVEL, SAGE3_P_DIRECT, SAGE3_P_TWO_LEVEL_LAZY, SAGE3_P_TWO_LEVEL_QSUM = 0, 1, 2, 3
_PQ = {"two_level": SAGE3_P_TWO_LEVEL, "direct": SAGE3_P_DIRECT, "lazy": SAGE3_P_TWO_LEVEL_LAZY,
       "qsum": SAGE3_P_TWO_LEVEL_QSUM}
_DT = {torch.float16: SAGE3_FP16, torch.bfloat16: SAGE3_BF16, torch.float32: SAGE3_FP32}

# Every function include/sage3.h declares (checked by tests/test_abi.py).
ABI_FUNCTIONS = (
    "sage3_fp4_qkv_sizes", "sage3_fp4_qkv_sizes_fmt", "sage3_smooth_q_sizes", "sage3_quantize_workspace_bytes", "sage3_kv_tile", "sage3_quantize_qkv",
    "sage3_attn_fwd", "sage3_attn_fwd_units", "sage3_attn_fwd_ex", "sage3_forward_host_scratch_bytes", "sage3_forward_host", "sage3_status_str",
    "sage3_last_cuda_error", "sage3_version", "sage3_int8_qkv_sizes", "sage3_int8_quantize_qkv", "sage3_int8_attn_fwd",
    "sage3_int8_bwd_workspace_bytes", "sage3_int8_attn_bwd",
)


class Sage3Error(RuntimeError):
    pass


class Tensor4(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("stride_b", ctypes.c_int64), ("stride_h", ctypes.c_int64),
                ("stride_n", ctypes.c_int64)]


class FP4QKVStruct(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int32), ("H", ctypes.c_int32), ("N", ctypes.c_int32), ("d", ctypes.c_int32),
                ("N_pad", ctypes.c_int32), ("fmt", ctypes.c_int32)] + [(n, ctypes.c_void_p) for n in (
                    "q_data", "k_data", "v_data", "q_sf", "k_sf", "v_sf", "k_mean", "q_mean", "ds")]


class INT8QKVStruct(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int32), ("H", ctypes.c_int32), ("N", ctypes.c_int32), ("d", ctypes.c_int32),
                ("N_pad", ctypes.c_int32)] + [(n, ctypes.c_void_p) for n in (
                    "q", "k", "v_t", "s_q", "s_k", "s_v", "k_mean")]


class AttnOptions(ctypes.Structure):
    _fields_ = [("causal", ctypes.c_int32), ("softmax_scale", ctypes.c_float), ("p_quant", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("unit_begin", ctypes.c_int64), ("unit_end", ctypes.c_int64)]


_lib = None


def load() -> ctypes.CDLL:
    """Load libsage3.so (built in-tree by ``python -m paper_2505_11594_b200.build``); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise Sage3Error(f"{LIB_PATH} is missing: build it with `python -m paper_2505_11594_b200.build` "
                         "(there is no fallback implementation)")
    L = ctypes.CDLL(LIB_PATH)
    sz = ctypes.c_size_t
    L.sage3_fp4_qkv_sizes.argtypes = [ctypes.c_int] * 4 + [ctypes.POINTER(sz)]
    L.sage3_fp4_qkv_sizes_fmt.argtypes = [ctypes.c_int] * 5 + [ctypes.POINTER(sz)]
    L.sage3_smooth_q_sizes.argtypes = [ctypes.c_int] * 4 + [ctypes.POINTER(sz)]
    L.sage3_quantize_workspace_bytes.argtypes = [ctypes.c_int] * 4
    L.sage3_quantize_workspace_bytes.restype = sz
    L.sage3_kv_tile.argtypes = [ctypes.c_int]
    L.sage3_quantize_qkv.argtypes = [Tensor4, Tensor4, Tensor4, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, ctypes.POINTER(FP4QKVStruct), ctypes.c_void_p, sz,
                                     ctypes.c_void_p, ctypes.c_void_p]
    L.sage3_attn_fwd.argtypes = [ctypes.POINTER(FP4QKVStruct), Tensor4, ctypes.c_int, ctypes.c_int, ctypes.c_float,
                                 ctypes.c_void_p, ctypes.c_void_p]
    L.sage3_attn_fwd_units.argtypes = [ctypes.POINTER(FP4QKVStruct), Tensor4, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_float, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_void_p]
    L.sage3_attn_fwd_ex.argtypes = [ctypes.POINTER(FP4QKVStruct), Tensor4, ctypes.c_int,
                                    ctypes.POINTER(AttnOptions), ctypes.c_void_p, ctypes.c_void_p]
    L.sage3_forward_host_scratch_bytes.argtypes = [ctypes.c_int] * 6
    L.sage3_forward_host_scratch_bytes.restype = sz
    L.sage3_forward_host.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 6 + [ctypes.c_float, ctypes.c_void_p,
                                                                                ctypes.c_int, ctypes.c_void_p, sz,
                                                                                ctypes.c_void_p]
    L.sage3_int8_qkv_sizes.argtypes = [ctypes.c_int] * 4 + [ctypes.POINTER(sz)]
    L.sage3_int8_quantize_qkv.argtypes = [Tensor4, Tensor4, Tensor4, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, ctypes.POINTER(INT8QKVStruct), ctypes.c_void_p,
                                          sz, ctypes.c_void_p, ctypes.c_void_p]
    L.sage3_int8_attn_fwd.argtypes = [ctypes.POINTER(INT8QKVStruct), Tensor4, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_float, ctypes.c_void_p, ctypes.c_void_p]
    L.sage3_int8_bwd_workspace_bytes.argtypes = [ctypes.c_int] * 4
    L.sage3_int8_bwd_workspace_bytes.restype = ctypes.c_size_t
    L.sage3_int8_attn_bwd.argtypes = [ctypes.POINTER(INT8QKVStruct), Tensor4, Tensor4, ctypes.c_int, Tensor4,
                                      ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_float, Tensor4, Tensor4,
                                      Tensor4, ctypes.c_int, ctypes.c_void_p, sz, ctypes.c_void_p]
    L.sage3_status_str.argtypes = [ctypes.c_int]
    L.sage3_status_str.restype = ctypes.c_char_p
    L.sage3_version.restype = ctypes.c_char_p
    _lib = L
    return L


def _check(status: int, what: str):
    if status != SAGE3_OK:
        L = load()
        msg = L.sage3_status_str(status).decode()
        if status == SAGE3_ERR_CUDA:
            msg += f" (cudaError {L.sage3_last_cuda_error()})"
        raise Sage3Error(f"{what}: {msg}")


def _stream(stream) -> ctypes.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _t4(x: torch.Tensor) -> Tensor4:
    if x.dim() != 4 or x.stride(3) != 1:
        raise Sage3Error(f"expected a [B, H, N, d] tensor with unit d-stride, got shape {tuple(x.shape)} "
                         f"strides {tuple(x.stride())}")
    return Tensor4(x.data_ptr(), x.stride(0), x.stride(1), x.stride(2))


def _check_out(o: torch.Tensor, shape, device, what: str):
    """An output the kernels write with the problem's B, H, N, d: shape and device must match exactly (the C ABI
    only sees a pointer and strides)."""
    if tuple(o.shape) != tuple(shape):
        raise Sage3Error(f"{what}: output shape {tuple(o.shape)} != {tuple(shape)}")
    if o.device != device:
        raise Sage3Error(f"{what}: output on {o.device}, inputs on {device}")


def _check_lse(lse: torch.Tensor | None, n: int, device, what: str):
    if lse is None:
        return
    if lse.dtype != torch.float32 or not lse.is_contiguous() or lse.numel() != n or lse.device != device:
        raise Sage3Error(f"{what}: lse must be a contiguous float32 tensor of B*H*N = {n} elements on {device}, got "
                         f"{lse.dtype} {tuple(lse.shape)} contiguous={lse.is_contiguous()} on {lse.device}")


def version() -> str:
    return load().sage3_version().decode()


def sage3_kv_tile(d: int) -> int:
    return int(load().sage3_kv_tile(d))


def sage3_fp4_qkv_sizes(B: int, H: int, N: int, d: int) -> list[int]:
    out = (ctypes.c_size_t * 7)()
    _check(load().sage3_fp4_qkv_sizes(B, H, N, d, out), "sage3_fp4_qkv_sizes")
    return list(out)


def sage3_fp4_qkv_sizes_fmt(B: int, H: int, N: int, d: int, fmt) -> list[int]:
    out = (ctypes.c_size_t * 7)()
    _check(load().sage3_fp4_qkv_sizes_fmt(B, H, N, d, _FMT.get(fmt, -1), out), "sage3_fp4_qkv_sizes_fmt")
    return list(out)


def sage3_smooth_q_sizes(B: int, H: int, N: int, d: int) -> list[int]:
    out = (ctypes.c_size_t * 2)()
    _check(load().sage3_smooth_q_sizes(B, H, N, d, out), "sage3_smooth_q_sizes")
    return list(out)


def sage3_quantize_workspace_bytes(B: int, H: int, N: int, d: int) -> int:
    return int(load().sage3_quantize_workspace_bytes(B, H, N, d))


class FP4QKV:
    """Device buffers of one FP4 Q/K/V set (layouts: include/sage3.h), allocated with torch.
    fmt: "nvfp4" (the method) or "mxfp4" (Tab1a ablation)."""

    NAMES = ("q_data", "k_data", "v_data", "q_sf", "k_sf", "v_sf", "k_mean")

    def __init__(self, B: int, H: int, N: int, d: int, device, smooth_q: bool = False, fmt="nvfp4"):
        self.B, self.H, self.N, self.d = B, H, N, d
        self.N_pad = (N + 127) // 128 * 128
        self.smooth_q = smooth_q
        if fmt not in _FMT:
            raise Sage3Error(f"unknown FP4 format {fmt!r}")
        self.fmt = _FMT[fmt]
        sizes = sage3_fp4_qkv_sizes_fmt(B, H, N, d, self.fmt)
        for name, nbytes in zip(self.NAMES, sizes):
            setattr(self, name, torch.empty(nbytes, dtype=torch.uint8, device=device))
        self.q_mean = self.ds = None
        if smooth_q:  # Alg1 L5 / L8 GEMV buffers
            qm_b, ds_b = sage3_smooth_q_sizes(B, H, N, d)
            self.q_mean = torch.empty(qm_b, dtype=torch.uint8, device=device)
            self.ds = torch.empty(ds_b, dtype=torch.uint8, device=device)
        self.workspace = torch.empty(max(sage3_quantize_workspace_bytes(B, H, N, d), 16), dtype=torch.uint8,
                                     device=device)
        self.struct = FP4QKVStruct(B, H, N, d, self.N_pad, self.fmt,
                                   *[getattr(self, n).data_ptr() for n in self.NAMES],
                                   self.q_mean.data_ptr() if smooth_q else None,
                                   self.ds.data_ptr() if smooth_q else None)

    def nbytes(self) -> int:
        return sum(getattr(self, n).numel() for n in self.NAMES)


def sage3_quantize_qkv(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: FP4QKV | None = None,
                       nonfinite: torch.Tensor | None = None, stream=None, smooth_q: bool = False,
                       fmt="nvfp4") -> FP4QKV:
    """Alg1 L2 + L7 (smoothing K, FP4 φ of Q, K, V; + L5 / L8's GEMV with smooth_q): see include/sage3.h.
    The format of a given `out` is its own (fmt applies when out is None)."""
    B, H, N, d = q.shape
    if not (k.shape == q.shape == v.shape and q.dtype == k.dtype == v.dtype
            and q.dtype in (torch.float16, torch.bfloat16) and q.device == k.device == v.device):
        raise Sage3Error("sage3_quantize_qkv: q, k, v must share shape, device and a 16-bit float dtype")
    if out is None:
        out = FP4QKV(B, H, N, d, q.device, smooth_q=smooth_q, fmt=fmt)
    elif (out.B, out.H, out.N, out.d) != (B, H, N, d) or out.q_data.device != q.device:
        raise Sage3Error(f"sage3_quantize_qkv: out holds {(out.B, out.H, out.N, out.d)} on {out.q_data.device}")
    flag = ctypes.c_void_p(nonfinite.data_ptr() if nonfinite is not None else None)
    st = load().sage3_quantize_qkv(_t4(q), _t4(k), _t4(v), _DT[q.dtype], B, H, N, d, ctypes.byref(out.struct),
                                   ctypes.c_void_p(out.workspace.data_ptr()), out.workspace.numel(), flag,
                                   _stream(stream))
    _check(st, "sage3_quantize_qkv")
    return out


def sage3_attn_fwd(qkv: FP4QKV, o: torch.Tensor | None = None, *, causal: bool = False,
                   softmax_scale: float = 0.0, lse: torch.Tensor | None = None, out_dtype=torch.bfloat16,
                   stream=None, p_quant: str = "two_level") -> torch.Tensor:
    """Alg1 L6-L13 (FP4 QK^T, online softmax, two-level P, FP4 PV, O/l): see include/sage3.h.
    p_quant="direct" selects the Tab1b ablation (sage3_attn_fwd_ex)."""
    if o is None:
        o = torch.empty(qkv.B, qkv.H, qkv.N, qkv.d, dtype=out_dtype, device=qkv.q_data.device)
    _check_out(o, (qkv.B, qkv.H, qkv.N, qkv.d), qkv.q_data.device, "sage3_attn_fwd")
    _check_lse(lse, qkv.B * qkv.H * qkv.N, qkv.q_data.device, "sage3_attn_fwd")
    if p_quant != "two_level":
        return sage3_attn_fwd_ex(qkv, o, causal=causal, softmax_scale=softmax_scale, lse=lse, stream=stream,
                                 p_quant=p_quant)
    lse_p = ctypes.c_void_p(lse.data_ptr() if lse is not None else None)
    st = load().sage3_attn_fwd(ctypes.byref(qkv.struct), _t4(o), _DT[o.dtype], 1 if causal else 0,
                               float(softmax_scale), lse_p, _stream(stream))
    _check(st, "sage3_attn_fwd")
    return o


def sage3_attn_fwd_ex(qkv: FP4QKV, o: torch.Tensor, *, causal: bool = False, softmax_scale: float = 0.0,
                      lse: torch.Tensor | None = None, stream=None, p_quant: str = "two_level", unit_begin: int = 0,
                      unit_end: int = -1) -> torch.Tensor:
    """sage3_attn_fwd_ex: the attention with a sage3_attn_options struct (P quantization mode, unit range)."""
    if p_quant not in _PQ:
        raise Sage3Error(f"unknown p_quant {p_quant!r}")
    _check_out(o, (qkv.B, qkv.H, qkv.N, qkv.d), qkv.q_data.device, "sage3_attn_fwd_ex")
    _check_lse(lse, qkv.B * qkv.H * qkv.N, qkv.q_data.device, "sage3_attn_fwd_ex")
    opts = AttnOptions(1 if causal else 0, float(softmax_scale), _PQ[p_quant], 0, int(unit_begin), int(unit_end))
    lse_p = ctypes.c_void_p(lse.data_ptr() if lse is not None else None)
    st = load().sage3_attn_fwd_ex(ctypes.byref(qkv.struct), _t4(o), _DT[o.dtype], ctypes.byref(opts), lse_p,
                                  _stream(stream))
    _check(st, "sage3_attn_fwd_ex")
    return o


def n_units(qkv: FP4QKV) -> int:
    """Work units of the (b·h, 128-row query tile) space (see sage3_attn_fwd_units)."""
    return qkv.B * qkv.H * ((qkv.N + 127) // 128)


def sage3_attn_fwd_units(qkv: FP4QKV, o: torch.Tensor, unit_begin: int, unit_end: int, *, causal: bool = False,
                         softmax_scale: float = 0.0, lse: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """sage3_attn_fwd on the work units [unit_begin, unit_end) only (rows of o outside them untouched)."""
    _check_out(o, (qkv.B, qkv.H, qkv.N, qkv.d), qkv.q_data.device, "sage3_attn_fwd_units")
    _check_lse(lse, qkv.B * qkv.H * qkv.N, qkv.q_data.device, "sage3_attn_fwd_units")
    lse_p = ctypes.c_void_p(lse.data_ptr() if lse is not None else None)
    st = load().sage3_attn_fwd_units(ctypes.byref(qkv.struct), _t4(o), _DT[o.dtype], 1 if causal else 0,
                                     float(softmax_scale), lse_p, int(unit_begin), int(unit_end), _stream(stream))
    _check(st, "sage3_attn_fwd_units")
    return o


def sage3_forward_host_scratch_bytes(B, H, N, d, in_dtype=torch.bfloat16, out_dtype=torch.bfloat16) -> int:
    return int(load().sage3_forward_host_scratch_bytes(B, H, N, d, _DT[in_dtype], _DT[out_dtype]))


def sage3_forward_host(q_host: torch.Tensor, k_host: torch.Tensor, v_host: torch.Tensor, o_host: torch.Tensor,
                       scratch: torch.Tensor, *, causal: bool = False, softmax_scale: float = 0.0, stream=None):
    """Host-buffer end-to-end path (H2D, quantize, attention, D2H enqueued on `stream`; not synchronized)."""
    B, H, N, d = q_host.shape
    for t in (q_host, k_host, v_host, o_host):
        if t.device.type != "cpu" or not t.is_contiguous() or tuple(t.shape) != (B, H, N, d):
            raise Sage3Error("sage3_forward_host: q, k, v, o must be contiguous host tensors of one [B, H, N, d] shape")
    if not (q_host.dtype == k_host.dtype == v_host.dtype):
        raise Sage3Error("sage3_forward_host: q, k, v must share a dtype")
    st = load().sage3_forward_host(ctypes.c_void_p(q_host.data_ptr()), ctypes.c_void_p(k_host.data_ptr()),
                                   ctypes.c_void_p(v_host.data_ptr()), _DT[q_host.dtype], B, H, N, d,
                                   1 if causal else 0, float(softmax_scale), ctypes.c_void_p(o_host.data_ptr()),
                                   _DT[o_host.dtype], ctypes.c_void_p(scratch.data_ptr()), scratch.numel(),
                                   _stream(stream))
    _check(st, "sage3_forward_host")
    return o_host


def attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, causal: bool = False,
              softmax_scale: float = 0.0, out_dtype=None, stream=None, smooth_q: bool = False,
              fmt="nvfp4", p_quant: str = "two_level") -> torch.Tensor:
    """Quantize + attention in one call (the two ABI calls, enqueued on the current stream)."""
    qkv = sage3_quantize_qkv(q, k, v, stream=stream, smooth_q=smooth_q, fmt=fmt)
    return sage3_attn_fwd(qkv, causal=causal, softmax_scale=softmax_scale, out_dtype=out_dtype or q.dtype,
                          stream=stream, p_quant=p_quant)


# ------------------------------------------------------------------ SageBwd 8-bit forward (NEXT #3)
def sage3_int8_qkv_sizes(B: int, H: int, N: int, d: int) -> list[int]:
    out = (ctypes.c_size_t * 7)()
    _check(load().sage3_int8_qkv_sizes(B, H, N, d, out), "sage3_int8_qkv_sizes")
    return list(out)


class INT8QKV:
    """Device buffers of SageBwd's INT8 Q/K/V (include/sage3.h sage3_int8_qkv), allocated with torch."""

    NAMES = ("q", "k", "v_t", "s_q", "s_k", "s_v", "k_mean")

    def __init__(self, B: int, H: int, N: int, d: int, device):
        self.B, self.H, self.N, self.d = B, H, N, d
        self.N_pad = (N + 127) // 128 * 128
        for name, nbytes in zip(self.NAMES, sage3_int8_qkv_sizes(B, H, N, d)):
            setattr(self, name, torch.empty(nbytes, dtype=torch.uint8, device=device))
        self.workspace = torch.empty(max(sage3_quantize_workspace_bytes(B, H, N, d), 16), dtype=torch.uint8,
                                     device=device)
        self.struct = INT8QKVStruct(B, H, N, d, self.N_pad, *[getattr(self, n).data_ptr() for n in self.NAMES])


def sage3_int8_quantize_qkv(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: INT8QKV | None = None,
                            nonfinite: torch.Tensor | None = None, stream=None) -> INT8QKV:
    """Alg2 L2 + L4: smooth-K and per-block INT8 ψ of Q, K, V (see include/sage3.h)."""
    B, H, N, d = q.shape
    if not (k.shape == q.shape == v.shape and q.dtype == k.dtype == v.dtype
            and q.dtype in (torch.float16, torch.bfloat16) and q.device == k.device == v.device):
        raise Sage3Error("sage3_int8_quantize_qkv: q, k, v must share shape, device and a 16-bit float dtype")
    if out is None:
        out = INT8QKV(B, H, N, d, q.device)
    elif (out.B, out.H, out.N, out.d) != (B, H, N, d) or out.q.device != q.device:
        raise Sage3Error(f"sage3_int8_quantize_qkv: out holds {(out.B, out.H, out.N, out.d)} on {out.q.device}")
    flag = ctypes.c_void_p(nonfinite.data_ptr() if nonfinite is not None else None)
    st = load().sage3_int8_quantize_qkv(_t4(q), _t4(k), _t4(v), _DT[q.dtype], B, H, N, d, ctypes.byref(out.struct),
                                        ctypes.c_void_p(out.workspace.data_ptr()), out.workspace.numel(), flag,
                                        _stream(stream))
    _check(st, "sage3_int8_quantize_qkv")
    return out


def sage3_int8_attn_fwd(qkv: INT8QKV, o: torch.Tensor | None = None, *, causal: bool = False,
                        softmax_scale: float = 0.0, lse: torch.Tensor | None = None, out_dtype=torch.bfloat16,
                        stream=None) -> torch.Tensor:
    """Alg2 L6-L14 (INT8 QKᵀ, online softmax, per-token INT8 P, INT8 PV, O/l, lse)."""
    if o is None:
        o = torch.empty(qkv.B, qkv.H, qkv.N, qkv.d, dtype=out_dtype, device=qkv.q.device)
    _check_out(o, (qkv.B, qkv.H, qkv.N, qkv.d), qkv.q.device, "sage3_int8_attn_fwd")
    _check_lse(lse, qkv.B * qkv.H * qkv.N, qkv.q.device, "sage3_int8_attn_fwd")
    lse_p = ctypes.c_void_p(lse.data_ptr() if lse is not None else None)
    st = load().sage3_int8_attn_fwd(ctypes.byref(qkv.struct), _t4(o), _DT[o.dtype], 1 if causal else 0,
                                    float(softmax_scale), lse_p, _stream(stream))
    _check(st, "sage3_int8_attn_fwd")
    return o


def default_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)


def sage3_int8_bwd_workspace_bytes(B: int, H: int, N: int, d: int) -> int:
    return int(load().sage3_int8_bwd_workspace_bytes(B, H, N, d))


def sage3_int8_attn_bwd(qkv: INT8QKV, v: torch.Tensor, o: torch.Tensor, dout: torch.Tensor, lse: torch.Tensor, *,
                        causal: bool = False, softmax_scale: float = 0.0, grad_dtype=torch.float32,
                        dq: torch.Tensor | None = None, dk: torch.Tensor | None = None, dv: torch.Tensor | None = None,
                        workspace: torch.Tensor | None = None, stream=None):
    """Alg3 (SageBwd backward): returns (dq, dk, dv) w.r.t. the unsmoothed q, k, v (see include/sage3.h)."""
    B, H, N, d = qkv.B, qkv.H, qkv.N, qkv.d
    dev = qkv.q.device
    for t, nm in ((v, "v"), (dout, "dout"), (o, "o")):
        _check_out(t, (B, H, N, d), dev, f"sage3_int8_attn_bwd {nm}")
    if v.dtype != dout.dtype:
        raise Sage3Error("sage3_int8_attn_bwd: v and dout must share a dtype")
    if lse is None:
        raise Sage3Error("sage3_int8_attn_bwd: lse is required")
    _check_lse(lse, B * H * N, dev, "sage3_int8_attn_bwd")
    mk = lambda t: t if t is not None else torch.empty(B, H, N, d, dtype=grad_dtype, device=v.device)
    dq, dk, dv = mk(dq), mk(dk), mk(dv)
    for t, nm in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
        _check_out(t, (B, H, N, d), dev, f"sage3_int8_attn_bwd {nm}")
    if workspace is None:
        workspace = torch.empty(sage3_int8_bwd_workspace_bytes(B, H, N, d), dtype=torch.uint8, device=v.device)
    st = load().sage3_int8_attn_bwd(ctypes.byref(qkv.struct), _t4(v), _t4(o), _DT[o.dtype], _t4(dout), _DT[v.dtype],
                                    ctypes.c_void_p(lse.data_ptr()), 1 if causal else 0, float(softmax_scale),
                                    _t4(dq), _t4(dk), _t4(dv), _DT[dq.dtype], ctypes.c_void_p(workspace.data_ptr()),
                                    workspace.numel(), _stream(stream))
    _check(st, "sage3_int8_attn_bwd")
    return dq, dk, dv

