"""CPU oracle for the SageAttention3 FP4 attention forward (arXiv 2505.11594, Algorithm 1).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product package
(``paper_2505_11594_b200``) never imports it, and the two share no code.

The arithmetic lives in ``sage3_oracle.c`` (plain C, fp64 except where the paper fixes fp32); this
module is a ctypes binding plus the paper's accuracy metrics (Appendix).  Every function
documents the passage it follows; readings of ambiguous points are SURVEY.md §8(c) c1-c16, copied into
DESIGN.md §3.

Parity status: codecs, φ, K-mean, FP4MM, two-level P and the online-softmax recurrence
are each pinned by tests/test_oracle_*.py to tables, closed forms, library routines or the plain
definition of attention.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sage3_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "sagebwd_oracle.c")]  # + SageBwd, Alg 2-3 (NEXT #3)
_LIB = os.path.join(_HERE, "liboracle.so")
_CFLAGS = ["-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC"]
_lock = threading.Lock()
_lib = None

PMODE_TWO_LEVEL, PMODE_DIRECT, PMODE_NONE, PMODE_LAZY, PMODE_QSUM = 0, 1, 2, 3, 4  # LAZY, QSUM: NEXT #2 variants (readings n1, n2)


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no fast-math, no FMA contraction, no FTZ/DAZ)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(f) for f in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.run(["gcc", *_CFLAGS, *_SRCS, "-o", tmp, "-lm"], check=True)
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build())
            u8p = ctypes.POINTER(ctypes.c_uint8)
            fp = ctypes.POINTER(ctypes.c_float)
            dp = ctypes.POINTER(ctypes.c_double)
            ip = ctypes.POINTER(ctypes.c_int)
            L.oracle_e2m1_encode.restype = ctypes.c_uint8
            L.oracle_e2m1_encode.argtypes = [ctypes.c_float]
            L.oracle_e2m1_decode.restype = ctypes.c_double
            L.oracle_e2m1_decode.argtypes = [ctypes.c_uint8]
            L.oracle_e4m3_encode.restype = ctypes.c_uint8
            L.oracle_e4m3_encode.argtypes = [ctypes.c_float]
            L.oracle_e4m3_decode.restype = ctypes.c_double
            L.oracle_e4m3_decode.argtypes = [ctypes.c_uint8]
            L.oracle_enumerate.restype = ctypes.c_int
            L.oracle_enumerate.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, dp]
            L.oracle_phi_nvfp4.argtypes = [fp, u8p, u8p]
            L.oracle_phi_mxfp4.argtypes = [fp, u8p, u8p]
            L.oracle_kmean.argtypes = [fp, ctypes.c_int, ctypes.c_int, fp]
            L.oracle_quantize_head.argtypes = [fp, fp, fp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                               u8p, u8p, u8p, u8p, u8p, u8p, fp]
            L.oracle_quantize_head_sq.argtypes = [fp, fp, fp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                  u8p, u8p, u8p, u8p, u8p, u8p, fp, fp, fp]
            L.oracle_quantize_head_fmt.argtypes = [fp, fp, fp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                   ctypes.c_int, u8p, u8p, u8p, u8p, u8p, u8p, fp, fp, fp]
            L.oracle_attn_fwd_fmt.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p, u8p, u8p, u8p, u8p, u8p,
                                              fp, fp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                              ctypes.c_int, ip, ctypes.c_int, dp, dp]
            L.oracle_attn_fwd_amb.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p, u8p, u8p, u8p, u8p, u8p,
                                              fp, fp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                              ctypes.c_int, ip, ctypes.c_int, dp, dp, ctypes.c_double, dp]
            L.oracle_dequant_fmt.argtypes = [u8p, u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp]
            L.oracle_qmean_tile.argtypes = [fp, ctypes.c_int, ctypes.c_int, ctypes.c_int, fp]
            L.oracle_attn_fwd_sq.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p, u8p, u8p, u8p, u8p, u8p,
                                             fp, fp, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int, ip,
                                             ctypes.c_int, dp, dp]
            L.oracle_dequant.argtypes = [u8p, u8p, ctypes.c_int, ctypes.c_int, dp]
            L.oracle_fp4mm.argtypes = [u8p, u8p, u8p, u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp]
            L.oracle_two_level_row.restype = ctypes.c_float
            L.oracle_two_level_row.argtypes = [fp, ctypes.c_int, ctypes.c_int, u8p, u8p]
            L.oracle_attn_fwd.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p, u8p, u8p, u8p, u8p, u8p,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int, ip,
                                          ctypes.c_int, dp, dp]
            L.oracle_attn_fwd_float.argtypes = [ctypes.c_int, ctypes.c_int, fp, fp, fp, ctypes.c_int, ctypes.c_int,
                                                ctypes.c_double, ctypes.c_int, ip, ctypes.c_int, dp, dp]
            L.oracle_reference_attention.argtypes = [ctypes.c_int, ctypes.c_int, fp, fp, fp, ctypes.c_int,
                                                     ctypes.c_double, ip, ctypes.c_int, dp]
            L.oracle_num_threads.restype = ctypes.c_int
            L.oracle_e2m1_encode_array.argtypes = [fp, ctypes.c_int64, u8p]
            i8p = ctypes.POINTER(ctypes.c_int8)
            L.sb_psi.restype = ctypes.c_float
            L.sb_psi.argtypes = [fp, ctypes.c_int, ctypes.c_int, i8p]
            L.sb_quantize_head.argtypes = [fp, fp, fp, ctypes.c_int, ctypes.c_int, i8p, i8p, i8p, fp, fp, fp, fp]
            L.sb_attn_fwd.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, i8p, i8p, i8p, fp, fp, fp,
                                      ctypes.c_int, ctypes.c_double, ip, ctypes.c_int, dp, dp]
            L.sb_attn_fwd_amb.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, i8p, i8p, i8p, fp, fp, fp,
                                      ctypes.c_int, ctypes.c_double, ip, ctypes.c_int, dp, dp, ctypes.c_double, dp]
            L.sb_bwd_head.argtypes = [ctypes.c_int, ctypes.c_int, i8p, i8p, fp, fp, fp, fp, fp, fp, fp,
                                      ctypes.c_int, ctypes.c_double, dp, dp, dp]
            L.oracle_e4m3_encode_array.argtypes = [fp, ctypes.c_int64, u8p]
            _lib = L
    return _lib


def _p(a: np.ndarray, ct):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


# ---------------------------------------------------------------------------------------- codecs
def e2m1_encode(x: float) -> int:
    """E2M1 round-to-nearest-even, saturating, sign kept (reading c1)."""
    return int(lib().oracle_e2m1_encode(float(np.float32(x))))


def e2m1_decode(c: int) -> float:
    return float(lib().oracle_e2m1_decode(int(c)))


def e4m3_encode(x: float) -> int:
    """E4M3 round-to-nearest-even, saturating at 448, never NaN (reading c2)."""
    return int(lib().oracle_e4m3_encode(float(np.float32(x))))


def e4m3_decode(c: int) -> float:
    return float(lib().oracle_e4m3_decode(int(c)))


def e2m1_encode_array(x) -> np.ndarray:
    x = _f32(x).ravel()
    out = np.zeros(x.shape[0], np.uint8)
    lib().oracle_e2m1_encode_array(_p(x, ctypes.c_float), x.shape[0], _p(out, ctypes.c_uint8))
    return out


def e4m3_encode_array(x) -> np.ndarray:
    x = _f32(x).ravel()
    out = np.zeros(x.shape[0], np.uint8)
    lib().oracle_e4m3_encode_array(_p(x, ctypes.c_float), x.shape[0], _p(out, ctypes.c_uint8))
    return out


def enumerate_values(fmt: str, lo: float, hi: float) -> np.ndarray:
    """Distinct representable values in [lo, hi] (appendix)."""
    out = np.zeros(256, dtype=np.float64)
    n = lib().oracle_enumerate(0 if fmt == "e2m1" else 1, lo, hi, _p(out, ctypes.c_double))
    return out[:n].copy()


def phi_nvfp4(x) -> tuple[np.ndarray, int]:
    """φ on one 1x16 block (Eq. 1): returns (16 E2M1 codes, E4M3 scale code)."""
    x = _f32(x)
    assert x.shape == (16,)
    codes = np.zeros(16, dtype=np.uint8)
    sc = np.zeros(1, dtype=np.uint8)
    lib().oracle_phi_nvfp4(_p(x, ctypes.c_float), _p(codes, ctypes.c_uint8), _p(sc, ctypes.c_uint8))
    return codes, int(sc[0])


def phi_mxfp4(x) -> tuple[np.ndarray, int]:
    """MXFP4 ablation φ on one 1x32 block (E8M0 rounded up)."""
    x = _f32(x)
    assert x.shape == (32,)
    codes = np.zeros(32, dtype=np.uint8)
    sc = np.zeros(1, dtype=np.uint8)
    lib().oracle_phi_mxfp4(_p(x, ctypes.c_float), _p(codes, ctypes.c_uint8), _p(sc, ctypes.c_uint8))
    return codes, int(sc[0])


def e2m1_table() -> np.ndarray:
    return np.array([e2m1_decode(c) for c in range(16)])


def e4m3_table() -> np.ndarray:
    return np.array([e4m3_decode(c) for c in range(256)])


def dequant_fmt(codes: np.ndarray, sf: np.ndarray, fmt: int) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    sf = np.ascontiguousarray(sf, dtype=np.uint8)
    out = np.zeros(codes.shape, np.float64)
    lib().oracle_dequant_fmt(_p(codes, ctypes.c_uint8), _p(sf, ctypes.c_uint8), codes.shape[0], codes.shape[1], fmt,
                             _p(out, ctypes.c_double))
    return out


def dequant(codes: np.ndarray, sf: np.ndarray) -> np.ndarray:
    """φ^-1 (Eq. 2) for codes [R][C] with scales [R][C/16]; exact fp64."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    sf = np.ascontiguousarray(sf, dtype=np.uint8)
    R, C = codes.shape
    out = np.zeros((R, C), dtype=np.float64)
    lib().oracle_dequant(_p(codes, ctypes.c_uint8), _p(sf, ctypes.c_uint8), R, C, _p(out, ctypes.c_double))
    return out


def fp4mm(a_codes, a_sf, b_codes, b_sf) -> np.ndarray:
    """FP4MM (Eq. 3): φ^-1(A) φ^-1(B)^T, A [M][K], B [N][K] (both blocked along K)."""
    a_codes = np.ascontiguousarray(a_codes, dtype=np.uint8)
    b_codes = np.ascontiguousarray(b_codes, dtype=np.uint8)
    a_sf = np.ascontiguousarray(a_sf, dtype=np.uint8)
    b_sf = np.ascontiguousarray(b_sf, dtype=np.uint8)
    M, K = a_codes.shape
    N = b_codes.shape[0]
    out = np.zeros((M, N), dtype=np.float64)
    lib().oracle_fp4mm(_p(a_codes, ctypes.c_uint8), _p(a_sf, ctypes.c_uint8), _p(b_codes, ctypes.c_uint8),
                       _p(b_sf, ctypes.c_uint8), M, N, K, _p(out, ctypes.c_double))
    return out


def two_level_row(P, p_mode: int = PMODE_TWO_LEVEL):
    """Two-level quantization of one row of P̃ (§3.2): returns (s_P1, codes, s_P2 codes)."""
    P = _f32(P)
    n = P.shape[0]
    codes = np.zeros(n, dtype=np.uint8)
    sf = np.zeros(n // 16, dtype=np.uint8)
    s = lib().oracle_two_level_row(_p(P, ctypes.c_float), n, p_mode, _p(codes, ctypes.c_uint8),
                                   _p(sf, ctypes.c_uint8))
    return float(np.float32(s)), codes, sf


def kmean(K) -> np.ndarray:
    """Smoothing-K mean (Alg1 L2) in the fixed order of reading c10."""
    K = _f32(K)
    N, d = K.shape
    km = np.zeros(d, dtype=np.float32)
    lib().oracle_kmean(_p(K, ctypes.c_float), N, d, _p(km, ctypes.c_float))
    return km


FMT_NVFP4, FMT_MXFP4 = 0, 1  # E4M3 scales per 16 (the method) / E8M0 scales per 32 (Tab1a ablation)


class QuantizedHead:
    """Logical-layout FP4 codes of one head (one code per byte): q/k [Np][d], v [d][Np]; fmt NVFP4 or MXFP4."""

    def __init__(self, N, d, fmt: int = FMT_NVFP4):
        Np = (N + 127) // 128 * 128
        G = 32 if fmt == FMT_MXFP4 else 16
        self.N, self.d, self.Np, self.fmt = N, d, Np, fmt
        self.q_codes = np.zeros((Np, d), np.uint8)
        self.k_codes = np.zeros((Np, d), np.uint8)
        self.v_codes = np.zeros((d, Np), np.uint8)
        self.q_sf = np.zeros((Np, d // G), np.uint8)
        self.k_sf = np.zeros((Np, d // G), np.uint8)
        self.v_sf = np.zeros((d, Np // G), np.uint8)
        self.km = np.zeros(d, np.float32)
        self.q_mean = None  # smoothing Q (Alg1 L5): [Np/128][d] fp32 q̄ per 128-row query tile
        self.ks = None      # smoothing Q: the full-precision smoothed K [Np][d] of Alg1 L8's GEMV


def quantize_head(Q, K, V, smooth_k: bool = True, smooth_q: bool = False, fmt: int = FMT_NVFP4) -> QuantizedHead:
    """Alg1 L2 (smoothing K), L5 (smoothing Q, optional) + φ of Q, K (along d) and V (along tokens, stored
    transposed); fmt = FMT_MXFP4 for the Tab1a data-type ablation."""
    Q, K, V = _f32(Q), _f32(K), _f32(V)
    N, d = Q.shape
    h = QuantizedHead(N, d, fmt)
    u8, fp = ctypes.c_uint8, ctypes.c_float
    if smooth_q:
        h.q_mean = np.zeros((h.Np // 128, d), np.float32)
        h.ks = np.zeros((h.Np, d), np.float32)
    lib().oracle_quantize_head_fmt(_p(Q, fp), _p(K, fp), _p(V, fp), N, d, 1 if smooth_k else 0,
                                  1 if smooth_q else 0, fmt, _p(h.q_codes, u8), _p(h.q_sf, u8), _p(h.k_codes, u8),
                                  _p(h.k_sf, u8), _p(h.v_codes, u8), _p(h.v_sf, u8), _p(h.km, fp),
                                  _p(h.q_mean, fp) if smooth_q else None, _p(h.ks, fp) if smooth_q else None)
    return h


def qmean_tile(Q, tile: int) -> np.ndarray:
    """q̄ of one 128-row query tile (Alg1 L5), in the fixed order of reading c10."""
    Q = _f32(Q)
    N, d = Q.shape
    out = np.zeros(d, np.float32)
    lib().oracle_qmean_tile(_p(Q, ctypes.c_float), N, d, tile, _p(out, ctypes.c_float))
    return out


def attn_fwd(heads: list[QuantizedHead], *, causal: bool, scale: float, rows=None, bkv: int = 128,
             p_mode: int = PMODE_TWO_LEVEL, want_lse: bool = False, amb_delta: float | None = None):
    """Alg1 L6-L13 on quantized heads (all same N, d; smoothing Q iff the heads carry q_mean/ks).
    Returns O [BH][nrows][d] fp64 (and lse).  With amb_delta: also amb [BH][nrows][d], the bound on how far O
    can move when every P quantization decision is re-taken on values within a relative amb_delta (test
    infrastructure for the GPU parity bound; see oracle_attn_fwd_amb).  Returns (O, lse, amb) then."""
    N, d, Np = heads[0].N, heads[0].d, heads[0].Np
    BH = len(heads)
    rows = np.arange(N, dtype=np.int32) if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    cat = lambda name: np.ascontiguousarray(np.stack([getattr(h, name) for h in heads]))
    qc, qs, kc, ks, vc, vs = (cat(n) for n in ("q_codes", "q_sf", "k_codes", "k_sf", "v_codes", "v_sf"))
    sq = heads[0].q_mean is not None
    qm, kf = (cat("q_mean"), cat("ks")) if sq else (None, None)
    O = np.zeros((BH, rows.shape[0], d), np.float64)
    lse = np.zeros((BH, rows.shape[0]), np.float64)
    amb = np.zeros((BH, rows.shape[0], d), np.float64) if amb_delta is not None else None
    u8, fp = ctypes.c_uint8, ctypes.c_float
    lib().oracle_attn_fwd_amb(BH, N, d, _p(qc, u8), _p(qs, u8), _p(kc, u8), _p(ks, u8), _p(vc, u8), _p(vs, u8),
                              _p(qm, fp) if sq else None, _p(kf, fp) if sq else None, heads[0].fmt, bkv,
                              1 if causal else 0,
                              float(scale), p_mode, _p(rows, ctypes.c_int), rows.shape[0], _p(O, ctypes.c_double),
                              _p(lse, ctypes.c_double), float(amb_delta or 0.0),
                              _p(amb, ctypes.c_double) if amb is not None else None)
    if amb is not None:
        return O, lse, amb
    return (O, lse) if want_lse else O


def attn_fwd_float(Q, K, V, *, causal: bool, scale: float, rows=None, bkv: int = 128,
                   p_mode: int = PMODE_NONE, want_lse: bool = False):
    """The same tiled recurrence on unquantized inputs (p_mode NONE = FlashAttention in fp64)."""
    Q, K, V = _f32(Q), _f32(K), _f32(V)
    N, d = Q.shape
    rows = np.arange(N, dtype=np.int32) if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    O = np.zeros((rows.shape[0], d), np.float64)
    lse = np.zeros(rows.shape[0], np.float64)
    fp = ctypes.c_float
    lib().oracle_attn_fwd_float(N, d, _p(Q, fp), _p(K, fp), _p(V, fp), bkv, 1 if causal else 0, float(scale),
                                p_mode, _p(rows, ctypes.c_int), rows.shape[0], _p(O, ctypes.c_double),
                                _p(lse, ctypes.c_double))
    return (O, lse) if want_lse else O


def reference_attention(Q, K, V, *, causal: bool, scale: float, rows=None) -> np.ndarray:
    """Plain fp64 softmax attention on the original inputs, for the accuracy metrics."""
    Q, K, V = _f32(Q), _f32(K), _f32(V)
    N, d = Q.shape
    rows = np.arange(N, dtype=np.int32) if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    O = np.zeros((rows.shape[0], d), np.float64)
    fp = ctypes.c_float
    lib().oracle_reference_attention(N, d, _p(Q, fp), _p(K, fp), _p(V, fp), 1 if causal else 0, float(scale),
                                     _p(rows, ctypes.c_int), rows.shape[0], _p(O, ctypes.c_double))
    return O


def num_threads() -> int:
    return int(lib().oracle_num_threads())


# ---------------------------------------------------------------------------------------- metrics
def accuracy_metrics(ref, test) -> dict:
    """Appendix metrics: CosSim = ΣOO'/(√ΣO²√ΣO'²), L1 = Σ|O-O'|/Σ|O|, RMSE = √(mean (O-O')²)."""
    a = np.asarray(ref, dtype=np.float64).ravel()
    b = np.asarray(test, dtype=np.float64).ravel()
    cos = float(np.dot(a, b) / (np.sqrt(np.dot(a, a)) * np.sqrt(np.dot(b, b))))
    l1 = float(np.abs(a - b).sum() / np.abs(a).sum())
    rmse = float(np.sqrt(np.mean((a - b) ** 2)))
    return {"cos_sim": cos, "l1": l1, "rmse": rmse}


# ------------------------------------------------------------------------------ SageBwd (NEXT #3)
class SbHead:
    """One head of SageBwd's INT8 per-block quantization (Alg2 L2 + L4): q, k, v int8 [Np][d], one fp32 scale
    per 128-token block (sq, sk, sv [Np/128]), the smooth-K mean km [d]."""

    def __init__(self, N, d):
        Np = (N + 127) // 128 * 128
        self.N, self.d, self.Np = N, d, Np
        self.q = np.zeros((Np, d), np.int8)
        self.k = np.zeros((Np, d), np.int8)
        self.v = np.zeros((Np, d), np.int8)
        self.sq = np.zeros(Np // 128, np.float32)
        self.sk = np.zeros(Np // 128, np.float32)
        self.sv = np.zeros(Np // 128, np.float32)
        self.km = np.zeros(d, np.float32)


def sb_psi(x) -> tuple[np.ndarray, float]:
    """ψ of one block (reading b1): (int8 codes, scale)."""
    x = _f32(x).reshape(-1)
    q = np.zeros(x.shape[0], np.int8)
    s = lib().sb_psi(_p(x, ctypes.c_float), x.shape[0], 1, _p(q, ctypes.c_int8))
    return q, float(s)


def sb_quantize_head(Q, K, V) -> SbHead:
    """Alg2 L2 (smooth-K) + L4 (ψ per 128-token block of Q, K, V) for one head of 16-bit values."""
    Q, K, V = _f32(Q), _f32(K), _f32(V)
    N, d = Q.shape
    h = SbHead(N, d)
    lib().sb_quantize_head(_p(Q, ctypes.c_float), _p(K, ctypes.c_float), _p(V, ctypes.c_float), N, d,
                           _p(h.q, ctypes.c_int8), _p(h.k, ctypes.c_int8), _p(h.v, ctypes.c_int8),
                           _p(h.sq, ctypes.c_float), _p(h.sk, ctypes.c_float), _p(h.sv, ctypes.c_float),
                           _p(h.km, ctypes.c_float))
    return h


def sb_attn_fwd(heads: list[SbHead], *, causal: bool, scale: float, rows=None, want_lse: bool = False,
                amb_delta: float | None = None):
    """Alg2 L6-L14 on quantized heads: O [BH][nrows][d] fp64 (and lse = scale·m + ln l).  With amb_delta also the
    decision-sensitivity bound amb [BH][nrows][d] (test infrastructure, see sb_attn_fwd_amb): returns (O, lse, amb)."""
    N, d, Np = heads[0].N, heads[0].d, heads[0].Np
    rows = np.arange(N, dtype=np.int32) if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    cat = lambda name: np.ascontiguousarray(np.concatenate([getattr(h, name) for h in heads]))  # noqa: E731
    q, k, v, sq, sk, sv = (cat(n) for n in ("q", "k", "v", "sq", "sk", "sv"))
    O = np.zeros((len(heads), len(rows), d), np.float64)
    lse = np.zeros((len(heads), len(rows)), np.float64)
    amb = np.zeros_like(O) if amb_delta is not None else None
    lib().sb_attn_fwd_amb(len(heads), N, d, _p(q, ctypes.c_int8), _p(k, ctypes.c_int8), _p(v, ctypes.c_int8),
                          _p(sq, ctypes.c_float), _p(sk, ctypes.c_float), _p(sv, ctypes.c_float), int(causal),
                          float(scale), _p(rows, ctypes.c_int), len(rows), _p(O, ctypes.c_double),
                          _p(lse, ctypes.c_double), float(amb_delta or 0.0),
                          _p(amb, ctypes.c_double) if amb is not None else None)
    if amb is not None:
        return O, lse, amb
    return (O, lse) if want_lse else O


def sb_attn_bwd(h: SbHead, V16, O, dO, L, *, causal: bool, scale: float):
    """Alg3 for one head: (dQ, dK, dV) [N][d] fp64.  V16 = the 16-bit V values (dP = dO·Vᵀ stays unquantized,
    P:329), O / L = the forward's output and lse, dO the incoming gradient."""
    V16, O, dO, L = _f32(V16), _f32(O), _f32(dO), _f32(L)
    N, d = h.N, h.d
    dQ, dK, dV = (np.zeros((N, d), np.float64) for _ in range(3))
    lib().sb_bwd_head(N, d, _p(h.q, ctypes.c_int8), _p(h.k, ctypes.c_int8), _p(h.sq, ctypes.c_float),
                      _p(h.sk, ctypes.c_float), _p(h.km, ctypes.c_float), _p(V16, ctypes.c_float),
                      _p(O, ctypes.c_float), _p(dO, ctypes.c_float), _p(L, ctypes.c_float), int(causal),
                      float(scale), _p(dQ, ctypes.c_double), _p(dK, ctypes.c_double), _p(dV, ctypes.c_double))
    return dQ, dK, dV
