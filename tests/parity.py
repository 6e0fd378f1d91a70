"""GPU-vs-oracle attention parity checks, shared by every GPU attention test.

Two gates, both on the SAME quantized codes (the oracle is fed either the GPU's decoded codes, after the
quantizer was asserted bit-exact, or its own quantize_head output):

1. north_star, per head: rel-L1 <= 2e-3 and cosine >= 0.9999 against the oracle rounded to the output dtype.
2. element-wise, every element:
       |gpu - round(oracle)| <= ulp_dtype + TIGHT * vmax + 1.01 * amb
   * ulp_dtype: one spacing of the output dtype at the element (both sides were rounded once);
   * TIGHT * vmax: fp32 accumulation order (S and PV on the tensor core, O += w PV, l) against fp64, relative
     to vmax = max |deq(V̂)| of the head, which bounds every convex combination of V rows;
   * amb: the oracle's decision-sensitivity bound (oracle.attn_fwd(amb_delta=AMB_DELTA)): the largest move of
     the element if every P quantization decision whose input lies within a relative AMB_DELTA of a rounding
     boundary were taken the other way.  The GPU evaluates P̃2 = 2688·2^(sl2(S - tmax)) with fp32 S from the
     tensor core, an FFMA2 exponent argument and MUFU/polynomial exp2; its values differ from the oracle's
     fp32 P̃2 by less than AMB_DELTA (relative), so only those decisions can legitimately differ.
   No row's allowance may exceed AMB_REL_MAX of the row's largest |O|, so the bound cannot go vacuous.
"""
import numpy as np
import torch

import oracle

REL_L1_MAX = 2e-3
COS_MIN = 0.9999
TIGHT = 2e-5
# Calibrated on the B200 (tools/parity_diag.py, profiles/r2_parity_calibration.txt): every GPU-vs-oracle
# difference above the tight part is covered from delta = 4e-6 on (N up to 32K, two-level and lazy); 1e-5 keeps a
# 2.5x margin.
AMB_DELTA = 1e-5
AMB_REL_MAX = 0.25  # no row's allowance may exceed this fraction of the row's largest |O|

_MANT = {torch.float32: 23, torch.bfloat16: 7, torch.float16: 10}


def round_to(x: np.ndarray, dtype) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(x)).to(dtype).double().numpy()


def dtype_spacing(x: np.ndarray, dtype) -> np.ndarray:
    """Spacing of `dtype` at |x| (normal range; the smallest normal's spacing below it)."""
    m = _MANT[dtype]
    tiny = {torch.float32: 2.0 ** -126, torch.bfloat16: 2.0 ** -126, torch.float16: 2.0 ** -14}[dtype]
    a = np.maximum(np.abs(x), tiny)
    return np.exp2(np.floor(np.log2(a)) - m)


def check(gpu: np.ndarray, ref: np.ndarray, dtype, what="", amb=None, vmax=None):
    """gpu, ref, amb: [rows, d] of one head.  Returns the north_star metrics."""
    r = round_to(ref, dtype)
    g = np.asarray(gpu, np.float64)
    assert np.all(np.isfinite(g)), f"{what}: non-finite output"
    m = oracle.accuracy_metrics(r, g)
    assert m["l1"] <= REL_L1_MAX and m["cos_sim"] >= COS_MIN, f"{what}: {m}"
    if amb is not None:
        vm = float(vmax) if vmax is not None else float(np.abs(ref).max())
        bound = dtype_spacing(np.maximum(np.abs(g), np.abs(r)), dtype) + TIGHT * vm + 1.01 * np.asarray(amb)
        err = np.abs(g - r)
        bad = np.argwhere(err > bound)
        assert bad.size == 0, (f"{what}: {len(bad)} elements outside the element-wise bound; first (row, col) "
                               f"{bad[:4].tolist()}: gpu {g[tuple(bad[0])]!r} oracle {ref[tuple(bad[0])]!r} "
                               f"err {err[tuple(bad[0])]:.3e} bound {bound[tuple(bad[0])]:.3e}")
        amb = np.asarray(amb)
        rel = float(np.max(amb.max(axis=1) / np.maximum(np.abs(ref).max(axis=1), 1e-30))) if amb.size else 0.0
        assert rel <= AMB_REL_MAX, f"{what}: a row's decision allowance reaches {rel:.2f} of its largest |O|"
        m["amb_rows"] = float(np.mean(amb.max(axis=1) > 0)) if amb.size else 0.0
        m["max_err_over_tight"] = float(np.max(err / (dtype_spacing(np.maximum(np.abs(g), np.abs(r)), dtype)
                                                      + TIGHT * vm))) if err.size else 0.0
    return m


def vmax_of(head) -> float:
    """max |deq(V̂)| of an oracle QuantizedHead (FP4 codes x block scales)."""
    return float(np.abs(oracle.dequant_fmt(head.v_codes, head.v_sf, head.fmt)).max())


def oracle_attention(heads, *, causal, scale, rows=None, p_mode=None, want_lse=False, bkv=128):
    """oracle.attn_fwd with the decision-sensitivity output; returns (O, lse, amb, vmax per head)."""
    kw = {} if p_mode is None else {"p_mode": p_mode}
    kw["bkv"] = bkv
    O, lse, amb = oracle.attn_fwd(heads, causal=causal, scale=scale, rows=rows, amb_delta=AMB_DELTA, **kw)
    return O, lse, amb, [vmax_of(h) for h in heads]
