"""SURVEY §4 layer 2: the hardware converts the kernels use (cvt.rn.satfinite.e2m1x2.f32 /
cvt.rn.satfinite.e4m3x2.f32 on the B200) against the oracle's brute-force nearest encoders — exhaustively
over every non-NaN fp32 bit pattern for E2M1, and over every pattern with |x| in [2^-12, 2^10) plus a
1/256 sample of the rest for E4M3.  This pins the oracle's reading of "FP4 rounding" (readings c1, c2:
RNE, satfinite, sign kept on underflow) to the hardware's definition.  The converts come from a test-helper
kernel (tests/cuda/cvt_probe.cu, built by __graft_entry__.build()), not from the product library."""
import ctypes
import os

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _probe():
    path = os.path.join(HERE, "cuda", "libcvt_probe.so")
    if not os.path.exists(path):
        import sys

        sys.path.insert(0, os.path.dirname(HERE))
        import __graft_entry__

        __graft_entry__.build_test_helpers()
    lib = ctypes.CDLL(path)
    lib.probe_cvt.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
    return lib


def test_exhaustive_fp32_sweep_of_hardware_converts():
    lib = _probe()
    chunk = 1 << 26
    n_e4m3 = 0
    for c in range((1 << 32) // chunk):
        bits = torch.arange(c * chunk, (c + 1) * chunk, dtype=torch.int64, device="cuda").to(torch.int32)
        x = bits.view(torch.float32)
        e2 = torch.empty(chunk, dtype=torch.uint8, device="cuda")
        e4 = torch.empty(chunk, dtype=torch.uint8, device="cuda")
        assert lib.probe_cvt(x.data_ptr(), e2.data_ptr(), e4.data_ptr(), chunk, None) == 0
        torch.cuda.synchronize()
        xh = x.cpu().numpy()
        ok = ~np.isnan(xh)
        got = e2.cpu().numpy()
        want = oracle.e2m1_encode_array(np.ascontiguousarray(xh[ok]))
        bad = np.flatnonzero(got[ok] != want)
        assert bad.size == 0, (c, xh[ok][bad[:4]], got[ok][bad[:4]], want[bad[:4]])
        ub = bits.cpu().numpy().view(np.uint32)
        ex = (ub >> 23) & 0xFF
        sel = ok & (((ex >= 127 - 12) & (ex < 127 + 10)) | ((ub & 0xFF) == 0x5A))
        got4 = e4.cpu().numpy()[sel]
        want4 = oracle.e4m3_encode_array(np.ascontiguousarray(xh[sel]))
        bad = np.flatnonzero(got4 != want4)
        assert bad.size == 0, (c, xh[sel][bad[:4]], got4[bad[:4]], want4[bad[:4]])
        n_e4m3 += int(sel.sum())
    print("E4M3 patterns compared:", n_e4m3)
