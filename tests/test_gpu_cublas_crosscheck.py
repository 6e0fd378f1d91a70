"""SURVEY §4 layer 5: a third implementation of the block-scaled FP4 product.  The bytes our quantizer writes
(E2M1 pairs, element 2k in the low nibble; E4M3 scales in 512-byte 128x4 SF atoms) are handed unchanged to
cuBLASLt's NVFP4 GEMM (torch._scaled_mm, VEC16_UE4M3 scales) as Q̂ K̂^T, and compared with the oracle's exact
FP4MM (Eq. 3) of the same codes decoded from those bytes.  Agreement validates the operand and
scale layouts the tcgen05 kernels consume against NVIDIA's own interpretation of them."""
import numpy as np
import pytest
import torch

import oracle
import paper_2505_11594_b200 as s3
import synth
from layout import decode_head

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,d", [(256, 128), (384, 64), (300, 128)])
def test_qk_fp4mm_bytes_agree_with_cublaslt(N, d):
    Q, K, V = synth.make_qkv(1, 1, N, d, seed=N + d, dtype=torch.bfloat16, device="cuda")
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    Np = qkv.N_pad
    a = qkv.q_data.view(Np, d // 2).view(torch.float4_e2m1fn_x2)
    b = qkv.k_data.view(Np, d // 2).view(torch.float4_e2m1fn_x2)
    sa = qkv.q_sf.view(torch.float8_e4m3fn)
    sb = qkv.k_sf.view(torch.float8_e4m3fn)
    S = torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.float32)
    torch.cuda.synchronize()
    h = decode_head(qkv, 0)
    ref = oracle.fp4mm(h["q_codes"], h["q_sf"], h["k_codes"], h["k_sf"])  # exact (fp64)
    got = S.double().cpu().numpy()
    # cuBLASLt accumulates in fp32: allow a few fp32 ulps of Σ|a||b| per entry
    bound = np.abs(oracle.dequant(h["q_codes"], h["q_sf"])) @ np.abs(oracle.dequant(h["k_codes"], h["k_sf"])).T
    tol = 8 * np.finfo(np.float32).eps * bound + 1e-30
    assert np.all(np.abs(got - ref) <= tol), np.abs(got - ref).max()
    print("max |cuBLASLt - oracle FP4MM| / bound:", float((np.abs(got - ref) / (bound + 1e-30)).max()))
