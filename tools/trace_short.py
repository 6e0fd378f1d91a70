"""Per-CTA fill / steady / drain breakdown of the FP4 attention kernel at short N (SAGE3_TRACE build).

  python tools/trace_short.py <libsage3_trace.so> [N]
"""
import ctypes
import os
import sys

import numpy as np
import torch

lib = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
os.environ["SAGE3_LIB"] = lib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_11594_b200 as s3  # noqa: E402
import synth  # noqa: E402

Q, K, V = synth.make_qkv(1, 32, N, 128, seed=0, dtype=torch.bfloat16, device="cuda")
qkv = s3.sage3_quantize_qkv(Q, K, V)
o = torch.empty_like(Q)
for _ in range(3):
    s3.sage3_attn_fwd(qkv, o)
torch.cuda.synchronize()
buf = np.zeros((2, 8, 128, 8), np.uint64)
L = s3.load()
L.sage3_debug_trace_copy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert L.sage3_debug_trace_copy(buf.ctypes.data, buf.nbytes) == 0
nkv = min(N // 128, 128)
for cta in range(2):
    t = buf[cta].astype(np.int64)
    t0 = t[0, 127, 0]
    r = lambda x: int(x - t0)  # noqa: E731
    print(f"== CTA {cta} (N={N}, {nkv} KV tiles), cycles from CTA start:")
    print(f"  prologue done {r(t[0,127,1])}; first S issued {r(t[5,0,3])}; softmax0 S wake {r(t[1,0,1])}, P ready {r(t[1,0,4])};"
          f" PV0 issued {r(t[6,0,3])}; correction tile0 done {r(t[4,0,3])}")
    print(f"  last tile: S issued {r(t[5,nkv-1,3])}; P ready {r(t[1 + (nkv-1)%2, nkv-1, 4])}; correction done {r(t[4,nkv-1,3])};"
          f" epilogue stores {r(t[4,127,2])}; all done {r(t[0,127,3])}")
    print(f"  epilogue: loop exit {r(t[4,126,0])}, normalized {r(t[4,126,1])}, staged {r(t[4,126,2])}, barrier {r(t[4,126,3])}")
    steady = (t[4, nkv - 1, 3] - t[4, 0, 3]) / max(nkv - 1, 1)
    print(f"  per-tile (correction done spacing) {steady:.0f}")
