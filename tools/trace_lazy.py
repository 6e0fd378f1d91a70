"""Per-role timeline of the lazy-reference attention kernel (attn_lazy.cu) from a SAGE3_TRACE build.

  python tools/trace_lazy.py build/variants/libsage3_trace.so [N]
"""
import ctypes
import os
import sys

import numpy as np
import torch

lib = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
os.environ["SAGE3_LIB"] = lib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_11594_b200 as s3  # noqa: E402
import synth  # noqa: E402

Q, K, V = synth.make_qkv(1, 32, N, 128, seed=0, dtype=torch.bfloat16, device="cuda")
qkv = s3.sage3_quantize_qkv(Q, K, V)
o = torch.empty_like(Q)
for _ in range(3):
    s3.sage3_attn_fwd(qkv, o, p_quant="lazy")
torch.cuda.synchronize()
buf = np.zeros((2, 8, 128, 8), np.uint64)
L = s3.load()
L.sage3_debug_trace_copy_lazy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert L.sage3_debug_trace_copy_lazy(buf.ctypes.data, buf.nbytes) == 0
nkv = min(N // 128, 128)
t = buf[0].astype(np.int64)
t0 = t[5, 0, 0]
js = range(8, nkv - 4)


def d(role, k1, k0, jj):
    v = [t[role, j, k1] - t[role, j, k0] for j in jj if t[role, j, k1] and t[role, j, k0]]
    return np.mean(v) if v else 0


for par in (0, 1):
    r = 1 + par
    jj = [j for j in js if j % 2 == par]
    period = np.mean([t[r, j + 2, 0] - t[r, j, 0] for j in jj if j + 2 < nkv])
    print(f"softmax WG{par}: wait_S {d(r,1,0,jj):6.0f}  ld+pass1 {d(r,2,1,jj):6.0f}  chain {d(r,3,2,jj):6.0f}"
          f"  scales+wait_P {d(r,4,3,jj):6.0f}  pass2 {d(r,5,4,jj):6.0f}  period {period:6.0f}")
print(f"correction: wait_x {d(4,1,0,js):6.0f}  work {d(4,2,1,js):6.0f}  period {np.mean([t[4,j+1,0]-t[4,j,0] for j in js]):6.0f}")
print(f"S-MMA: wait_s_empty {d(5,1,0,js):6.0f}  wait_K {d(5,2,1,js):6.0f}  issue {d(5,3,2,js):6.0f}"
      f"  period {np.mean([t[5,j+1,0]-t[5,j,0] for j in js]):6.0f}")
print(f"PV-MMA: wait_P {d(6,1,0,js):6.0f}  wait_V {d(6,2,1,js):6.0f}  wait_o_ready {d(6,3,2,js):6.0f}  issue {d(6,4,3,js):6.0f}")
lat_s = [t[1 + j % 2, j, 1] - t[5, j, 3] for j in js if t[1 + j % 2, j, 0] < t[5, j, 3]]
print(f"S issue -> softmax wake (when waiting) {np.mean(lat_s) if lat_s else 0:6.0f} (n={len(lat_s)})")
lat_se = [t[5, j + 2, 1] - t[1 + j % 2, j, 2] for j in js if j + 2 < nkv]
print(f"softmax pass1 done (S_j free) -> S_(j+2) s_empty wake {np.mean(lat_se):6.0f}")
tot = t[4, nkv - 1, 2] - t0
print(f"span {tot} cycles / {nkv} tiles = {tot / nkv:.0f} cycles/tile")
for j in range(10, 16):
    sm = 1 + j % 2
    print(f" tile {j}: S {[int(x - t0) for x in t[5, j, :4]]} soft {[int(x - t0) for x in t[sm, j, :6]]}"
          f" corr {[int(x - t0) for x in t[4, j, :3]]} PV {[int(x - t0) for x in t[6, j, :5]]}")
