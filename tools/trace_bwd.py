"""Per-role timeline of the SageBwd backward kernel from a SAGE3_TRACE build (clock64 stamps, bwd_i8.cu).

  python tools/trace_bwd.py <libsage3_trace.so> [N]
Roles: 1 WG1 (element-wise), 2 MMA issuer, 3 TMA producer, 4 WG3 (dK, dQ flush), 5 WG2 (dV).
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

H, d = 32, 128
Q, K, V = synth.make_qkv(1, H, N, d, seed=0, dtype=torch.bfloat16, device="cuda")
dO = torch.randn_like(Q)
qkv = s3.sage3_int8_quantize_qkv(Q, K, V)
lse = torch.empty(1, H, N, dtype=torch.float32, device="cuda")
O = s3.sage3_int8_attn_fwd(qkv, causal=False, lse=lse)
for _ in range(3):
    s3.sage3_int8_attn_bwd(qkv, V, O, dO, lse)
torch.cuda.synchronize()
buf = np.zeros((2, 8, 128, 8), np.uint64)
L = s3.load()
L.sage3_debug_trace_copy_bwd.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert L.sage3_debug_trace_copy_bwd(buf.ctypes.data, buf.nbytes) == 0
nt = min(N // 128, 128)
names = {1: ["wait_q+S", "A+redA", "wait_dP/sp", "B", "redB", "wait_sds", "C"],
         2: ["S(t+1)", "dV(t)", "dKQ(t)", "dP(t+1)"], 3: ["wait_qe", "wait_doe", "wait_dq8e"],
         4: ["wait_kq", "dKp", "dQflush"], 5: ["wait_dvp", "dVacc"]}
sub = {4: [(2, 4, "flush0: ld+wait"), (4, 5, "flush0: compute+sts"), (5, 6, "flush0: fence"), (6, 3, "rest")]}
for cta in range(2):
    t = buf[cta].astype(np.int64)
    js = range(4, nt - 4)
    print(f"== CTA {cta}: tile period WG1 {np.mean([t[1, j + 1, 0] - t[1, j, 0] for j in js]):.0f} cycles")
    for role, nm in names.items():
        segs = []
        for k in range(len(nm)):
            v = [t[role, j, k + 1] - t[role, j, k] for j in js if t[role, j, k + 1] and t[role, j, k]]
            segs.append(f"{nm[k]} {np.mean(v):6.0f}" if v else f"{nm[k]} -")
        print(f"  role {role}: " + " | ".join(segs))
        for k0, k1, nm2 in sub.get(role, []):
            v = [t[role, j, k1] - t[role, j, k0] for j in js if t[role, j, k1] and t[role, j, k0]]
            print(f"      {nm2} {np.mean(v):6.0f}")
    # cross-role latencies
    lat = lambda a, b: np.mean([t[b[0], j + b[2], b[1]] - t[a[0], j, a[1]] for j in js])  # noqa: E731
    print(f"  ds_full(t) -> MMA dKQ issued {lat((1, 7, 0), (2, 3, 0)):6.0f};  dKQ issued -> WG3 kq {lat((2, 3, 0), (4, 1, 0)):6.0f};"
          f"  WG3 y_empty -> dP(t+1) issued {lat((4, 2, 0), (2, 4, 0)):6.0f};  dP issued -> WG1 B(t+1) start {lat((2, 4, 0), (1, 3, 1)):6.0f}")
