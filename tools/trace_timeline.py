"""Per-role timeline of the attention kernel from a SAGE3_TRACE build (clock64 stamps, see attn.cu).

  python tools/trace_timeline.py build/variants/libsage3_trace.so [N] [causal]
"""
import ctypes
import os
import sys

import numpy as np
import torch

lib = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
causal = len(sys.argv) > 3 and sys.argv[3] == "causal"
os.environ["SAGE3_LIB"] = lib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_11594_b200 as s3  # noqa: E402
import synth  # noqa: E402

Q, K, V = synth.make_qkv(1, 32, N, 128, seed=0, dtype=torch.bfloat16, device="cuda")
qkv = s3.sage3_quantize_qkv(Q, K, V)
o = torch.empty_like(Q)
for _ in range(3):
    s3.sage3_attn_fwd(qkv, o, causal=causal)
torch.cuda.synchronize()
buf = np.zeros((2, 8, 128, 8), np.uint64)
L = s3.load()
L.sage3_debug_trace_copy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert L.sage3_debug_trace_copy(buf.ctypes.data, buf.nbytes) == 0
nkv = N // 128 if not causal else N // 128
for cta in range(2):
    t = buf[cta].astype(np.int64)
    t0 = t[5, 0, 0]
    print(f"== CTA {cta} (cycles relative to first S issue)")
    def d(role, k1, k0, js):
        v = [t[role, j, k1] - t[role, j, k0] for j in js if t[role, j, k1] and t[role, j, k0]]
        return (np.mean(v), np.max(v)) if v else (0, 0)
    js = range(4, min(nkv, 128) - 4)
    for par in (0, 1):
        r = 1 + par
        jj = [j for j in js if j % 2 == par]
        period = np.mean([t[r, j + 2, 0] - t[r, j, 0] for j in jj if j + 2 < nkv and t[r, j + 2, 0]])
        print(f" softmax WG{par}: wait_S {d(r,1,0,jj)[0]:7.0f}  pass1+scales {d(r,2,1,jj)[0]:6.0f}  wait_P {d(r,3,2,jj)[0]:6.0f}"
              f"  pass2 {d(r,4,3,jj)[0]:6.0f}   tile period {period:7.0f}")
    print(f" correction: wait_x {d(4,1,0,js)[0]:6.0f}  wait_pv {d(4,2,1,js)[0]:6.0f}  compute {d(4,3,2,js)[0]:6.0f}"
          f"  period {np.mean([t[4,j+1,0]-t[4,j,0] for j in js]):6.0f}")
    print(f" S-MMA:  wait_buf {d(5,1,0,js)[0]:6.0f}  wait_K {d(5,2,1,js)[0]:6.0f}  issue {d(5,3,2,js)[0]:6.0f}")
    print(f" PV-MMA: wait_P {d(6,1,0,js)[0]:6.0f}  wait_V {d(6,2,1,js)[0]:6.0f}  issue {d(6,3,2,js)[0]:6.0f}")
    # latencies: S issued -> softmax sees it; P ready -> PV issued; PV issued -> correction sees it
    lat_s = [t[1 + j % 2, j, 1] - t[5, j, 3] for j in js if t[1 + j % 2, j, 0] < t[5, j, 3]]
    lat_pv = [t[4, j, 2] - t[6, j, 3] for j in js if t[4, j, 1] < t[6, j, 3]]
    lat_b = [t[5, j + 3, 1] - t[4, j, 3] for j in js if j + 3 < nkv and t[5, j + 3, 0] < t[4, j, 3]]
    print(f" latency S-issue->softmax wake {np.mean(lat_s) if lat_s else 0:6.0f} (n={len(lat_s)})"
          f"  PV-issue->correction wake {np.mean(lat_pv) if lat_pv else 0:6.0f} (n={len(lat_pv)})"
          f"  b_empty->S issue {np.mean(lat_b) if lat_b else 0:6.0f} (n={len(lat_b)})")
    nl = min(nkv, 128)
    tot = t[4, nl - 1, 3] - t0
    print(f" CTA span {tot} cycles for {nl} tiles = {tot / nl:.0f} cycles/tile")
    for j in (10, 11, 12):
        print(f"  tile {j}: S issued {t[5,j,3]-t0}, softmax start {t[1+j%2,j,1]-t0}, P ready {t[1+j%2,j,4]-t0},"
              f" PV issued {t[6,j,3]-t0}, corr pv-wake {t[4,j,2]-t0}, corr done {t[4,j,3]-t0}")

print("\nraw events CTA 0 (relative cycles): role: [k0 k1 k2 k3 k4]")
t = buf[0].astype(np.int64)
t0 = t[5, 0, 0]
for j in range(8, 15):
    sm = 1 + j % 2
    print(f" tile {j:2d} | S-MMA {[int(x - t0) for x in t[5, j, :4]]} | PV-MMA {[int(x - t0) for x in t[6, j, :4]]}"
          f" | softmax{sm-1} {[int(x - t0) for x in t[sm, j, :5]]} | corr {[int(x - t0) for x in t[4, j, :4]]}")

print("\nper-warp softmax completion (k4..k7 = warps 0..3 of the warpgroup, relative to the warpgroup's S wake):")
for j in range(8, 20):
    sm = 1 + j % 2
    w0 = t[sm, j, 1]
    print(f" tile {j:2d} WG{sm-1}: " + " ".join(f"{int(t[sm, j, 4 + w] - w0):6d}" for w in range(4)))

print("\nsoftmax sub-events (relative to the warpgroup's S wake k1): -, S loads waited, tmax, -, scales done, pass2-ld0-wait, pass2-ld3-wait, P ready")
for j in range(8, 20):
    sm = 1 + j % 2
    sub = 0 if sm == 1 else 3
    w0 = t[sm, j, 1]
    print(f" tile {j:2d} WG{sm-1}: " + " ".join(f"{int(t[sub, j, k] - w0):6d}" for k in range(7)) + f" {int(t[sm, j, 4] - w0):6d}")

print("\ncorrection pass 1 (role 7): s_full wait, loads+maxes, scales+stores, p_empty wait, SF store+arrive; then O update (role 4)")
for j in range(8, 20):
    e = t[7, j]
    if not e[0]:
        continue
    print(f" tile {j:2d}: start {int(e[0]-t0):7d}  wait_S {int(e[1]-e[0]):5d}  ld+max {int(e[2]-e[1]):5d}  scales {int(e[3]-e[2]):5d}"
          f"  wait_Pbuf {int(e[4]-e[3]):5d}  tail {int(e[5]-e[4]):5d} | O-upd({j-2}) row-wait {int(t[4,j-2,1]-t[4,j-2,0]):5d}"
          f" pv-wait {int(t[4,j-2,2]-t[4,j-2,1]):5d} compute {int(t[4,j-2,3]-t[4,j-2,2]):5d}")
