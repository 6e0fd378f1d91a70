"""Per-role timeline of attn3.cu from a SAGE3_TRACE build (clock64 stamps, see attn3.cu A3_EV).

  python -c 'from paper_2505_11594_b200 import build as b; b.build(out="build/variants/libsage3_trace3.so",
             defines=["SAGE3_TRACE"], only=["attn3.cu"])'
  SAGE3_ATTN_KERNEL=3 python tools/trace_a3.py build/variants/libsage3_trace3.so [N] [causal]
Roles: 1-3 softmax WG (k0 wait S, k1 S ready, k2 pass 1 + scales done, k3 P̂2 published), 4 correction warp 0
(k0 start, k1 x ready, k2 PV ready, k3 done), 5 S issue (k0 entry, k1 buffer free, k2 K ready, k3 committed),
6 PV issue (k0 entry, k1 P ready, k2 V ready, k3 committed), 7 per-warp P̂2 publication (k = warp of the WG).
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
os.environ.setdefault("SAGE3_ATTN_KERNEL", "3")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_11594_b200 as s3  # noqa: E402
import synth  # noqa: E402

Q, K, V = synth.make_qkv(1, 32, N, 128, seed=0, dtype=torch.bfloat16, device="cuda")
qkv = s3.sage3_quantize_qkv(Q, K, V)
o = torch.empty_like(Q)
for _ in range(3):
    s3.sage3_attn_fwd(qkv, o, causal=causal)
torch.cuda.synchronize()
buf = np.zeros((2, 10, 128, 8), np.uint64)
L = s3.load()
L.sage3_debug_trace_copy3.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert L.sage3_debug_trace_copy3(buf.ctypes.data, buf.nbytes) == 0
nkv = min(N // 128, 128)
for cta in range(2):
    t = buf[cta].astype(np.int64)
    t0 = t[5, 12, 0]
    js = range(9, 36)

    def d(role, k1, k0, jj):
        v = [t[role, j, k1] - t[role, j, k0] for j in jj if t[role, j, k1] and t[role, j, k0]]
        return np.mean(v) if v else 0.0

    print(f"== CTA {cta}")
    for w in (1, 2, 3):
        jj = [j for j in js if j % 3 == w - 1]
        per = np.mean([t[w, j + 3, 1] - t[w, j, 1] for j in jj if j + 3 < nkv])
        print(f" softmax WG{w}: wait_S {d(w,1,0,jj):6.0f}  pass1+scales {d(w,2,1,jj):6.0f}  pass2+publish {d(w,3,2,jj):6.0f}"
              f"  cycle (3 tiles) {per:6.0f}")
    print(f" correction: wait_x {d(4,1,0,js):6.0f}  wait_pv {d(4,2,1,js):6.0f}  compute {d(4,3,2,js):6.0f}"
          f"  period {np.mean([t[4, j + 1, 0] - t[4, j, 0] for j in js]):6.0f}")
    print(f" S issue:  wait_buf {d(5,1,0,js):6.0f}  wait_K {d(5,2,1,js):6.0f}  issue {d(5,3,2,js):6.0f}")
    print(f" PV issue: wait_P {d(6,1,0,js):6.0f}  wait_V {d(6,2,1,js):6.0f}  issue {d(6,3,2,js):6.0f}")
    # the S-issue chain: softmax j publishes -> PV_j issued -> correction sees PV_j -> correction done -> S_{j+3}
    # issued -> softmax j+3 sees S
    ch = []
    for j in js:
        if j + 3 >= nkv:
            continue
        w = 1 + j % 3
        pub = t[7, j, :4].max()
        cdone = max(t[8 + k // 2, j, 4 * (k % 2) + 3] for k in range(4))  # last correction warp done with PV_j
        ch.append([t[6, j, 0] - pub, t[6, j, 3] - t[6, j, 0], t[4, j, 2] - t[6, j, 3],
                   cdone - t[4, j, 2], t[5, j + 3, 1] - cdone, t[5, j + 3, 3] - t[5, j + 3, 1],
                   t[1 + (j + 3) % 3, j + 3, 1] - t[5, j + 3, 3], pub - t[7, j, :4].min()])
    ch = np.array(ch).mean(0)
    print(" chain: last publish -> PV entry %.0f, PV issue %.0f, -> corr0 PV wake %.0f, -> last corr done %.0f,"
          " -> S leader wake %.0f, S issue %.0f, -> softmax wake %.0f; warp skew of publish %.0f" % tuple(ch))
    print(f" tiles 10..34: {(t[4, 34, 3] - t[4, 10, 3]) / 24:.0f} cycles/tile")
mm = [(t[6, j, 1] - t[6, j, 3], t[5, j, 4] - t[5, j, 3]) for j in range(12, 36) if t[6, j, 1] > t[6, j, 3] > 0]
if mm:
    print("\nMMA completion after commit (SAGE3_TRACE_MMA build): PV %.0f  S %.0f cycles" % tuple(np.mean(mm, 0)))
print("\nper-warp correction events (start, x ready, PV ready, done) relative to warp 0's start:")
for j in range(12, 19):
    base = t[8, j, 0]
    ev = [[int(t[8 + w // 2, j, 4 * (w % 2) + e] - base) for e in range(4)] for w in range(4)]
    print(f" tile {j:2d}: " + "  ".join(str(e) for e in ev))
print("\nraw CTA 0, relative cycles")
t = buf[0].astype(np.int64)
t0 = t[5, 12, 0]
for j in range(12, 19):
    w = 1 + j % 3
    print(f" tile {j:2d} | S {[int(x - t0) for x in t[5, j, :4]]} | PV {[int(x - t0) for x in t[6, j, :4]]}"
          f" | sm{w} {[int(x - t0) for x in t[w, j, :4]]} pub {[int(x - t0) for x in t[7, j, :4]]}"
          f" | corr {[int(x - t0) for x in t[4, j, :4]]}")
