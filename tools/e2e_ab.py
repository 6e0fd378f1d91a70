"""Same-box A/B of the host-buffer path (sage3_forward_host) across library builds: TOPS end to end at the bench
shape (B=1, H=32, N=32768, d=128, pinned host buffers).  python tools/e2e_ab.py libA.so libB.so ..."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import torch

    import paper_2505_11594_b200 as s3
    import synth

    B, H, N, d = 1, 32, 32768, 128
    Q, K, V = synth.make_qkv(B, H, N, d, seed=0, dtype=torch.bfloat16, device="cuda")
    qh, kh, vh = (x.cpu().pin_memory() for x in (Q, K, V))
    oh = torch.empty(B, H, N, d, dtype=torch.bfloat16).pin_memory()
    scratch = torch.empty(s3.sage3_forward_host_scratch_bytes(B, H, N, d), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(2):
        s3.sage3_forward_host(qh, kh, vh, oh, scratch, stream=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(8):
        s3.sage3_forward_host(qh, kh, vh, oh, scratch, stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 8
    print("RESULT", json.dumps({"ms": ms, "TOPS": 4 * B * H * N * N * d / ms / 1e9}))
    sys.exit(0)
for rep in range(2):
    for lib in sys.argv[1:]:
        p = subprocess.run([sys.executable, __file__, "--child"], env=dict(os.environ, SAGE3_LIB=os.path.abspath(lib)),
                           capture_output=True, text=True)
        line = [x for x in p.stdout.splitlines() if x.startswith("RESULT")]
        print(os.path.basename(lib), line[0][7:] if line else p.stderr[-500:], flush=True)
