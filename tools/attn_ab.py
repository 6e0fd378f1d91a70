"""Same-box A/B of attention-kernel variants: each library (built with different -D flags) is loaded in its own
subprocess (SAGE3_LIB) and timed on the same inputs; the libraries alternate for `--reps` rounds.

    python tools/attn_ab.py build/lib_a.so build/lib_b.so [--shapes 32768:0,32768:1,1024:0] [--reps 2]

A variant may also be `lib.so@VAR=VAL[,VAR=VAL]`: the same library run with extra environment variables
(e.g. `paper_2505_11594_b200/libsage3.so@SAGE3_ATTN_KERNEL=3`).
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(shapes, d, heads, p_quant):
    sys.path.insert(0, ROOT)
    import torch

    import paper_2505_11594_b200 as s3
    import synth

    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    out = []
    for n, c in shapes:
        q, k, v = synth.make_qkv(1, heads, n, d, seed=1, dtype=torch.bfloat16, device=dev)
        f = s3.sage3_quantize_qkv(q, k, v, stream=st)
        o = torch.empty_like(q)
        ops = 4.0 * heads * n * n * d * (0.5 if c else 1.0)
        reps = max(5, int(3e13 / ops))
        for _ in range(3):
            s3.sage3_attn_fwd(f, o, causal=bool(c), stream=st, p_quant=p_quant)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        for _ in range(reps):
            s3.sage3_attn_fwd(f, o, causal=bool(c), stream=st, p_quant=p_quant)
        a1.record(st)
        torch.cuda.synchronize()
        ms = a0.elapsed_time(a1) / reps
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(st)
        s3.sage3_quantize_qkv(q, k, v, out=f, stream=st)
        t1.record(st)
        torch.cuda.synchronize()
        out.append({"N": n, "causal": c, "ms": round(ms, 4), "TOPS": round(ops / ms / 1e9, 1),
                    "quant_ms": round(t0.elapsed_time(t1), 4)})
    print("RESULT " + json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="*")
    ap.add_argument("--shapes", default="32768:0,32768:1,8192:0,1024:0,1024:1")
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--p-quant", default="two_level")
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    shapes = [tuple(int(x) for x in s.split(":")) for s in a.shapes.split(",")]
    if a.child:
        child(shapes, a.d, a.heads, a.p_quant)
        return
    res = {lib: [] for lib in a.libs}
    for _ in range(a.reps):
        for lib in a.libs:
            path, _, extra = lib.partition("@")
            env = dict(os.environ, SAGE3_LIB=os.path.abspath(path))
            env.update(kv.split("=", 1) for kv in extra.split(",") if kv)
            p = subprocess.run([sys.executable, __file__, "--child", "--shapes", a.shapes, "--d", str(a.d),
                                "--heads", str(a.heads), "--p-quant", a.p_quant], env=env, capture_output=True,
                               text=True, timeout=600)
            line = [x for x in p.stdout.splitlines() if x.startswith("RESULT ")]
            if not line:
                print(lib, "FAILED", p.stderr[-2000:])
                continue
            r = json.loads(line[0][7:])
            res[lib].append(r)
            print(os.path.basename(lib), " ".join(f"{x['N']}{'c' if x['causal'] else 'n'}:{x['TOPS']}" for x in r),
                  "q%.4f" % r[0]["quant_ms"], flush=True)
    print("SUMMARY (best of reps)")
    for lib, rs in res.items():
        if not rs:
            continue
        best = [max(r[i]["TOPS"] for r in rs) for i in range(len(shapes))]
        print(f"{os.path.basename(lib):28s}", " ".join(f"{n}{'c' if c else 'n'}:{b}" for (n, c), b in zip(shapes, best)))


if __name__ == "__main__":
    main()
