"""Per-region stall breakdown of an ncu report's SASS source page.

Regions are split at USETMAXREG instructions (the warp-role entry points of the attention kernel):
prologue | WG0 (producers, MMA) | softmax | correction/epilogue.
usage: python tools/stall_regions.py report.ncu-rep [top_n_instructions]
"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = [r for r in csv.reader(out.splitlines())]
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
iS = h.index("Source")
iE = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "(Not Issued)" not in c]
idx = {c: h.index(c) for c in reasons}
names = ["prologue", "wg0", "softmax", "correction"]
region, cur = [], 0
for r in data:
    if "USETMAXREG" in r[iS]:
        cur = min(cur + 1, 3)
    region.append(cur)
for k in range(4):
    tot = collections.Counter()
    inst = 0
    for r, g in zip(data, region):
        if g != k:
            continue
        inst += int(r[iE] or 0)
        for c in reasons:
            tot[c] += int(r[idx[c]] or 0)
    s = sum(tot.values())
    print(f"== {names[k]}: {inst} warp-instr, {s} stall samples")
    for c, v in tot.most_common(8):
        print(f"   {c:24s} {v:8d} {100 * v / max(s, 1):5.1f}%")
    ranked = sorted(((sum(int(r[idx[c]] or 0) for c in reasons), r[iS].strip()) for r, g in zip(data, region) if g == k),
                    reverse=True)[:top]
    for v, src in ranked:
        print(f"      {v:7d}  {src[:90]}")
