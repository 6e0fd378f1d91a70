"""Summarise an ncu report: per-opcode executed instructions and stall samples (SASS source page)."""
import csv, collections, re, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ops, stall, total, tstall = collections.Counter(), collections.Counter(), 0, 0
for r in rows[2:]:
    if len(r) < len(h):
        continue
    src = r[iS].strip()
    n, w = int(r[iE] or 0), int(r[iW] or 0)
    op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
    ops[op] += n; stall[op] += w; total += n; tstall += w
print("total warp instr", total, "stall samples", tstall)
for op, n in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{op:45s} {n:14d} {n/total*100:6.2f}%  stall {stall[op]/max(tstall,1)*100:5.1f}%")
