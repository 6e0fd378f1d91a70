"""Static SASS opcode histogram per warp-role region of the attention kernel (split at USETMAXREG).

usage: python tools/region_hist.py <libsage3.so> [D=128] [top]
"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1]
D = sys.argv[2] if len(sys.argv) > 2 else "128"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
start = sass.index(f"attn_fwd_kernelILi{D}E")
body = sass[start:]
end = body.find("Function :", 10)
body = body[: end if end > 0 else None]
regions, cur = collections.defaultdict(collections.Counter), 0
names = ["prologue", "wg0", "softmax", "correction+tail"]
for line in body.splitlines():
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(.*?);", line)
    if not m:
        continue
    ins = m.group(1)
    op = re.sub(r"^@!?U?P\w+\s+", "", ins).split(" ")[0]
    if "USETMAXREG" in op:
        cur = min(cur + 1, 3)
    regions[names[cur]][op] += 1
for n in names:
    c = regions[n]
    print(f"== {n}: {sum(c.values())} instructions")
    print("   " + ", ".join(f"{op} {k}" for op, k in c.most_common(top)))
