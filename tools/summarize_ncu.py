"""Write the committed profile summaries under profiles/ from a round's gpurun_out/ captures.

usage: python tools/summarize_ncu.py <tag> <workload-name>
  reads  gpurun_out/<tag>_prof_attn.ncu-rep, gpurun_out/<tag>_prof_quant.ncu-rep, gpurun_out/<tag>_launches.csv
  writes profiles/<tag>_attn_ncu.txt, profiles/<tag>_quant_ncu.txt, profiles/<tag>_launches.txt,
         profiles/ncu_summary.json (read by bench.py for roofline.traffic)
"""
import collections
import csv
import json
import os
import subprocess
import sys

tag, workload = sys.argv[1], sys.argv[2]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
os.makedirs(P, exist_ok=True)

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_tma.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    kernels = []
    for v in rows[2:]:
        kernels.append({h[i]: (v[i], u[i]) for i in range(len(h))})
    return kernels


def stalls(k):
    items = [(float(v[0]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")) for n, v in k.items()
             if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued") and v[0] not in ("", "n/a")]
    tot = sum(x for x, _ in items) or 1
    return [(n, round(100 * x / tot, 1)) for x, n in sorted(items, reverse=True)[:10]]


def opcode_hist(rep, n=16):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    h = rows[1]
    iS, iE = h.index("Source"), h.index("Instructions Executed")
    c = collections.Counter()
    for r in rows[2:]:
        if len(r) == len(h):
            op = r[iS].split()
            op = (op[1] if op[0].startswith("@") and len(op) > 1 else op[0]) if op else "?"
            c[op] += int(r[iE] or 0)
    tot = sum(c.values()) or 1
    return [(op, v, round(100 * v / tot, 2)) for op, v in c.most_common(n)]


summary = {}
for kind in ("attn", "quant"):
    rep = os.path.join(G, f"{tag}_prof_{kind}.ncu-rep")
    if not os.path.exists(rep):
        continue
    lines = [f"ncu --set full summary ({tag}, {kind}); workload {workload}; source: {os.path.basename(rep)}"]
    for k in raw(rep):
        name = k.get("Kernel Name", ("?",))[0]
        lines.append(f"\n== {name}")
        for key in KEYS:
            if key in k:
                lines.append(f"  {key:70s} {k[key][0]:>18s} {k[key][1]}")
        lines.append("  stall reasons (% of samples): " + ", ".join(f"{n} {p}" for n, p in stalls(k)))
        rd = float(k["dram__bytes_read.sum"][0]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(k["dram__bytes_read.sum"][1], 1)
        wr = float(k["dram__bytes_write.sum"][0]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(k["dram__bytes_write.sum"][1], 1)
        if kind == "attn":
            summary["attn_fwd"] = {"workload": workload, "dram_bytes_per_launch": rd + wr, "kernel": name, "tag": tag}
        else:
            summary.setdefault("quantize", []).append({"kernel": name, "dram_bytes": rd + wr})
    if kind == "attn":
        lines.append("\nSASS opcode histogram (executed warp instructions):")
        for op, v, pct in opcode_hist(rep):
            lines.append(f"  {op:45s} {v:14d} {pct:6.2f}%")
    open(os.path.join(P, f"{tag}_{kind}_ncu.txt"), "w").write("\n".join(lines) + "\n")

lc = os.path.join(G, f"{tag}_launches.csv")
if os.path.exists(lc):
    rows = [r for r in csv.reader(open(lc)) if len(r) > 5]
    h = rows[0]
    iN, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    t = collections.defaultdict(list)
    for r in rows[1:]:
        if r[iM] == "gpu__time_duration.sum":
            t[r[iN]].append(float(r[iV].replace(",", "")))
    tot = sum(sum(v) for v in t.values())
    lines = [f"ncu launch list ({tag}; --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised;"
             " compare shares, not absolutes). Command: bench.py --steps 2 --warmup 3 (5 steps of 4 launches each"
             " + the synthetic-input generation kernels)",
             f"{'kernel':90s} {'launches':>8s} {'mean_us':>10s} {'share%':>7s}"]
    for name, v in sorted(t.items(), key=lambda x: -sum(x[1])):
        lines.append(f"{name[:90]:90s} {len(v):8d} {sum(v) / len(v) / 1e3:10.2f} {100 * sum(v) / tot:7.2f}")
    open(os.path.join(P, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")

json.dump(summary, open(os.path.join(P, "ncu_summary.json"), "w"), indent=1)
print(json.dumps(summary, indent=1))
