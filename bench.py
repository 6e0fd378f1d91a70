#!/usr/bin/env python3
"""Benchmark of the SageAttention3 FP4 attention forward hot path on B200 (BASELINE.json metric:
"FP4 attention fwd TOPS per B200 (d=128, N=1K-32K) and % of dense FP4 peak").

A step = one pass of the whole hot path over one batch of synthetic input:
sage3_quantize_qkv (K mean, φ of Q, K, Vᵀ) + sage3_attn_fwd (FP4 QKᵀ, online softmax, two-level P,
FP4 PV, O/l).  Ops = 4·B·H·N²·d (halved for causal), counted per step on every rank.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--n 32768] [--causal] [--impl reference]

Multi-GPU: one process per GPU.  `--gpus N` re-executes itself under torch.distributed.run (127.0.0.1) when
not already launched by it.  The path shards by (b·h, query-tile) units with no data exchange
(multigpu.ShardPlan); the timed step is every rank's units of a (N·32)-head problem (weak scaling: 32 heads per
GPU), time = max over ranks.  Off the timed step: the launcher's per-head pipelined path with its final gather
to rank 0, and the C4 strong-scaling block (BASELINE configs[3], 24 heads split over the GPUs).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

FP4_OVER_BF16 = 9.0 / 2.25  # nominal dense FP4 : BF16 tensor ratio (B200_PROFILING.md nominal table)
FALLBACK_HBM_GBS, FALLBACK_BF16_TFLOPS = 6650.0, 1590.0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return j["hbm_gbs"], j["bf16_tflops"], "measured (MEASURED_PEAKS.json)"
    return FALLBACK_HBM_GBS, FALLBACK_BF16_TFLOPS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def attn_ops(B, H, N, d, causal):
    ops = 4.0 * B * H * N * N * d
    return ops / 2 if causal else ops


def cpu_baseline(args, d, timeout_s=12.0):
    """The oracle as it stands (oracle/, plain C fp64 + OpenMP) on a bounded sample of the workload: quantize
    head 0, then Algorithm 1 for R query rows of it, extrapolated (linear in rows) to the whole head."""
    import numpy as np

    import oracle

    N = args.n
    q, k, v = synth.make_head(N, d, seed=0, b=0, h=0, H=args.heads, dtype=torch.bfloat16, device="cpu")
    Q, K, V = (x.float().numpy() for x in (q, k, v))
    nthr = oracle.num_threads()
    t0 = time.perf_counter()
    h = oracle.quantize_head(Q, K, V, fmt=oracle.FMT_MXFP4 if getattr(args, "fmt", "nvfp4") == "mxfp4" else
                             oracle.FMT_NVFP4)
    tq = time.perf_counter() - t0
    # grow the row sample until one timed call takes about timeout_s (or covers all rows)
    R = max(4 * nthr, 16)
    while True:
        rows = np.linspace(0, N - 1, min(R, N)).astype(np.int32)
        t0 = time.perf_counter()
        oracle.attn_fwd([h], causal=args.causal, scale=1 / math.sqrt(d), rows=rows)
        ta = time.perf_counter() - t0
        if ta >= 0.5 * timeout_s or R >= N:
            break
        R = int(R * min(8.0, timeout_s / max(ta, 1e-3)))
    R = len(rows)
    # extrapolated to the whole head (the oracle's cost is linear in query rows): quantize the head once, then
    # Algorithm 1 for all N rows at the measured per-row time; ops of the whole head (halved when causal)
    t_head = tq + ta * N / R
    ops = attn_ops(1, 1, N, d, args.causal)
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"value": ops / t_head / 1e12, "unit": "TOPS", "cores": nthr, "kind": "oracle", "cpu_model": model,
            "extrapolated": True,
            "sample": f"oracle_quantize_head on head 0 ({tq:.2f} s) + Alg1 for {R} evenly spaced query rows of head 0 "
                      f"at N={N}, d={d} ({ta:.2f} s); extrapolated to the whole head (quantize + N rows = "
                      f"{t_head:.1f} s); TOPS = 4*N^2*d{'/2' if args.causal else ''} / that time",
            "seconds": ta + tq}


def run_reference(args):
    """--impl reference: the oracle timed as the reference arm (bounded sample per step)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    d = 128
    steps = []
    for _ in range(args.warmup):
        cpu_baseline(args, d, timeout_s=4.0)
    for _ in range(args.steps):
        steps.append(cpu_baseline(args, d, timeout_s=8.0))
    val = statistics.median(s["value"] for s in steps)
    cb = dict(steps[-1])
    cb["value"] = val
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "TOPS", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.median(s["seconds"] for s in steps) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 (oracle)",
        "data": "synthetic", "config": workload_config(args, d),
        "cpu_baseline": cb, "e2e": {"value": val, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# our kernels per step: kmean_kernel, kmean_final_kernel, quant_stream_kernel (sage3_quantize_qkv) + attn_fwd_kernel
# (+ smooth_q_ds_kernel with --smooth-q)
LAUNCHES_PER_STEP = 4
METRIC = "FP4 attention fwd TOPS per B200 (d=128, N=1K-32K) and % of dense FP4 peak"


def workload_config(args, d):
    name = f"B=1,H={args.heads},N={args.n},d={d},{'causal' if args.causal else 'non-causal'}"
    if getattr(args, "smooth_q", False):
        name += ",smooth-q"
    if getattr(args, "fmt", "nvfp4") != "nvfp4":
        name += "," + args.fmt
    if getattr(args, "p_quant", "two_level") != "two_level":
        name += ",p-" + args.p_quant
    return {"workload": name, "B": 1, "H": args.heads, "N": args.n, "d": d, "causal": bool(args.causal),
            "per_rank": True, "parallelism": f"heads-sharded x{args.gpus}",
            "l2": "inputs larger than L2 (3 x %.0f MB bf16 vs 126 MB)" % (args.heads * args.n * d * 2 / 1e6)}


def fp64_metrics(Q, K, V, O, rows, causal, d):
    """The paper's accuracy metrics (CosSim, relative L1, RMSE) of the step's output O against plain
    fp64 softmax attention on the original inputs, on sampled query rows of one head (host, torch fp64)."""
    q = Q.double().cpu()[rows]
    k, v = K.double().cpu(), V.double().cpu()
    s = (q @ k.T) / math.sqrt(d)
    if causal:
        s = s.masked_fill(torch.arange(k.shape[0])[None, :] > torch.as_tensor(rows)[:, None], float("-inf"))
    ref = torch.softmax(s, dim=-1) @ v
    o = O.double().cpu()[rows]
    a, b = ref.flatten(), o.flatten()
    return {"cos_sim": float(a @ b / (a.norm() * b.norm())), "l1": float((a - b).abs().sum() / a.abs().sum()),
            "rmse": float(((a - b) ** 2).mean().sqrt()), "rows": len(rows), "head": 0,
            "reference": "fp64 softmax attention on the bf16 inputs (torch, host)"}


def probe_traffic(args):
    """--probe-traffic (run under ncu by measure_traffic): one quantize + attention at the bench shape."""
    import paper_2505_11594_b200 as s3

    dev = torch.device("cuda", 0)
    Q, K, V = synth.make_qkv(1, args.heads, args.n, 128, seed=0, dtype=torch.bfloat16, device=dev)
    qkv = s3.sage3_quantize_qkv(Q, K, V)
    O = torch.empty_like(Q)
    s3.sage3_attn_fwd(qkv, O, causal=args.causal, p_quant=args.p_quant)
    torch.cuda.synchronize()


def measure_traffic(args):
    """DRAM bytes (read + write) of one attention launch at the bench shape, measured in this run by ncu on a
    child process (--probe-traffic).  None if ncu is unavailable or fails."""
    import shutil
    import subprocess

    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control", "none", "-k",
           "regex:attn_fwd", "-c", "1", "--csv", sys.executable, os.path.abspath(__file__), "--probe-traffic",
           "--n", str(args.n), "--heads", str(args.heads), "--p-quant", args.p_quant] + (["--causal"] if args.causal else [])
    try:
        p = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    except Exception as e:  # noqa: BLE001
        return None, f"ncu failed: {e}"
    import csv

    tot, unit_scale = 0.0, {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    rows = [r for r in csv.reader(l for l in p.stdout.splitlines() if l.startswith('"'))]
    if len(rows) < 2:
        return None, "ncu produced no metrics: " + (p.stderr or p.stdout)[-300:].replace("\n", " ")
    h = rows[0]
    try:
        iM, iU, iV = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    except ValueError:
        return None, "unexpected ncu csv"
    for r in rows[1:]:
        if r[iM] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(r[iV].replace(",", "")) * unit_scale.get(r[iU], 1)
    return (tot if tot > 0 else None), "ncu dram__bytes_read.sum + dram__bytes_write.sum, one launch, this run"


def strong_c4(args, s3, multigpu, rank, world, dev, stream):
    """BASELINE configs[3] (HunyuanVideo-shaped: B=1, H=24, N=118800, d=128, non-causal) split over this run's
    GPUs (strong scaling: fixed total work).  Per GPU: this rank's units as one quantize + one unit-range attention
    launch (device time, max over ranks); then the launcher's per-head pipelined path (compute head by head, each
    finished head's rows sent to rank 0 while the next computes) timed end to end with the gather."""
    B, H, N, d = 1, 24, 118800, 128
    plan = multigpu.ShardPlan(B, H, N, False, world, rank)
    nh = plan.h1 - plan.h0
    Q = torch.empty(1, nh, N, d, dtype=torch.bfloat16, device=dev)
    K, V = torch.empty_like(Q), torch.empty_like(Q)
    for i in range(nh):
        Q[0, i], K[0, i], V[0, i] = synth.make_head(N, d, seed=0, b=0, h=plan.h0 + i, H=H, dtype=torch.bfloat16,
                                                    device=dev)
    qkv = s3.FP4QKV(1, nh, N, d, dev)
    O = torch.empty_like(Q)
    lo, hi = plan.u0 - plan.h0 * plan.T, plan.u1 - plan.h0 * plan.T

    def step():
        s3.sage3_quantize_qkv(Q, K, V, out=qkv, stream=stream)
        s3.sage3_attn_fwd_units(qkv, O, lo, hi, stream=stream)

    def timed(fn, reps):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / reps], device=dev)
        ts = [t.clone() for _ in range(world)] if world > 1 else [t]
        if world > 1:
            torch.distributed.all_gather(ts, t)
        return [x.item() for x in ts]

    step()
    per_rank = timed(step, 3)
    head_in = lambda h, n: (Q[:, h - plan.h0: h - plan.h0 + n], K[:, h - plan.h0: h - plan.h0 + n],
                            V[:, h - plan.h0: h - plan.h0 + n])
    pipe = lambda: multigpu.pipelined_forward_gather(plan, d, head_in, None, dtype=torch.bfloat16, device=dev)
    pipe()
    wall = timed(pipe, 2)
    ops = 4.0 * B * H * N * N * d
    tmax = max(per_rank)
    del Q, K, V, O, qkv
    torch.cuda.empty_cache()
    return {"config": "C4 HunyuanVideo-shaped B=1,H=24,N=118800,d=128,non-causal", "scaling": "strong",
            "gpus": world, "heads_per_gpu": [e - s for s, e in
                                             ((r0 // plan.T, (r1 - 1) // plan.T + 1) for r0, r1 in plan.ranges)],
            "units_per_gpu": [e - s for s, e in plan.ranges],
            "ms_compute_per_gpu": [round(x, 3) for x in per_rank], "ms_compute_max": round(tmax, 3),
            "tops_compute": ops / (tmax * 1e-3) / 1e12,
            "ms_with_pipelined_gather": round(max(wall), 3),
            "tops_with_gather": ops / (max(wall) * 1e-3) / 1e12,
            "gather_bytes_into_rank0": int(B * H * N * d * 2 * (world - 1) / world) if world > 1 else 0,
            "balance": sum(per_rank) / (world * tmax),
            "note": "strong-scaling efficiency = ms_compute_max(1 GPU) / (G * ms_compute_max(G GPUs)) across runs"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--causal", action="store_true")
    ap.add_argument("--impl", default="sage3", choices=["sage3", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-strong", action="store_true", help="skip the C4 strong-scaling block")
    ap.add_argument("--no-traffic", action="store_true", help="skip the ncu DRAM-traffic probe of the attention")
    ap.add_argument("--probe-traffic", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--smooth-q", action="store_true", help="Alg1 with smoothing Q (NEXT #1; off on the north_star path)")
    ap.add_argument("--fmt", default="nvfp4", choices=["nvfp4", "mxfp4"],
                    help="FP4 format: nvfp4 (the method) or mxfp4 (Tab1a data-type ablation, NEXT #4)")
    ap.add_argument("--p-quant", default="two_level", choices=["two_level", "direct", "lazy", "qsum"],
                    help="P quantization: two_level (the method), direct (Tab1b ablation, NEXT #4), lazy / qsum "
                         "(NEXT #2 variants)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.probe_traffic:
        probe_traffic(args)
        return

    from paper_2505_11594_b200 import multigpu

    # one process per GPU: re-executes under torch.distributed.run when --gpus N > 1 and not already launched
    multigpu.self_launch(args.gpus, sys.argv[1:], os.path.abspath(__file__))
    import paper_2505_11594_b200 as s3

    if int(os.environ.get("WORLD_SIZE", "1")) > 1:  # NCCL's init log (transport, NVLS) on stderr, for the record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    rank, world, local = multigpu.init_from_env("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = torch.distributed if world > 1 else None
    d, B, H, N, causal = 128, 1, args.heads, args.n, args.causal
    # weak scaling: a (world·H)-head problem split by the launcher's unit plan; with equal heads every rank's
    # unit range is exactly H whole heads (global ids rank·H .. rank·H + H - 1), generated on this GPU only
    plan = multigpu.ShardPlan(B, H * world, N, causal, world, rank)
    assert plan.h1 - plan.h0 == H and plan.u1 - plan.u0 == H * plan.T, (plan.ranges, H)
    Q = torch.empty(B, H, N, d, dtype=torch.bfloat16, device=dev)
    K, V = torch.empty_like(Q), torch.empty_like(Q)
    for i in range(H):
        Q[0, i], K[0, i], V[0, i] = synth.make_head(N, d, seed=0, b=0, h=plan.h0 + i, H=H * world,
                                                    dtype=torch.bfloat16, device=dev)
    qkv = s3.FP4QKV(B, H, N, d, dev, smooth_q=args.smooth_q, fmt=args.fmt)
    O = torch.empty(B, H, N, d, dtype=torch.bfloat16, device=dev)
    stream = torch.cuda.current_stream(dev)
    u_lo, u_hi = plan.u0 - plan.h0 * plan.T, plan.u1 - plan.h0 * plan.T  # this rank's units, local numbering

    n_steps = args.steps
    ev_q = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_steps)]
    ev_a = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_steps)]

    def step(i=None):
        if i is not None:
            ev_q[i][0].record(stream)
        s3.sage3_quantize_qkv(Q, K, V, out=qkv, stream=stream)
        if i is not None:
            ev_q[i][1].record(stream)
            ev_a[i][0].record(stream)
        s3.sage3_attn_fwd_ex(qkv, O, causal=causal, stream=stream, p_quant=args.p_quant, unit_begin=u_lo,
                             unit_end=u_hi)
        if i is not None:
            ev_a[i][1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t_start.record(stream)
        for i in range(n_steps):
            step(i)
        t_end.record(stream)
        torch.cuda.synchronize()
    elapsed_ms = t_start.elapsed_time(t_end)
    if dist:
        t = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = t.item()
        dist.barrier()
    torch.cuda.synchronize()
    ms_step = elapsed_ms / n_steps
    ops_rank = attn_ops(B, H, N, d, causal)
    value = ops_rank * world / (ms_step * 1e-3) / 1e12
    q_ms = statistics.mean(a.elapsed_time(b) for a, b in ev_q)
    a_ms = statistics.mean(a.elapsed_time(b) for a, b in ev_a)
    # paper metrics of this step's output on sampled rows of the first head
    acc = None
    if rank == 0:
        rows = torch.linspace(0, N - 1, 64).long().tolist()
        acc = fp64_metrics(Q[0, 0], K[0, 0], V[0, 0], O[0, 0], rows, causal, d)

    # the launcher's product path once more with its final gather (off the timed step): head by head, every finished
    # head's O rows sent to rank 0 while the next head computes (NCCL point-to-point over NVLink)
    gather = None
    if args.fmt == "nvfp4" and args.p_quant == "two_level" and not args.smooth_q:
        head_in = lambda h, n: (Q[:, h - plan.h0: h - plan.h0 + n], K[:, h - plan.h0: h - plan.h0 + n],
                                V[:, h - plan.h0: h - plan.h0 + n])
        run = lambda: multigpu.pipelined_forward_gather(plan, d, head_in, None, dtype=torch.bfloat16, device=dev)
        run()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        run()
        g1.record(stream)
        torch.cuda.synchronize()
        gms = g0.elapsed_time(g1)
        if dist:
            t = torch.tensor([gms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            gms = t.item()
        gather = {"ms_per_head_compute_plus_gather": gms, "ms_step": ms_step,
                  "bytes_into_rank0": (world - 1) * O.numel() * O.element_size(),
                  "path": "multigpu.pipelined_forward_gather (per-head sage3_quantize_qkv + sage3_attn_fwd_units, "
                          "isend/irecv of each finished head to rank 0)"}

    hbm_gbs, bf16_tf, peak_src = peaks()
    fp4_peak = bf16_tf * FP4_OVER_BF16
    cfg = workload_config(args, d)
    cfg["parallelism"] = f"(b*h, q-tile) units x{world} (weak: {H} heads per GPU)"
    attn_tflops = ops_rank / (a_ms * 1e-3) / 1e12
    traffic, traffic_src = (None, "skipped (--no-traffic)")
    if rank == 0 and world == 1 and not args.no_traffic:
        traffic, traffic_src = measure_traffic(args)
    # the timed instantiation (csrc/attn.cu: D, kSQ, kMX, kDirect, kEarly (N >= 4K), kQSum, kMC; d = 64 with causal masking
    # or N >= 8K runs attn3.cu's attn3_fwd_kernel<64>)
    if args.p_quant == "lazy":
        kname = "attn_lazy_kernel (csrc/attn_lazy.cu)"
    elif d == 64 and (args.causal or N >= 8192) and args.p_quant in ("two_level",) and not args.smooth_q \
            and args.fmt == "nvfp4":
        kname = "attn3_fwd_kernel<64>"
    else:
        kname = "attn_fwd_kernel<%d, %d, %d, %d, %d, %d, 0>" % (d, int(args.smooth_q), int(args.fmt == "mxfp4"),
                                                                 int(args.p_quant == "direct"),
                                                                 int(N >= 4096 and args.p_quant != "direct"),
                                                                 int(args.p_quant == "qsum"))
    roofline = {"bound": "tensor", "kernel": kname,
                "achieved": attn_tflops, "peak": fp4_peak,
                "unit": "TFLOP/s", "frac": attn_tflops / fp4_peak, "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_bytes": B * H * N * d * (3 * 0.5 + 3 / 16 + 2),
                "peak_source": f"{peak_src}: bf16_tflops {bf16_tf} x {FP4_OVER_BF16:g} (nominal dense FP4:BF16)",
                "algorithmic": "4*B*H*N^2*d (x0.5 causal) per launch / mean CUDA-event launch time"}
    E = B * H * N * d
    q_bytes = E * (3 * 2) + E * 3 * (0.5 + (1 / 32 if args.fmt == "mxfp4" else 1 / 16))  # read bf16; write codes + scales
    quant = {"ms": q_ms, "algorithmic_bytes": q_bytes, "achieved_GBps": q_bytes / (q_ms * 1e-3) / 1e9,
             "peak_GBps": hbm_gbs, "frac": q_bytes / (q_ms * 1e-3) / 1e9 / hbm_gbs, "bound": "hbm"}

    # ---- e2e: the same step through the C-ABI host-buffer entry point (H2D + quantize + attn + D2H)
    e2e = None
    if not args.no_e2e and args.fmt == "nvfp4" and args.p_quant == "two_level" and not args.smooth_q:
        qh, kh, vh = (x.cpu().pin_memory() for x in (Q, K, V))
        oh = torch.empty(B, H, N, d, dtype=torch.bfloat16).pin_memory()
        scratch = torch.empty(s3.sage3_forward_host_scratch_bytes(B, H, N, d), dtype=torch.uint8, device=dev)
        for _ in range(2):
            s3.sage3_forward_host(qh, kh, vh, oh, scratch, causal=causal, stream=stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        k_e2e = max(3, min(n_steps, 10))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k_e2e):
            s3.sage3_forward_host(qh, kh, vh, oh, scratch, causal=causal, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = t.item()
        e2e = {"value": ops_rank * world / (ems / k_e2e * 1e-3) / 1e12, "unit": "TOPS",
               "ms_per_step": ems / k_e2e, "h2d_bytes_per_step": 3 * E * 2, "d2h_bytes_per_step": E * 2,
               "api": "sage3_forward_host (pinned host buffers)"}
        del scratch

    # ---- attention-only sweep over the metric's N range (device-timed, this GPU)
    sweep = None
    if not args.no_sweep and rank == 0:
        sweep = []
        for n in (1024, 2048, 4096, 8192, 16384, 32768):
            for c in (False, True):
                q2, k2, v2 = synth.make_qkv(1, H, n, d, seed=1, dtype=torch.bfloat16, device=dev)
                f = s3.sage3_quantize_qkv(q2, k2, v2, stream=stream, fmt=args.fmt)
                o2 = torch.empty_like(q2)
                reps = max(3, int(2e13 / attn_ops(1, H, n, d, c) / 50))
                for _ in range(3):
                    s3.sage3_attn_fwd(f, o2, causal=c, stream=stream, p_quant=args.p_quant)
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                for _ in range(reps):
                    s3.sage3_attn_fwd(f, o2, causal=c, stream=stream, p_quant=args.p_quant)
                a1.record(stream)
                torch.cuda.synchronize()
                ms = a0.elapsed_time(a1) / reps
                tops = attn_ops(1, H, n, d, c) / (ms * 1e-3) / 1e12
                sweep.append({"N": n, "causal": c, "attn_ms": round(ms, 4), "attn_TOPS": round(tops, 1),
                              "pct_fp4_peak": round(100 * tops / fp4_peak, 2)})
                del q2, k2, v2, f, o2

    strong = None
    if not args.no_strong and args.fmt == "nvfp4" and args.p_quant == "two_level" and not args.smooth_q:
        del qkv
        torch.cuda.empty_cache()
        strong = strong_c4(args, s3, multigpu, rank, world, dev, stream)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args, d)
            cpu.pop("seconds", None)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "TOPS", "cores": None, "kind": "oracle", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": world, "steps": n_steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None,
            "dtype": ("nvfp4 (e2m1 codes, e4m3 1x16 scales)" if args.fmt == "nvfp4" else
                      "mxfp4 (e2m1 codes, e8m0 1x32 scales)") + ", fp32 accumulate; bf16 in/out",
            "data": "synthetic (seeded Gaussian Q/K/V with outlier channels; synth/)",
            "config": cfg, "pct_fp4_peak": 100 * value / world / fp4_peak,
            "breakdown_ms": {"quantize": q_ms, "attention": a_ms},
            "clocks": clk.summary(), "e2e": e2e, "gpu_launches": (LAUNCHES_PER_STEP + args.smooth_q) * n_steps,
            "launches_per_step": LAUNCHES_PER_STEP + args.smooth_q,
            "accuracy_vs_fp64": acc,
            "roofline": roofline, "quantize_roofline": quant, "cpu_baseline": cpu, "sweep": sweep,
            "final_gather": gather, "strong_scaling_c4": strong,
            "gpus_requested": args.gpus,
            "context": {"paper_RTX5090_TOPS": 1038, "paper_B200_theoretical_TOPS": 10000},
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
