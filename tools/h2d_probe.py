"""Raw pinned host <-> device copy bandwidth on this box, one direction at a time and both at once (the bound of
bench.py's e2e line, which moves 805 MB in and 268 MB out per step)."""
import torch

n = 805306368
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    with torch.cuda.stream(s):
        d.copy_(h, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


def both():
    h2d()
    d2h()


for name, fn, by in (("H2D", h2d, n), ("D2H", d2h, n), ("H2D+D2H concurrent", both, 2 * n)):
    ms = timed(fn)
    print(f"{name}: {by / ms / 1e6:.1f} GB/s ({ms:.2f} ms for {by / 1e6:.0f} MB)")
