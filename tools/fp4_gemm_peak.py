"""Practical dense FP4 tensor peak on this B200: cuBLASLt NVFP4 GEMM through
torch._scaled_mm (E2M1 operands, E4M3 scales per 16 elements, fp32 accumulate, bf16 out), M=N=K=8192.
Prints one JSON line.  (Library GEMM: a measurement reference, not part of the product path.)"""
import json
import sys

import torch


def main():
    M = N = K = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    dev = torch.device("cuda")
    a = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
    b = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
    # one E4M3 scale per 16 elements along K, in cuBLAS's blocked (128x4 atom) layout
    sa = torch.full((M * K // 16,), 1.0, device=dev).to(torch.float8_e4m3fn)
    sb = torch.full((N * K // 16,), 1.0, device=dev).to(torch.float8_e4m3fn)
    f = lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"what": "cuBLASLt NVFP4 GEMM via torch._scaled_mm", "M": M, "N": N, "K": K, "ms": ms,
                      "tflops": 2.0 * M * N * K / (ms * 1e-3) / 1e12}))


if __name__ == "__main__":
    main()
