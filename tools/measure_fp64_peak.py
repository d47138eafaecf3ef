"""Measure the FP64 (and complex128) GEMM peak of the local GPU with cuBLAS via torch.

Used once to add an FP64 denominator next to MEASURED_PEAKS.json (which only
records HBM and bf16); the result is written to profiles/fp64_peak.json.
"""
import json
import os
import sys
import time

import torch


def bench(dtype, n, iters=10):
    a = torch.randn(n, n, dtype=dtype, device="cuda")
    b = torch.randn(n, n, dtype=dtype, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(iters):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    mult = 8 if dtype.is_complex else 2
    return mult * n ** 3 / best / 1e12


def main():
    out = {
        "gpu": torch.cuda.get_device_name(0),
        "fp64_gemm_tflops_8192": bench(torch.float64, 8192),
        "c128_gemm_tflops_4096": bench(torch.complex128, 4096),
        "how": "torch.matmul (cuBLAS) best of 10 after 3 warm-ups, CUDA events; "
               "flops = 2n^3 real / 8n^3 complex",
        "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
    }
    print(json.dumps(out))
    path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/fp64_peak.json"
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
