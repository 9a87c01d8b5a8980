"""Measure the B200's fp64 GEMM peak (cuBLAS DGEMM through torch.matmul float64).

Burst = best of 10 single 8192^3 products (CUDA events); sustained = back-to-back products for
~4 s.  2*N^3 flops per product.  Writes one JSON line (and profiles/fp64_peak.json when asked).
This is the denominator the FD contraction's roofline fraction is stated against.
"""

import json
import os
import sys
import time

import torch


def main(out=None):
    n = 8192
    dev = torch.device("cuda:0")
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    c = torch.empty(n, n, dtype=torch.float64, device=dev)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    flops = 2.0 * n ** 3
    burst = flops / best / 1e12
    # sustained
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_end = time.time() + 4.0
    reps = 0
    e0.record()
    while time.time() < t_end:
        for _ in range(4):
            torch.matmul(a, b, out=c)
        reps += 4
        torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    sustained = reps * flops / (e0.elapsed_time(e1) / 1e3) / 1e12
    # small-batched shape typical of the FD contraction (65x65 / 129x129 / 258x258 operands)
    small = {}
    for m, batch in ((65, 4096), (129, 1024), (258, 256)):
        x = torch.randn(batch, m, m, dtype=torch.float64, device=dev)
        y = torch.randn(batch, m, m, dtype=torch.float64, device=dev)
        for _ in range(3):
            torch.bmm(x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            torch.bmm(x, y)
        e1.record()
        e1.synchronize()
        small[f"bmm_{m}x{m}x{m}_b{batch}"] = 10 * 2.0 * batch * m ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12
    res = {"fp64_tflops": burst, "fp64_tflops_sustained": sustained, "how":
           "torch.matmul float64 8192^3 (2 N^3 flops, cuBLAS DGEMM): best of 10 (burst), back to back ~4 s "
           "(sustained); CUDA events", "batched_small_tflops": small,
           "gpu": torch.cuda.get_device_name(0)}
    line = json.dumps(res)
    print(line, flush=True)
    if out:
        with open(out, "w") as fh:
            fh.write(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
