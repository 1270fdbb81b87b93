"""Standalone timings of the HBM-bound token-side kernels at cfg2 sizes (one GPU).

    python scripts/kernel_bench.py

Prints one JSON line: median microseconds per kernel and the achieved GB/s of the
algorithmic bytes (the kernel's roofline is HBM)."""

import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2502_02581_b200 import _native as N  # noqa: E402
from paper_2502_02581_b200 import ops  # noqa: E402


def timeit(fn, reps=30):
    """Median µs of one entry point's kernels (native launch-timing window: no host time)."""
    for _ in range(5):
        fn()
    ts = []
    for _ in range(reps):
        timers = {}
        N.timed_launch(timers, "k", fn)
        torch.cuda.synchronize()
        s, e = timers["k"][0]
        ts.append(s.elapsed_time(e) * 1e3)
    return float(np.median(ts))


def main():
    dev = torch.device("cuda", 0)
    T, d, E, k = 16384, 1024, 16, 2
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(T, d, device=dev, generator=g).bfloat16()
    wg = torch.randn(E, d, device=dev, generator=g) / d ** 0.5
    bias = torch.zeros(E, device=dev)
    idx, w, rank, tc, _ = ops.gate_topk(x, wg, k, bias=bias)
    dlogit = torch.randn(T, k, device=dev, generator=g)
    ws = torch.empty(((T + 63) // 64) * E * d, device=dev)
    dwg = torch.empty(E, d, device=dev)
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    res = {}
    res["gate_topk_us"] = timeit(lambda: ops.gate_topk(x, wg, k, bias=bias))
    res["gate_wgrad_us"] = timeit(lambda: N.call(
        "fssdp_gate_wgrad", ops._ptr(x), ops._ptr(idx), ops._ptr(dlogit), T, d, E, k,
        ops._ptr(ws), ops._ptr(dwg), stream))
    xb = T * d * 2
    res["gate_topk_gbs"] = xb / (res["gate_topk_us"] * 1e-6) / 1e9
    res["gate_wgrad_gbs"] = xb / (res["gate_wgrad_us"] * 1e-6) / 1e9
    print("KBENCH " + json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
