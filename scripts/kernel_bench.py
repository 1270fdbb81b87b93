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


_FLUSH = None


def flush_l2():
    """Evict the 126 MB L2 (inputs then come from HBM, as inside a step)."""
    global _FLUSH
    if _FLUSH is None:
        _FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    _FLUSH.fill_(1)


def timeit(fn, reps=30, cold=True):
    """Median µs of one entry point's kernels (native launch-timing window: no host time);
    cold: L2 flushed before every timed call."""
    for _ in range(5):
        fn()
    ts = []
    for _ in range(reps):
        if cold:
            flush_l2()
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
    # the layer's fused gate (K1 + K2 tail, N = 1: local dispatch + GEMM tables, counts push)
    from paper_2502_02581_b200.comm import HeapLayout, emulated_group
    from paper_2502_02581_b200.plan_tables import _layout
    layout = HeapLayout()
    layout.add("counts", 64 * 4)
    (grp,) = emulated_group(layout, 1)
    tiles = (T + 63) // 64
    tidx = torch.empty(T, k, dtype=torch.int32, device=dev)
    tw = torch.empty(T, k, dtype=torch.float32, device=dev)
    trk = torch.empty(T, k, dtype=torch.int32, device=dev)
    ttc = torch.empty(tiles, E, dtype=torch.int32, device=dev)
    tpf = torch.empty(tiles, E, dtype=torch.int32, device=dev)
    gws = torch.zeros(1 + E, dtype=torch.int32, device=dev)
    blob = torch.zeros(_layout(E, 1)[1], dtype=torch.uint8, device=dev)
    host = torch.zeros(32, dtype=torch.int32, pin_memory=True)
    gws = torch.empty(int(N.LIB.fssdp_gate_gemm_ws_bytes(T, d)), dtype=torch.uint8, device=dev)
    tc_gate = [False]
    ep = [0]

    def route():
        ep[0] += 1
        N.call("fssdp_gate_route", ops._ptr(x), ops._ptr(wg), ops._ptr(bias), T, d, E, k,
               ops._ptr(tidx), ops._ptr(tw), ops._ptr(trk), ops._ptr(ttc), ops._ptr(tpf),
               ops._ptr(gws), C.c_void_p(grp.peer_bases.data_ptr()), layout.offset("counts"),
               layout.offset("flags"), 0, 1, -1, 0, ops._ptr(blob), 4096, 2, 0,
               C.c_void_p(host.data_ptr()), 64, C.c_void_p(host.data_ptr() + 64),
               C.c_uint32(ep[0]), ops._ptr(gws) if tc_gate[0] else None,
               gws.numel() if tc_gate[0] else 0, stream)
    res["gate_route_cold_us"] = timeit(route)
    res["gate_route_warm_us"] = timeit(route, cold=False)
    tc_gate[0] = True  # the tensor-core gate path
    res["gate_route_tc_cold_us"] = timeit(route)
    res["gate_route_tc_warm_us"] = timeit(route, cold=False)
    res["gate_topk_warm_us"] = timeit(lambda: ops.gate_topk(x, wg, k, bias=bias), cold=False)
    res["gate_wgrad_us"] = timeit(lambda: N.call(
        "fssdp_gate_wgrad", ops._ptr(x), ops._ptr(idx), ops._ptr(dlogit), T, d, E, k,
        ops._ptr(ws), ops._ptr(dwg), stream))
    xb = T * d * 2
    res["gate_topk_gbs"] = xb / (res["gate_topk_us"] * 1e-6) / 1e9
    res["gate_route_cold_gbs"] = xb / (res["gate_route_cold_us"] * 1e-6) / 1e9
    res["gate_wgrad_gbs"] = xb / (res["gate_wgrad_us"] * 1e-6) / 1e9
    print("KBENCH " + json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
