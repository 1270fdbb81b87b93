"""Host<->device copy bandwidth probe (pinned memory), one GPU: single stream, two
streams, H2D+D2H concurrently — what the e2e leg of bench.py is bound by."""
import json
import time

import torch


def bw(fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t) / 1e9


def main():
    n = 32 << 20
    h = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(3)]
    d = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(3)]
    s = [torch.cuda.Stream() for _ in range(3)]
    res = {}
    res["h2d_1x32MiB"] = bw(lambda: d[0].copy_(h[0], non_blocking=True), n)
    res["d2h_1x32MiB"] = bw(lambda: h[0].copy_(d[0], non_blocking=True), n)

    def two_h2d():
        for i in range(2):
            with torch.cuda.stream(s[i]):
                d[i].copy_(h[i], non_blocking=True)
    res["h2d_2streams"] = bw(two_h2d, 2 * n)

    def duplex():
        with torch.cuda.stream(s[0]):
            d[0].copy_(h[0], non_blocking=True)
        with torch.cuda.stream(s[1]):
            h[1].copy_(d[1], non_blocking=True)
    res["h2d+d2h_concurrent"] = bw(duplex, 2 * n)
    s4 = [torch.cuda.Stream() for _ in range(8)]
    h4 = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(4)]
    d4 = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(4)]
    for ways in (2, 4):  # each direction's 64 MiB as `ways` chunks on `ways` streams
        def duplex_ways():
            c = n // (ways // 2)
            for i in range(ways):
                o = (i // 2) * c
                with torch.cuda.stream(s4[i]):
                    d4[i % 2][o:o + c].copy_(h4[i % 2][o:o + c], non_blocking=True)
                with torch.cuda.stream(s4[4 + i]):
                    h4[2 + i % 2][o:o + c].copy_(d4[2 + i % 2][o:o + c], non_blocking=True)
        res[f"duplex_64MiB_each_way_{ways}streams"] = bw(duplex_ways, 4 * n)
    def duplex64():
        with torch.cuda.stream(s[0]):
            d4[0].copy_(h4[0], non_blocking=True)
            d4[1].copy_(h4[1], non_blocking=True)
        with torch.cuda.stream(s[1]):
            h4[2].copy_(d4[2], non_blocking=True)
            h4[3].copy_(d4[3], non_blocking=True)
    res["duplex_64MiB_each_way_1stream"] = bw(duplex64, 4 * n)
    # the same duplex while the SMs run bf16 GEMMs on another stream (as inside a step)
    a = torch.randn(8192, 8192, device="cuda").bfloat16()
    gs = torch.cuda.Stream()

    def duplex_under_load():
        with torch.cuda.stream(gs):
            for _ in range(3):
                a @ a
        duplex64()
    res["duplex_64MiB_each_way_under_gemm"] = bw(duplex_under_load, 4 * n)
    big = 256 << 20
    hb = torch.empty(big, dtype=torch.uint8).pin_memory()
    db = torch.empty(big, dtype=torch.uint8, device="cuda")
    res["h2d_1x256MiB"] = bw(lambda: db.copy_(hb, non_blocking=True), big, 4)
    print("PCIE " + json.dumps({k: round(v, 1) for k, v in res.items()}))


if __name__ == "__main__":
    main()
