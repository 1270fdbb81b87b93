"""NVLink peer-bandwidth probe on one box (one process driving every visible GPU).

    python scripts/nvlink_probe.py [--mib 256] [--iters 10] [--out profiles/r2_nvlink_peak.json]

Measures, per direction, on GPU 0 (CUDA events on the launching stream, best and median of
`iters` after warm-up):

* ce_pull_1: the copy engines pulling S bytes from one peer (cudaMemcpyAsync, peer access on);
* ce_pull_all: GPU 0 pulling S from every peer at once (one stream per peer) — inbound bound;
* sm_pull_1 / sm_pull_all: libfssdp's TMA-bulk pull kernel (fssdp_gather_slots, the SpAG
  transport) from one peer / from every peer in one launch;
* sm_push_1: the same kernel writing into a peer (local reads, remote stores — the direction
  of the dispatch / SpRS-push transports);
* sprs_pull_all: fssdp_sprs_pull summing one fp32 partial from every peer into GPU 0's slot;
* a2a_ce: every GPU pulling S from every other GPU at once (per-GPU inbound under full
  all-to-all load), timed on each GPU, max over GPUs.

GB/s = bytes crossing into (or out of) GPU 0 ÷ time.  The JSON is what bench.py uses as
the NVLink roofline denominator (`nvlink_gbs` = best of sm_pull_all / ce_pull_all).  Run
the same command under `ncu --metrics nvlrx__bytes.sum,nvltx__bytes.sum,...` for the
per-kernel link counters (the copy-engine rows are not kernels).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2502_02581_b200 import _native as N  # noqa: E402


def cudart():
    for p in (Path(torch.__file__).parent / "lib", Path("/usr/local/cuda/lib64")):
        for cand in sorted(p.glob("libcudart.so*")):
            try:
                return C.CDLL(str(cand))
            except OSError:
                continue
    nv = Path(torch.__file__).parent.parent / "nvidia" / "cuda_runtime" / "lib"
    for cand in sorted(nv.glob("libcudart.so*")):
        return C.CDLL(str(cand))
    raise RuntimeError("libcudart not found")


def enable_peers(n):
    rt = cudart()
    for a in range(n):
        torch.cuda.set_device(a)
        for b in range(n):
            if a != b:
                rc = rt.cudaDeviceEnablePeerAccess(b, 0)
                if rc not in (0, 704):  # 704: already enabled
                    raise RuntimeError(f"cudaDeviceEnablePeerAccess({a}->{b}) = {rc}")
    torch.cuda.set_device(0)


def timed(fn, iters, dev=0):
    torch.cuda.set_device(dev)
    times = []
    for i in range(iters + 3):
        for d in range(torch.cuda.device_count()):
            torch.cuda.synchronize(d)
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        fn()
        e.record()
        for d in range(torch.cuda.device_count()):
            torch.cuda.synchronize(d)
        if i >= 3:
            times.append(s.elapsed_time(e) * 1e-3)
    return min(times), statistics.median(times)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    n = torch.cuda.device_count()
    if n < 2:
        print(json.dumps({"error": "needs >= 2 GPUs"}))
        return
    enable_peers(n)
    S = args.mib << 20
    bufs = [torch.empty(n * S, dtype=torch.uint8, device=f"cuda:{d}") for d in range(n)]
    for d in range(n):
        bufs[d].fill_(d + 1)
    s0 = torch.cuda.current_stream(0)
    res = {}

    def rec(name, nbytes, t):
        best, med = t
        res[name] = {"bytes": nbytes, "best_s": best, "median_s": med,
                     "gbs_best": nbytes / best / 1e9, "gbs_median": nbytes / med / 1e9}

    # copy engines
    rec("ce_pull_1", S, timed(lambda: bufs[0][:S].copy_(bufs[1][:S], non_blocking=True),
                              args.iters))
    streams = [torch.cuda.Stream(device=0) for _ in range(n)]

    def ce_all():
        main = torch.cuda.current_stream(0)
        for p in range(1, n):
            streams[p].wait_stream(main)
            with torch.cuda.stream(streams[p]):
                bufs[0][p * S:(p + 1) * S].copy_(bufs[p][:S], non_blocking=True)
        for p in range(1, n):
            main.wait_stream(streams[p])
    rec("ce_pull_all", (n - 1) * S, timed(ce_all, args.iters))

    # libfssdp's pull kernel: peer_bases[r] = GPU r's buffer
    pb = torch.tensor(np.array([b.data_ptr() for b in bufs], dtype=np.uint64).view(np.int64),
                      device="cuda:0")
    sp = C.c_void_p(s0.cuda_stream)

    def gather(rank, copies):
        tab = torch.tensor(copies, dtype=torch.int32, device="cuda:0")
        return lambda: N.call("fssdp_gather_slots", C.c_void_p(pb.data_ptr()), rank, 0, 0, S, 0,
                              C.c_void_p(tab.data_ptr()), len(copies), 0, sp), tab
    f1, t1 = gather(0, [(1, 1, 0)])
    rec("sm_pull_1", S, timed(f1, args.iters))
    fa, ta = gather(0, [(p, p, p) for p in range(1, n)])
    rec("sm_pull_all", (n - 1) * S, timed(fa, args.iters))
    fp, tp = gather(1, [(0, 0, 0)])  # launched on GPU 0, destination = GPU 1's buffer
    rec("sm_push_1", S, timed(fp, args.iters))
    # SpRS pull: GPU 0 sums its own fp32 partial and one from every peer
    jobs = torch.tensor([[0, 0, n]], dtype=torch.int32, device="cuda:0")
    srcs = torch.tensor([[r, 0] for r in range(n)], dtype=torch.int32, device="cuda:0")
    for d in range(n):
        bufs[d][:S].view(torch.float32).fill_(1.0)
    rec("sprs_pull_all", (n - 1) * S, timed(
        lambda: N.call("fssdp_sprs_pull", C.c_void_p(pb.data_ptr()), 0, 0, S // 4, 4,
                       C.c_void_p(jobs.data_ptr()), 1, C.c_void_p(srcs.data_ptr()), sp),
        args.iters))

    # full all-to-all on the copy engines: every GPU pulls S from every other GPU
    a2a_streams = {(d, p): torch.cuda.Stream(device=d) for d in range(n) for p in range(n) if p != d}

    def a2a():
        for d in range(n):
            with torch.cuda.device(d):
                main = torch.cuda.current_stream(d)
                for p in range(n):
                    if p == d:
                        continue
                    st = a2a_streams[(d, p)]
                    st.wait_stream(main)
                    with torch.cuda.stream(st):
                        bufs[d][p * S:(p + 1) * S].copy_(bufs[p][:S], non_blocking=True)
                for p in range(n):
                    if p != d:
                        main.wait_stream(a2a_streams[(d, p)])
    # time on GPU 0 with every GPU's streams joined back: events around the whole exchange
    rec("a2a_ce_inbound_per_gpu", (n - 1) * S, timed(a2a, args.iters))

    best = max(res["sm_pull_all"]["gbs_best"], res["ce_pull_all"]["gbs_best"])
    out = {"n_gpus": n, "gpu": torch.cuda.get_device_name(0), "size_mib": args.mib,
           "iters": args.iters, "results": res,
           "nvlink_gbs": best,
           "nvlink_gbs_note": "measured inbound peer bandwidth of one GPU (best of the "
                              "all-peers pulls, SM kernel or copy engines); nominal 900 "
                              "GB/s per direction"}
    line = json.dumps(out)
    print(line, flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
