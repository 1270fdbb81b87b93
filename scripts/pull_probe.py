"""Small host<->device transfers on the planning critical path while a SparseAllGather
streams over NVLink on another stream (the early SpAG of the planning gap).

For each transport of a 6 KiB table blob — SM pull from mapped pinned memory
(fssdp_pull_host), copy engine (cudaMemcpyAsync) — and the 256 B counts readback
(fssdp_push_host), time it alone and with a concurrent 4 x 16 MiB SpAG pull per rank.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/pull_probe.py
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2502_02581_b200 import _native as N  # noqa: E402
from paper_2502_02581_b200.comm import HeapLayout, PeerGroup  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    S, n_copies = 16 << 20, 4
    layout = HeapLayout()
    layout.add("params", (n_copies + 1) * S)
    group = PeerGroup(layout, rank, world, dev, "dist")
    poff = layout.offset("params")
    pb = C.c_void_p(group.peer_bases.data_ptr())
    # replicas pulled from the other ranks in turn (a ring when world > 2)
    copies = torch.tensor([[(rank + 1 + i % (world - 1)) % world, 0, 1 + i]
                           for i in range(n_copies)], dtype=torch.int32, device=dev)
    side = torch.cuda.Stream(dev)
    main = torch.cuda.current_stream(dev)
    blob_h = torch.zeros(6144, dtype=torch.uint8).pin_memory()
    blob_d = torch.empty(6144, dtype=torch.uint8, device=dev)
    cnt_d = torch.zeros(64, dtype=torch.int32, device=dev)
    cnt_h = torch.zeros(64 + 4, dtype=torch.int32).pin_memory()
    flag = C.c_void_p(cnt_h.data_ptr() + 256)
    epoch = [0]

    def spag():
        with torch.cuda.stream(side):
            N.call("fssdp_gather_slots", pb, rank, poff, poff, S, 0, C.c_void_p(copies.data_ptr()),
                   n_copies, 0, C.c_void_p(side.cuda_stream))

    transports = {
        "pull_host_6k": lambda: N.call("fssdp_pull_host", C.c_void_p(blob_d.data_ptr()),
                                       C.c_void_p(blob_h.data_ptr()), 6144,
                                       C.c_void_p(main.cuda_stream)),
        "memcpy_h2d_6k": lambda: blob_d.copy_(blob_h, non_blocking=True),
        "push_host_256": lambda: N.call("fssdp_push_host", C.c_void_p(cnt_d.data_ptr()),
                                        C.c_void_p(cnt_h.data_ptr()), 256, flag,
                                        epoch[0], C.c_void_p(main.cuda_stream)),
    }
    out = {}
    for name, fn in transports.items():
        for busy in (0, 20000, 100000):
            times = []
            for it in range(25):
                epoch[0] += 1
                dist.barrier()
                torch.cuda.synchronize()
                if busy:
                    spag()
                    torch.cuda._sleep(busy)  # let the SpAG run first (cycles: ~10 / 50 us)
                s, e = torch.cuda.Event(True), torch.cuda.Event(True)
                s.record()
                fn()
                e.record()
                torch.cuda.synchronize()
                if it >= 5:
                    times.append(1e3 * s.elapsed_time(e))
            out[f"{name}{f'_spag+{busy // 2000}us' if busy else ''}"] = round(float(np.median(times)), 1)
    rows = [None] * world
    dist.all_gather_object(rows, out)
    if rank == 0:
        for r, row in enumerate(rows):
            print("PULLPROBE " + json.dumps({"rank": r, **row}), flush=True)
    dist.barrier()
    group.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
