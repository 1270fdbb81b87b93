"""Host<->device copy bandwidth with every rank copying at once (the e2e leg of bench.py
at N > 1): what bounds e2e when N GPUs share the host's memory and PCIe.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/pcie_multi.py
"""
import json
import os
import time

import torch
import torch.distributed as dist


def measure(dev, n=64 << 20, reps=10):
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n // 2, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device=dev)
    d_out = torch.empty(n // 2, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def once():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)

    res = {}
    for name, fn, nbytes in (
            ("h2d", lambda: d_in.copy_(h_in, non_blocking=True), n),
            ("duplex_64in_32out", once, n + n // 2)):
        fn()
        torch.cuda.synchronize(dev)
        dist.barrier()
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize(dev)
        res[name] = round(nbytes * reps / (time.perf_counter() - t) / 1e9, 1)
        dist.barrier()
    return res


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo")
    out = {"rank": rank, "world": world, "cpus": len(os.sched_getaffinity(0))}
    out.update(measure(dev))
    rows = [None] * world
    dist.all_gather_object(rows, out)
    if rank == 0:
        for r in rows:
            print("PCIEMULTI " + json.dumps(r), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
