"""SparseAllGather / SparseReduceScatter bandwidth sweep (BASELINE.json config 5).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/sparse_sweep.py [--quick]

E = N experts, even single-owner partition; the post-placement adds expert e to devices
(e+1 .. e+r-1) mod N (balanced ring: every GPU pulls (r-1)·S in SpAG and its owner pulls
(r-1)·S_grad in SpRS).  A "hot" variant materializes expert 0 on r devices only.  Times are
CUDA events around the kernel, max over ranks; GB/s = per-GPU inbound bytes / time
(SpAG) and the reference's bottleneck bytes / time (costmodel.py:75-84).  SpRS moves the
layer's gradients (--grad-dtype bf16: S_grad = S, the reference's expert_bytes pricing;
fp32: S_grad = 2·S) the way the layer does: the shared-prefix wgrad launches push each
holder's partial into its owner's staging slot through the epilogue's TMA stores (run
here with K = 0, i.e. the store path alone), then a barrier and the owner's local
reduction.  "sprs_pull" times the pull transport alone: the partials already sit in the
holders' own grads slots and each owner pulls them over NVLink and sums them in one
pass (fssdp_sprs_pull).  Prints one JSON line per case on rank 0.
"""

import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2502_02581_b200 as F  # noqa: E402
from paper_2502_02581_b200 import _native as N  # noqa: E402
from paper_2502_02581_b200 import ops  # noqa: E402
from paper_2502_02581_b200.comm import HeapLayout, PeerGroup  # noqa: E402
from paper_2502_02581_b200.plan_tables import NativeTables  # noqa: E402


_PEAK_FILE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                          "profiles", "r2_nvlink_peak_n4.json")
NVLINK_PEAK = (json.load(open(_PEAK_FILE))["nvlink_gbs"] if os.path.exists(_PEAK_FILE)
               else 770.0)  # measured inbound peer peak (scripts/nvlink_probe.py)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--grad-dtype", default="bf16", choices=["bf16", "fp32"])
    args = ap.parse_args()
    gbytes = 2 if args.grad_dtype == "bf16" else 4
    gdt = torch.bfloat16 if gbytes == 2 else torch.float32
    epi = ops.EPI_BF16 if gbytes == 2 else ops.EPI_F32
    wire = gbytes / 2  # gradient bytes per parameter byte
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    sizes_mb = [1, 4, 16, 64, 256] if args.quick else [1, 2, 4, 8, 16, 32, 64, 128, 256]
    smax = max(sizes_mb) << 20
    slots = world  # owned slot + up to world-1 replicas
    layout = HeapLayout()
    layout.add("params", slots * smax)
    layout.add("grads", slots * 2 * smax)
    layout.add("stage", (world - 1) * 2 * smax)
    group = PeerGroup(layout, rank, world, dev, "dist")
    poff, goff = layout.offset("params"), layout.offset("grads")
    soff = layout.offset("stage")
    dummy = torch.zeros(64, 1 << 18, dtype=torch.bfloat16, device=dev)  # never read (K = 0)
    bar_epoch = [0]
    heap = group.local
    heap.tensor(poff, (slots * smax // 2,), torch.bfloat16).normal_()
    heap.tensor(goff, (slots * smax // 2,), gdt).normal_()
    topo = F.ClusterTopology.for_nvswitch(world)
    stream = torch.cuda.current_stream(dev)
    sp = C.c_void_p(stream.cuda_stream)
    flags_off = layout.offset("flags")
    grads = heap.tensor(goff, (slots * smax // 2,), gdt)

    def push(tab, blob, maps, d_, f_):
        """The shared-prefix wgrad launches with K = 0: replica partials (zeros) stored
        into the owners' staging slots, owned shared slots locally."""
        n_sh, t1, t2 = tab.wgrad_split
        for name, ldc, tiles, a_w, b_w in (("wgrad1", d_, t1, f_, d_), ("wgrad2", f_, t2, d_, f_)):
            if tiles == 0:
                continue
            a = dummy[:, :a_w]
            b = dummy[:, :b_w]
            N.call("fssdp_grouped_gemm", 1, 1, epi, ops._ptr(a), a_w, 64, ops._ptr(b),
                   b_w, 64, C.c_void_p(blob.data_ptr() + tab.offsets[name]), n_sh,
                   tab.gemm[name][1], tiles, ops._ptr(grads), None, None, ops._ptr(maps[name]),
                   ldc, grads.numel() // ldc, 2, None, sp)
    pb = C.c_void_p(group.peer_bases.data_ptr())
    E = world
    base = F.make_even_partition(E, topo)
    for variant in ("ring", "hot"):
        for r in range(2, world + 1):
            if variant == "ring":
                extra = [(e, (e + i) % world) for e in range(E) for i in range(1, r)]
            else:
                extra = [(0, i) for i in range(1, r)]
            post = base.union(extra)
            owner = base.owners()
            route = np.zeros((world, E, world), dtype=np.int64)
            for mb in sizes_mb:
                S = mb << 20
                d_, f_ = 256, mb * 1024   # one slot = [W1 | W2] = 4 d f bytes = S
                tab = NativeTables(rank, owner, post.mask, route, d_, f_)
                blob = torch.from_numpy(tab.blob[:tab.nbytes].copy()).to(dev)
                maps = {}
                for name, ldc in (("wgrad1", d_), ("wgrad2", f_)):
                    raw = b"".join(ops.epilogue_tmap(epi, b + soff, ldc,
                                                     (world - 1) * 2 * d_ * f_ // ldc)
                                   for b in group.bases)
                    maps[name] = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(dev)
                spag_t = C.c_void_p(blob.data_ptr() + tab.offsets["spag"])
                jobs_t = C.c_void_p(blob.data_ptr() + tab.offsets["sprs_jobs"])
                srcs_t = C.c_void_p(blob.data_ptr() + tab.offsets["sprs_srcs"])
                pull_t = C.c_void_p(blob.data_ptr() + tab.offsets["sprs_pull"])
                res = {}
                for kind in ("spag", "sprs", "sprs_pull"):
                    times = []
                    for it in range(args.iters + 2):
                        dist.barrier()
                        torch.cuda.synchronize()
                        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
                        s.record()
                        if kind == "spag" and tab.n_spag:
                            N.call("fssdp_spag", pb, rank, poff, S, spag_t, tab.n_spag, sp)
                        if kind == "sprs":
                            push(tab, blob, maps, d_, f_)
                            bar_epoch[0] += 1
                            N.call("fssdp_barrier", pb, flags_off, rank, world, 0,
                                   C.c_uint32(bar_epoch[0]), sp)
                            if tab.n_sprs_jobs:
                                N.call("fssdp_sprs", pb, rank, goff, soff, S // 2, gbytes,
                                       jobs_t,
                                       tab.n_sprs_jobs, srcs_t, sp)
                        if kind == "sprs_pull" and tab.n_sprs_jobs:
                            # partials already in the holders' own grads slots (a wgrad
                            # without c_dest writes them there): the owners' pull + sum alone
                            N.call("fssdp_sprs_pull", pb, rank, goff, S // 2, gbytes, jobs_t,
                                   tab.n_sprs_jobs, pull_t, sp)
                        e.record()
                        torch.cuda.synchronize()
                        if it >= 2:
                            times.append(s.elapsed_time(e))
                    t = torch.tensor([float(np.median(times))], device=dev, dtype=torch.float64)
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                    res[kind] = float(t.item())
                tr, rep = F.spag_traffic(base, post, S)
                inbound_spag = float(tr.data[:, rank].sum())
                g = torch.tensor([inbound_spag], device=dev, dtype=torch.float64)
                dist.all_reduce(g, op=dist.ReduceOp.MAX)
                max_in = float(g.item())
                if rank == 0:
                    line = {
                        "n_gpus": world, "variant": variant, "replicas": r, "expert_mib": mb,
                        "spag_ms": res["spag"], "sprs_ms": res["sprs"],
                        "spag_bottleneck_bytes": rep.bottleneck_bytes,
                        "spag_gbs_bottleneck": rep.bottleneck_bytes / (res["spag"] * 1e-3) / 1e9,
                        "spag_gbs_inbound_max": max_in / (res["spag"] * 1e-3) / 1e9,
                        "grad_dtype": args.grad_dtype,
                        "sprs_gbs_bottleneck": wire * rep.bottleneck_bytes / (res["sprs"] * 1e-3) / 1e9,
                        "sprs_path": "wgrad epilogue TMA-store push (K=0) + barrier + local reduce",
                        "sprs_pull_ms": res["sprs_pull"],
                        "sprs_pull_gbs_bottleneck":
                            wire * rep.bottleneck_bytes / (res["sprs_pull"] * 1e-3) / 1e9,
                        "sprs_pull_gbs_inbound_max": wire * max_in / (res["sprs_pull"] * 1e-3) / 1e9,
                        "nvlink_peak_gbs": NVLINK_PEAK,
                        "spag_frac_of_peak": rep.bottleneck_bytes / (res["spag"] * 1e-3) / 1e9
                                             / NVLINK_PEAK,
                        # the reference's bottleneck bytes (costmodel.py:75-84; sprs_traffic is
                        # spag_traffic transposed) x gradient bytes per parameter byte
                        "sprs_pull_frac_of_peak": wire * rep.bottleneck_bytes
                                                  / (res["sprs_pull"] * 1e-3) / 1e9 / NVLINK_PEAK,
                    }
                    print("SWEEP " + json.dumps(line), flush=True)
    dist.barrier()
    group.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
