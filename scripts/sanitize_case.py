"""A small FSSDP workload for compute-sanitizer (memcheck / racecheck / synccheck), one tool
per run:  compute-sanitizer --tool <t> python scripts/sanitize_case.py

Covers every P2P kernel of the layer with 4 emulated ranks on one GPU (separate heaps,
real cross-heap peer addressing; device barriers disabled by the emulation): gate+count
all-gather, early and late SpAG (gather_slots / spag), dispatch, combine, dispatch_grad,
combine_dx, the push-SpRS (wgrad epilogue stores into peers' staging) + owner reduce, and
the standalone sparse_all_gather / sparse_reduce_scatter pull kernels; plus one N=1 step."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2502_02581_b200 as F  # noqa: E402
from paper_2502_02581_b200.comm import HeapLayout, emulated_group  # noqa: E402
from paper_2502_02581_b200.layer import (FssdpMoE, LayerGeometry, default_slots,  # noqa: E402
                                         run_lockstep_backward, run_lockstep_forward)


def layers(world, E, d, f, T, pol, act="gelu"):
    m = pol.capacity_override if pol.capacity_override is not None else E
    geom = LayerGeometry(d, f, E, 2, T, world, default_slots(E, world, m), act)
    layout = HeapLayout()
    geom.add_regions(layout, "L0.")
    groups = emulated_group(layout, world)
    topo = F.ClusterTopology.for_nvswitch(world)
    cfg = F.ModelConfig(1, E, geom.expert_bytes, 2 * d, 1e-3, 1e-6)
    p = 1.0 / np.arange(1, E + 1) ** 1.3
    bias = torch.tensor(np.log(p / p.sum()), dtype=torch.float32, device="cuda")
    out = []
    for r in range(world):
        ly = FssdpMoE(geom, groups[r], F.FssdpPlanner(cfg, topo, pol), 0, 3)
        ly.gate_bias.copy_(bias)
        out.append(ly)
    return out


def main():
    D, E, d, f, Tr = 4, 8, 256, 512, 256
    pol = F.Policy(F.PolicyKind.FSSDP, overlap_override=8, capacity_override=2,
                   rematerialize=True)
    multi = layers(D, E, d, f, Tr, pol)
    g = torch.Generator(device="cuda").manual_seed(1)
    for it in range(3):
        x = torch.randn(D * Tr, d, device="cuda", generator=g).bfloat16()
        dy = (torch.randn(D * Tr, d, device="cuda", generator=g) * 0.05).bfloat16()
        run_lockstep_forward(multi, list(x.split(Tr)))
        run_lockstep_backward(multi, list(dy.split(Tr)), rematerialize=True)
        for ly in multi:
            ly.planner.finish()
    torch.cuda.synchronize()
    reps = len(multi[0].decision.target.entries) - E
    # standalone sparse collectives
    topo = F.ClusterTopology.for_nvswitch(D)
    base = F.make_even_partition(D, topo)
    post = base.union([(e, (e + 1) % D) for e in range(D)])
    layout = HeapLayout()
    S = 1 << 16
    off = layout.add("chunks", 2 * S)
    bufs = [F.ChunkBuffer(gr, off, S, 2) for gr in emulated_group(layout, D)]
    for b in bufs:
        F.sparse_all_gather(base, post, b)
    for b in bufs:
        F.sparse_reduce_scatter(post, base, b)
    # one rank, SwiGLU, 128-wide N tiles
    (one,) = layers(1, E, d, 384, 512, pol, "swiglu")
    x = torch.randn(512, d, device="cuda", generator=g).bfloat16()
    one.forward(x)
    one.backward((x * 0.05).contiguous())
    torch.cuda.synchronize()
    print(f"SANITIZE CASE OK (replicas {reps})", flush=True)


if __name__ == "__main__":
    main()
