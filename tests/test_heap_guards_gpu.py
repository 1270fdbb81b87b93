"""Out-of-bounds writes into the symmetric heaps (compute-sanitizer is closed on the GPU
pool, so the heaps carry their own canaries): every heap region is followed by a 64 KiB
guard filled with 0xA5; after multi-rank FSSDP steps (emulated ranks: every P2P writer —
dispatch and dispatch_grad pushes, early/late SpAG, the wgrad epilogue's stores into peers'
staging slots, SpRS, re-shard moves, the standalone sparse collectives) no guard of any
rank's heap may have changed."""

import numpy as np
import pytest
import torch

import paper_2502_02581_b200 as F
from paper_2502_02581_b200.comm import HeapLayout, emulated_group
from paper_2502_02581_b200.layer import (FssdpMoE, layer_geometries, run_lockstep_backward,
                                         run_lockstep_forward)

pytestmark = pytest.mark.gpu

GUARD = 64 << 10


def zipf_bias(E, s, seed):
    p = 1.0 / np.arange(1, E + 1) ** s
    p = p[np.random.default_rng(seed).permutation(E)]
    return torch.tensor(np.log(p / p.sum()), dtype=torch.float32, device="cuda")


@pytest.mark.parametrize("world,L,E,f,act,kw", [
    (4, 1, 8, 512, "gelu", dict(overlap_override=8, capacity_override=2, rematerialize=True)),
    (8, 2, 16, 384, "swiglu", dict(overlap_override=6, capacity_override=2, reshard_interval=2)),
    (2, 1, 16, 1408, "swiglu", dict(overlap_override=8, capacity_override=4)),
])
def test_no_kernel_writes_past_a_heap_region(world, L, E, f, act, kw):
    d, Tr = 256, 384
    pol = F.Policy(F.PolicyKind.FSSDP, **kw)
    nm = 3 if act == "swiglu" else 2
    topo = F.ClusterTopology.for_nvswitch(world)
    cfg = F.ModelConfig(L, E, 2 * nm * d * f, 2 * d, 1e-3, 1e-6)
    planners = [F.FssdpPlanner(cfg, topo, pol) for _ in range(world)]
    geoms = layer_geometries(planners[0], d, f, 2, Tr, kw["capacity_override"], act)
    layout = HeapLayout(guard=GUARD)
    for li, g in enumerate(geoms):
        g.add_regions(layout, f"L{li}.")
    S = 1 << 16
    chunks_off = layout.add("chunks", 2 * S)
    groups = emulated_group(layout, world)
    for g in groups:
        g.local.fill_guards(layout)
    model = [[FssdpMoE(geoms[li], groups[r], planners[r], li, 3, prefix=f"L{li}.")
              for r in range(world)] for li in range(L)]
    for li, row in enumerate(model):
        for ly in row:
            ly.gate_bias.copy_(zipf_bias(E, 1.4, li))
    gen = torch.Generator(device="cuda").manual_seed(2)
    replicas = 0
    for it in range(4):
        h = list(torch.randn(world * Tr, d, device="cuda", generator=gen).bfloat16().split(Tr))
        for row in model:
            h = run_lockstep_forward(row, h)
        gr = list((torch.randn(world * Tr, d, device="cuda", generator=gen) * 0.05)
                  .bfloat16().split(Tr))
        for row in reversed(model):
            gr = run_lockstep_backward(row, gr, rematerialize=pol.rematerialize)
        for r in range(world):
            planners[r].finish()
        replicas += sum(len(row[0].decision.target.entries) - E for row in model)
    base = F.make_even_partition(world, topo)
    post = base.union([(e, (e + 1) % world) for e in range(world)])
    bufs = [F.ChunkBuffer(g, chunks_off, S, 2) for g in groups]
    for b in bufs:
        F.sparse_all_gather(base, post, b)
    for b in bufs:
        F.sparse_reduce_scatter(post, base, b)
    torch.cuda.synchronize()
    assert replicas > 0
    for r, g in enumerate(groups):
        bad = g.local.check_guards(layout)
        assert not bad, f"rank {r}: writes past the end of {bad}"


def test_guard_check_is_live():
    """Negative control: a copy-engine write one byte past a region is reported."""
    import ctypes as C
    from paper_2502_02581_b200 import _native as N

    layout = HeapLayout(guard=GUARD)
    off = layout.add("x", 4096)
    (g,) = emulated_group(layout, 1)
    g.local.fill_guards(layout)
    src = torch.zeros(8, dtype=torch.uint8, device="cuda")
    N.call("fssdp_copy_async", C.c_void_p(g.local.ptr + off + 4096), C.c_void_p(src.data_ptr()),
           1, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert g.local.check_guards(layout) == ["x"]
