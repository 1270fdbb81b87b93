"""SparseAllGather / SparseReduceScatter kernels on their own (K3, K8), N logical ranks
emulated on one GPU (separate symmetric heaps, real cross-heap addressing).

SpAG: every replica slot becomes a bit-exact copy of its owner's shard.  SpRS (push's
owner-local reduce and the pull kernel): each owned slot becomes the fp32 sum, in listed
(ascending-rank) order, of the holders' partials — checked BIT-EXACTLY against a float32
sequential sum (bf16 gradients: of the partials widened to fp32, rounded once at the end).  Schedules come from the product tables (build_rank_tables) of
ring and hot-expert placements (sparse sweep shapes) and random ones; slot sizes include
ragged ones (not a multiple of the kernels' 8 KB sub-chunks).
"""

import ctypes as C

import numpy as np
import pytest
import torch

import paper_2502_02581_b200 as F
from paper_2502_02581_b200 import _native as N
from paper_2502_02581_b200.comm import HeapLayout, emulated_group
from paper_2502_02581_b200.plan_tables import NativeTables

pytestmark = pytest.mark.gpu


def placements(world, E, kind, seed=0):
    topo = F.ClusterTopology.for_nvswitch(world)
    base = F.make_even_partition(E, topo)
    if kind == "ring":
        extra = [(e, (base.owner(e) + i) % world) for e in range(E) for i in range(1, world)]
    elif kind == "hot":
        extra = [(0, d) for d in range(world)]
    else:
        rng = np.random.default_rng(seed)
        extra = [(e, d) for e in range(E) for d in range(world) if rng.random() < 0.4]
    return base, base.union(extra)


def setup(world, E, slot_elems, kind, seed=0):
    base, post = placements(world, E, kind, seed)
    owner = np.asarray(base.owners(), dtype=np.int32)
    route = np.zeros((world, E, world), dtype=np.int64)
    tabs = [NativeTables(r, owner, post.mask, route, 256, 256) for r in range(world)]
    slots = max(t.n_slots for t in tabs)
    n_stage = max(1, max(t.n_stage for t in tabs))
    layout = HeapLayout()
    layout.add("params", slots * slot_elems * 2)
    layout.add("grads", slots * slot_elems * 4)  # fp32-sized: either gradient dtype fits
    layout.add("stage", n_stage * slot_elems * 4)
    groups = emulated_group(layout, world)
    return base, post, tabs, layout, groups, slots, n_stage


@pytest.mark.parametrize("world,E,kind,slot_elems", [
    (2, 2, "ring", 1 << 20), (4, 4, "ring", 3 * 4096 + 1000), (4, 8, "hot", 1 << 18),
    (8, 8, "ring", 12344 * 4), (8, 16, "random", 77776 * 4)])
def test_spag_copies_owner_shards(world, E, kind, slot_elems):
    base, post, tabs, layout, groups, slots, _ = setup(world, E, slot_elems, kind)
    poff = layout.offset("params")
    g = torch.Generator(device="cuda").manual_seed(1)
    params = [grp.local.tensor(poff, (slots, slot_elems), torch.bfloat16) for grp in groups]
    for p in params:
        p.copy_(torch.randn(slots, slot_elems, generator=g, device="cuda"))
    for r, t in enumerate(tabs):
        blob = torch.from_numpy(t.blob[:t.nbytes].copy()).cuda()
        if t.n_spag:
            N.call("fssdp_spag", C.c_void_p(groups[r].peer_bases.data_ptr()), r, poff,
                   slot_elems * 2, C.c_void_p(blob.data_ptr() + t.offsets["spag"]), t.n_spag,
                   C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    for r, t in enumerate(tabs):
        for e, s in t.slots.items():
            o = base.owner(e)
            assert torch.equal(params[r][s], params[o][tabs[o].slots[e]]), (r, e)


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("pull", [False, True])
@pytest.mark.parametrize("world,E,kind,slot_elems", [
    (2, 2, "ring", 1 << 20), (4, 4, "ring", 3 * 2048 + 504), (4, 8, "hot", 1 << 18),
    (8, 8, "ring", 12345 * 8), (8, 16, "random", 77777 * 8)])
def test_sprs_sums_partials_in_rank_order(world, E, kind, slot_elems, pull, dt):
    """Partials sit where the transport expects them — push: the owner's staging slots;
    pull: the holders' own grads slots — and the owner's grads slot ends up holding the
    ascending-rank fp32 sum (bit-exact; bf16 slots: rounded once)."""
    base, post, tabs, layout, groups, slots, n_stage = setup(world, E, slot_elems, kind, seed=3)
    goff, soff = layout.offset("grads"), layout.offset("stage")
    g = torch.Generator(device="cuda").manual_seed(2)
    grads = [grp.local.tensor(goff, (slots, slot_elems), dt) for grp in groups]
    stage = [grp.local.tensor(soff, (n_stage, slot_elems), dt) for grp in groups]
    eb = 4 if dt == torch.float32 else 2
    partial = {}  # (expert, holder) -> its partial
    for r, t in enumerate(tabs):
        grads[r].copy_(torch.randn(slots, slot_elems, generator=g, device="cuda"))
        for e, s in t.slots.items():
            partial[(e, r)] = grads[r][s].clone()
    # push: place the replicas' partials where the wgrad epilogue stores them (c_dest, the
    # owner's staging slots); pull: they stay in the holders' own grads slots
    if not pull:
        for r, t in enumerate(tabs):
            for dst_slot, b, n in t.sprs_jobs:
                for h, idx in t.sprs_srcs[b:b + n]:
                    if h != r:
                        e = [x for x, s in t.slots.items() if s == dst_slot][0]
                        stage[r][idx].copy_(partial[(e, int(h))])
    torch.cuda.synchronize()
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    blobs = [torch.from_numpy(t.blob[:t.nbytes].copy()).cuda() for t in tabs]
    for r, t in enumerate(tabs):
        pb, jobs = C.c_void_p(groups[r].peer_bases.data_ptr()), t.offsets["sprs_jobs"]
        if pull:
            N.call("fssdp_sprs_pull", pb, r, goff, slot_elems, eb,
                   C.c_void_p(blobs[r].data_ptr() + jobs), t.n_sprs_jobs,
                   C.c_void_p(blobs[r].data_ptr() + t.offsets["sprs_pull"]), stream)
        else:
            N.call("fssdp_sprs", pb, r, goff, soff, slot_elems, eb,
                   C.c_void_p(blobs[r].data_ptr() + jobs), t.n_sprs_jobs,
                   C.c_void_p(blobs[r].data_ptr() + t.offsets["sprs_srcs"]), stream)
    torch.cuda.synchronize()
    reduced = 0
    for r, t in enumerate(tabs):
        for e, s in t.slots.items():
            if base.owner(e) != r:
                continue
            holders = [d for d in range(world) if post.mask[e, d]]
            want = torch.zeros(slot_elems, dtype=torch.float32)
            for h in holders:
                want = want + partial[(e, h)].cpu().float()   # float32, ascending rank
            got = grads[r][s].cpu()
            if len(holders) > 1:
                reduced += 1
                assert torch.equal(got, want.to(dt)), (r, e)
            else:
                assert torch.equal(got, partial[(e, r)].cpu())
    assert reduced > 0
