"""sparse_all_gather / sparse_reduce_scatter (the north_star's Python entry points) on the
GPU: N logical ranks' symmetric heaps on one device (PeerGroup "emulated"; the pull kernels
address every heap through the peer table exactly as over NVSwitch).  SpAG replicas are
bit-exact owner copies; SpRS owner slots are bit-exact fp32 sums in ascending device order
(PAPER.md:370-386).  Placements: balanced ring, hot expert, and the valid cases of the
reference-generated traffic corpus."""

import numpy as np
import pytest
import torch

import paper_2502_02581_b200 as F
from paper_2502_02581_b200.comm import HeapLayout, emulated_group

from _golden import goldens

pytestmark = pytest.mark.gpu


def _groups(D, S, slots):
    layout = HeapLayout()
    off = layout.add("chunks", slots * S)
    groups = emulated_group(layout, D)
    return [F.ChunkBuffer(g, off, S, slots) for g in groups]


def run_spag(pre, post, S, seed):
    D, E = pre.num_devices, pre.num_chunks
    slots = max(len(post.chunks_on(d)) for d in range(D))
    bufs = _groups(D, S, slots)
    g = torch.Generator(device="cuda").manual_seed(seed)
    content = torch.randint(0, 256, (E, S), dtype=torch.uint8, device="cuda", generator=g)
    for d in range(D):
        m = F.chunk_slots(pre, post, d)
        v = bufs[d].view(rank=d)
        v.zero_()
        for e in pre.chunks_on(d):
            v[m[e]].copy_(content[e])
    for d in range(D):
        rep = F.sparse_all_gather(pre, post, bufs[d])
    torch.cuda.synchronize()
    for d in range(D):
        m = F.chunk_slots(pre, post, d)
        v = bufs[d].view(rank=d)
        for e in post.chunks_on(d):
            assert torch.equal(v[m[e]], content[e]), f"chunk {e} on device {d}"
    return rep


def run_sprs(pre, post, S, seed):
    """pre = materialized holders, post = the owner partition."""
    D, E = pre.num_devices, pre.num_chunks
    slots = max(len(pre.chunks_on(d)) for d in range(D))
    bufs = _groups(D, S, slots)
    g = torch.Generator(device="cuda").manual_seed(seed)
    parts = {}
    for d in range(D):
        m = F.chunk_slots(post, pre, d)
        v = bufs[d].view(torch.float32, rank=d)
        for e in pre.chunks_on(d):
            parts[(e, d)] = torch.randn(S // 4, device="cuda", generator=g)
            v[m[e]].copy_(parts[(e, d)])
    for d in range(D):
        rep = F.sparse_reduce_scatter(pre, post, bufs[d])
    torch.cuda.synchronize()
    for e in range(E):
        o = post.owner(e)
        acc = torch.zeros(S // 4, device="cuda")
        for h in sorted(pre.devices_of(e)):
            acc = acc + parts[(e, h)]
        got = bufs[o].view(torch.float32, rank=o)[F.chunk_slots(post, pre, o)[e]]
        assert torch.equal(got, acc), f"chunk {e} owner {o}"
    return rep


@pytest.mark.parametrize("D,r,variant", [(4, 2, "ring"), (4, 4, "ring"), (8, 3, "ring"),
                                         (4, 4, "hot"), (2, 2, "ring")])
def test_spag_sprs_ring_and_hot(D, r, variant):
    topo = F.ClusterTopology.for_nvswitch(D)
    E = D
    base = F.make_even_partition(E, topo)
    extra = ([(e, (e + i) % D) for e in range(E) for i in range(1, r)] if variant == "ring"
             else [(0, i) for i in range(1, r)])
    post = base.union(extra)
    S = 1 << 20
    rep = run_spag(base, post, S, seed=D * 10 + r)
    tr, exp = F.spag_traffic(base, post, S)
    assert rep == exp
    rep2 = run_sprs(post, base, S, seed=D * 10 + r + 1)
    assert rep2 == F.sprs_traffic(post, base, S)[1]
    assert rep2.total_interdevice_bytes == exp.total_interdevice_bytes


def test_reference_corpus_valid_pairs():
    cases = [c for c in goldens()["traffic"]
             if "error" not in c["spag"] and c["topo"][0] * c["topo"][1] <= 8]
    assert len(cases) >= 20
    for i, c in enumerate(cases[:40]):
        D = int(c["topo"][0]) * int(c["topo"][1])
        pre = F.ChunkPlacement.from_pairs(c["E"], D, c["pre"])
        post = F.ChunkPlacement.from_pairs(c["E"], D, c["post"])
        S = 64 << 10
        run_spag(pre, post, S, seed=i)
        if "error" not in c["sprs"]:
            run_sprs(post, pre, S, seed=1000 + i)


def test_invalid_pair_raises_before_device_work():
    topo = F.ClusterTopology.for_nvswitch(4)
    base = F.make_even_partition(4, topo)
    bufs = _groups(4, 1 << 16, 4)
    not_superset = F.ChunkPlacement.from_pairs(4, 4, [(0, 1), (1, 1), (2, 2), (3, 3)])
    with pytest.raises(F.InvalidPairError):
        F.sparse_all_gather(base, not_superset, bufs[0])
    with pytest.raises(F.InvalidPairError):
        F.sparse_reduce_scatter(base.union([(0, 2)]), not_superset, bufs[0])
    with pytest.raises(F.DimensionError):  # more chunks per rank than the buffer's slots
        F.sparse_all_gather(base, base.union([(e, 0) for e in range(4)]),
                            F.ChunkBuffer(bufs[0].group, bufs[0].offset, 1 << 16, 2))
