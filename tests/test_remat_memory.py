"""Re-materialization saves memory (moesim memory_report, engine.py:188-226): the heap
holds every layer's OWNED slots, and replica slots for all layers (retain: Σ over layers)
or ONE shared set (rematerialize: max over layers) — equal to memory_report's
materialized bytes of a worst-case plan (every device adds its m replicas in every layer).
Pure host logic (heap layout), CPU."""

import numpy as np
import pytest

import paper_2502_02581_b200 as F
from paper_2502_02581_b200.comm import HeapLayout
from paper_2502_02581_b200.layer import (layer_geometries, model_regions, replica_region_bytes,
                                         replica_slots)


class _Mat:
    def __init__(self, added):
        self.added_per_device = tuple(added)


@pytest.mark.parametrize("remat", [False, True])
@pytest.mark.parametrize("L,E,D,m", [(3, 16, 4, 4), (4, 8, 8, 2), (1, 16, 8, 4)])
def test_replica_region_equals_memory_report(remat, L, E, D, m):
    d, f = 256, 512
    S = 2 * 2 * d * f
    topo = F.ClusterTopology.for_nvswitch(D)
    cfg = F.ModelConfig(L, E, S, 2 * d, 1e-3, 1e-6)
    pol = F.Policy(F.PolicyKind.FSSDP, overlap_override=4, capacity_override=m,
                   rematerialize=remat, reshard_interval=0)
    planner = F.FssdpPlanner(cfg, topo, pol)
    assert replica_slots(planner) == m
    geoms = model_regions(HeapLayout(), layer_geometries(planner, d, f, 2, 256, m), remat)
    worst = [_Mat([m] * D) for _ in range(L)]
    rep = F.memory_report(planner.shards, worst, cfg, "rematerialize" if remat else "retain")
    assert replica_region_bytes(geoms) == rep.materialized_bytes.max()
    # owned slots: every layer's shard of this device, once (with re-sharding on, each layer
    # reserves what a re-shard could give it: test_reshard_capacity_covers_slot_totals)
    assert sum(g.owned_cap for g in geoms) * S == rep.param_bytes.max()
    if remat and L > 1:
        assert len({g.replica_base for g in geoms}) == 1
    # gradients: owned slots only (a replica's partial is pushed to its owner's staging)
    layout = HeapLayout()
    geoms = model_regions(layout, layer_geometries(planner, d, f, 2, 256, m), remat)
    grads = sum(layout.regions[f"L{li}.grads"][1] for li in range(L))
    assert grads == rep.param_bytes.max()  # bf16: the reference's grad bytes = param bytes
    layout = HeapLayout()
    geoms = model_regions(layout, layer_geometries(planner, d, f, 2, 256, m, grad_dtype="fp32"),
                          remat)
    grads = sum(layout.regions[f"L{li}.grads"][1] for li in range(L))
    assert grads == 2 * rep.param_bytes.max()  # fp32 = 2x the bf16 expert bytes


def test_free_bytes_sizes_the_replica_slots():
    """With no capacity_override, m = free_bytes_per_device // expert_bytes (engine.py:389-402)."""
    S = 2 * 2 * 256 * 512
    cfg = F.ModelConfig(2, 16, S, 512, 1e-3, 1e-6)
    pol = F.Policy(F.PolicyKind.FSSDP, overlap_override=4, free_bytes_per_device=3 * S + 5)
    assert replica_slots(F.FssdpPlanner(cfg, F.ClusterTopology.for_nvswitch(4), pol)) == 3
    ep = F.Policy(F.PolicyKind.EP)
    assert replica_slots(F.FssdpPlanner(cfg, F.ClusterTopology.for_nvswitch(4), ep)) == 0


def test_reshard_capacity_covers_slot_totals():
    """Re-sharding may hand one layer up to the device's whole ShardPlan slot total
    (placement.py:240-250): each layer's owned capacity covers it."""
    L, E, D = 3, 16, 4
    S = 2 * 2 * 256 * 512
    cfg = F.ModelConfig(L, E, S, 512, 1e-3, 1e-6)
    pol = F.Policy(F.PolicyKind.FSSDP, overlap_override=4, capacity_override=2,
                   reshard_interval=5)
    planner = F.FssdpPlanner(cfg, F.ClusterTopology.for_nvswitch(D), pol)
    geoms = layer_geometries(planner, 256, 512, 2, 256, 2)
    assert all(g.owned_cap >= planner.shards.slots_per_device for g in geoms)
