"""Re-materialization with ONE replica region shared by every layer (model_regions,
rematerialize=True): a layer's forward replicas are overwritten by the next layers'
SpAGs, so its backward must re-gather them (FssdpMoE.backward -> phase_spag(refetch_early)).
Multi-rank (4 emulated ranks, 3 layers, model-level parameter region) vs one rank: y and dx
of every layer bit-exact, owners' SpRS-reduced gradients within fp32 reordering; the
retain layout (per-layer replica slots) the same."""

import numpy as np
import pytest
import torch

import paper_2502_02581_b200 as F
from _torch_ref import grad_excess
from paper_2502_02581_b200.comm import HeapLayout, emulated_group
from paper_2502_02581_b200.layer import (FssdpMoE, layer_geometries, model_regions,
                                         replica_region_bytes, replica_slots,
                                         run_lockstep_backward, run_lockstep_forward)

pytestmark = pytest.mark.gpu


def build(world, L, E, d, f, T, pol, remat, bias):
    topo = F.ClusterTopology.for_nvswitch(world)
    cfg = F.ModelConfig(L, E, 2 * 2 * d * f, 2 * d, 1e-3, 1e-6)
    planners = [F.FssdpPlanner(cfg, topo, pol) for _ in range(world)]
    geoms = layer_geometries(planners[0], d, f, 2, T, replica_slots(planners[0]))
    layout = HeapLayout()
    geoms = model_regions(layout, geoms, remat)
    groups = emulated_group(layout, world)
    model = [[FssdpMoE(geoms[li], groups[r], planners[r], li, 11, prefix=f"L{li}.")
              for r in range(world)] for li in range(L)]
    for li, row in enumerate(model):
        for ly in row:
            ly.gate_bias.copy_(bias[li])
    return model, geoms


@pytest.mark.parametrize("remat", [True, False])
def test_shared_replica_region_remat_matches_single_rank(remat):
    world, L, E, d, f, Tr = 4, 3, 8, 256, 512, 384
    pol = F.Policy(F.PolicyKind.FSSDP, overlap_override=8, capacity_override=2,
                   rematerialize=remat, reshard_interval=0)
    rng = np.random.default_rng(2)
    bias = []
    for li in range(L):
        p = 1.0 / np.arange(1, E + 1) ** 1.3
        bias.append(torch.tensor(np.log(p[rng.permutation(E)] / p.sum()), dtype=torch.float32,
                                 device="cuda"))
    multi, geoms = build(world, L, E, d, f, Tr, pol, remat, bias)
    single, _ = build(1, L, E, d, f, world * Tr, F.Policy(F.PolicyKind.EP, reshard_interval=0),
                      False, bias)
    S = geoms[0].slot_param_bytes
    if remat:
        assert len({g.replica_base for g in geoms}) == 1
        assert replica_region_bytes(geoms) == 2 * S
    else:
        assert replica_region_bytes(geoms) == L * 2 * S
    gen = torch.Generator(device="cuda").manual_seed(3)
    replicas = 0
    for it in range(3):
        x = torch.randn(world * Tr, d, device="cuda", generator=gen).bfloat16()
        dy = (torch.randn(world * Tr, d, device="cuda", generator=gen) * 0.05).bfloat16()
        h, hs, ys, yss = list(x.split(Tr)), [x], [], []
        for li in range(L):
            h = run_lockstep_forward(multi[li], h)
            hs = run_lockstep_forward(single[li], hs)
            ys.append(torch.cat(h))
            yss.append(hs[0])
        g, gs, dxs, dxss = list(dy.split(Tr)), [dy], [], []
        for li in reversed(range(L)):
            g = run_lockstep_backward(multi[li], g, rematerialize=remat)
            gs = run_lockstep_backward(single[li], gs)
            dxs.append(torch.cat(g))
            dxss.append(gs[0])
        multi[0][0].planner.finish()
        for r in range(1, world):
            multi[0][r].planner.finish()
        single[0][0].planner.finish()
        torch.cuda.synchronize()
        for li in range(L):
            assert torch.equal(ys[li], yss[li]), f"it {it} layer {li} y"
            assert torch.equal(dxs[li], dxss[li]), f"it {it} layer {L - 1 - li} dx"
            dec = multi[li][0].decision
            replicas += len(dec.target.entries) - E
            for e in range(E):
                o = dec.base.owner(e)
                for gm, gs_ in zip(multi[li][o].expert_grad(e), single[li][0].expert_grad(e)):
                    assert grad_excess(gm, gs_) <= 0, f"it {it} layer {li} expert {e} grad"
    assert replicas > 0
