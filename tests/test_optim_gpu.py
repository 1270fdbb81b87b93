"""The training step over FSSDP shards: the fused AdamW kernel against a plain fp32 torch
AdamW, and — over emulated ranks with heterogeneous re-sharding on — the optimizer state
moving with its expert (params + fp32 master + both moments: the reference's 7x
expert_bytes per moved expert, engine.py:233, 444-453), replicas pulled from the UPDATED
owner shards, and the multi-rank run tracking the single-rank one."""

import ctypes as C

import numpy as np
import pytest
import torch

import paper_2502_02581_b200 as F
from paper_2502_02581_b200 import _native as N
from paper_2502_02581_b200.comm import HeapLayout, emulated_group
from paper_2502_02581_b200.layer import (FssdpMoE, layer_geometries, run_lockstep_backward,
                                         run_lockstep_forward)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("gdt", [torch.float32, torch.bfloat16])
def test_adam_kernel_matches_torch_adamw(gdt):
    torch.manual_seed(0)
    n = 1 << 20
    master = torch.randn(n, device="cuda")
    m = torch.randn(n, device="cuda") * 1e-3
    v = torch.rand(n, device="cuda") * 1e-4
    params = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    lr, b1, b2, eps, wd, step = 3e-3, 0.9, 0.95, 1e-8, 0.1, 7
    refs = (master.clone(), m.clone(), v.clone())
    for s in range(step, step + 3):
        g = torch.randn(n, device="cuda").to(gdt)
        rw, rm, rv = refs
        g32 = g.float()
        rm.mul_(b1).add_((1 - b1) * g32)
        rv.mul_(b2).add_((1 - b2) * g32 * g32)
        bc1, bc2 = 1 - b1 ** s, 1 - b2 ** s
        rw.sub_(lr * wd * rw)
        rw.sub_(lr * (rm / bc1) / ((rv / bc2).sqrt() + eps))
        N.call("fssdp_adam_step", C.c_void_p(params.data_ptr()), C.c_void_p(master.data_ptr()),
               C.c_void_p(m.data_ptr()), C.c_void_p(v.data_ptr()), C.c_void_p(g.data_ptr()),
               int(gdt == torch.bfloat16), n,
               lr, b1, b2, eps, wd, s, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    for name, got, ref in (("master", master, refs[0]), ("m", m, refs[1]), ("v", v, refs[2])):
        excess = ((got - ref).abs() - (3e-6 * ref.abs() + 1e-6 * ref.abs().max())).max().item()
        assert excess <= 0, f"{name}: {excess:.3g} over bound"  # 1-b1: f32 here, f64 in torch
    assert torch.equal(params, master.bfloat16())  # the working copy is the rounded master


def _model(world, pol, L, E, d, f, Tr, bias, grad_dtype="bf16"):
    topo = F.ClusterTopology.for_nvswitch(world)
    cfg = F.ModelConfig(L, E, 2 * 2 * d * f, 2 * d, 1e-3, 1e-6)
    planners = [F.FssdpPlanner(cfg, topo, pol) for _ in range(world)]
    m = pol.capacity_override if pol.capacity_override is not None else E
    geoms = layer_geometries(planners[0], d, f, 2, Tr, m, "gelu", optimizer=True,
                             grad_dtype=grad_dtype)
    layout = HeapLayout()
    for li, g in enumerate(geoms):
        g.add_regions(layout, f"L{li}.")
    groups = emulated_group(layout, world)
    model = [[FssdpMoE(geoms[li], groups[r], planners[r], li, 5, prefix=f"L{li}.")
              for r in range(world)] for li in range(L)]
    for li, row in enumerate(model):
        for ly in row:
            ly.gate_bias.copy_(bias[li])
    opts = [F.FssdpAdam([row[r] for row in model], lr=1e-3, weight_decay=0.01, gate=False)
            for r in range(world)]
    return model, opts, planners


def _owner_state(model, li, e, opts):
    """(params, master, m, v) of expert e of layer li on its current owner."""
    for r, ly in enumerate(model[li]):
        if e in ly._owned_expert_ids:
            st = opts[r].state_of(ly, e)
            s = ly._owned_expert_ids.index(e)
            return (ly.params[s].clone(), st["master"].clone(), st["m"].clone(), st["v"].clone())
    raise AssertionError(f"expert {e} of layer {li} has no owner")


@pytest.mark.parametrize("grad_dtype,drift", [("fp32", 0.05), ("bf16", 0.15)])
def test_optimizer_state_moves_with_reshard_and_replicas_follow_updates(grad_dtype, drift):
    """drift: bound on |Δ update| / |update| between the sharded and the single-rank run.
    Adam's first steps are ~lr·sign(g): an element whose holders' partials nearly cancel can
    flip sign under reduction-order (fp32) or partial-rounding (bf16 gradients) noise."""
    world, L, E, d, f, Tr = 4, 2, 8, 256, 512, 256
    pol = F.Policy(F.PolicyKind.FSSDP, overlap_override=4, capacity_override=2,
                   reshard_interval=2)
    rng = np.random.default_rng(4)
    bias = []
    for li in range(L):  # per-layer skews that differ, so heterogeneous sharding moves experts
        p = 1.0 / np.arange(1, E + 1) ** (1.0 + li)
        bias.append(torch.tensor(np.log(p[rng.permutation(E)] / p.sum()), dtype=torch.float32,
                                 device="cuda"))
    multi, opts, planners = _model(world, pol, L, E, d, f, Tr, bias, grad_dtype)
    single, sopts, _ = _model(1, F.Policy(F.PolicyKind.EP), L, E, d, f, world * Tr, bias,
                              grad_dtype)
    gen = torch.Generator(device="cuda").manual_seed(8)
    moved = replicas = 0
    init = {(li, e): _owner_state(single, li, e, sopts)[1] for li in range(L) for e in range(E)}
    for it in range(6):
        before = {(li, e): _owner_state(multi, li, e, opts) for li in range(L) for e in range(E)}
        x = torch.randn(world * Tr, d, device="cuda", generator=gen).bfloat16()
        dy = (torch.randn(world * Tr, d, device="cuda", generator=gen) * 0.05).bfloat16()
        h, hs = list(x.split(Tr)), [x]
        for li in range(L):
            h = run_lockstep_forward(multi[li], h)
            hs = run_lockstep_forward(single[li], hs)
        torch.cuda.synchronize()
        moved += len(planners[0].last_reshard_moves)
        for li in range(L):
            for e in range(E):  # the (possibly new) owner holds exactly the old owner's state
                after = _owner_state(multi, li, e, opts)
                for a, b in zip(before[(li, e)], after):
                    assert torch.equal(a, b), f"it {it}: state of L{li} e{e} changed in transit"
            for r, ly in enumerate(multi[li]):  # replicas = the owners' updated shards
                dec = ly.decision
                for e, s in ly.tables.slots.items():
                    o = dec.base.owner(e)
                    if o != r:
                        replicas += 1
                        assert torch.equal(ly.params[s], _owner_state(multi, li, e, opts)[0])
        g, gs = list(dy.split(Tr)), [dy]
        for li in reversed(range(L)):
            g = run_lockstep_backward(multi[li], g)
            gs = run_lockstep_backward(single[li], gs)
        for p_ in planners:
            p_.finish()
        single[0][0].planner.finish()
        for o in opts + sopts:
            o.step()
        torch.cuda.synchronize()
        lr = opts[0].lr
        for li in range(L):  # the sharded run tracks the single-rank one.  Adam's update is
            for e in range(E):  # ~sign(g)·lr: a gradient within fp32 reordering of zero may
                _, mm, _, _ = _owner_state(multi, li, e, opts)  # flip one element's step, so
                _, ms, _, _ = _owner_state(single, li, e, sopts)  # compare the updates' norms
                upd = (ms - init[(li, e)]).norm().item()
                assert (mm - ms).abs().max().item() <= 2.5 * lr * (it + 1), f"it {it} L{li} e{e}"
                assert (mm - ms).norm().item() <= drift * upd, \
                    f"it {it} L{li} e{e}: update differs"
    assert moved > 0, "the per-layer skews should trigger a re-shard"
    assert replicas > 0
