"""End-to-end FSSDP MoE layer (gate -> counts all-gather -> plan -> SpAG -> dispatch ->
grouped FFN -> combine; backward A2A -> dgrad/wgrad -> dX combine -> SpRS) on the GPU,
against the numpy oracle and across world sizes.

Multi-rank cases run N logical ranks in lockstep on one GPU (PeerGroup "emulated"):
separate symmetric heaps, real cross-heap peer addressing in every kernel.

Tolerances: bf16 outputs |Δ| <= 2e-2·max|ref| + 1e-3; fp32 gradients
|Δ| <= 2e-2·max|ref| + 1e-5.  Placement-independence is checked BIT-EXACTLY: y and dx
of a token do not depend on which rank computed its experts.
"""

import numpy as np
import pytest
import torch

import paper_2502_02581_b200 as F
from _torch_ref import grad_excess
from oracle import tensor_oracle as TO
from paper_2502_02581_b200.comm import HeapLayout, emulated_group
from paper_2502_02581_b200.layer import (FssdpMoE, LayerGeometry, default_slots,
                                         run_lockstep_backward, run_lockstep_forward)

pytestmark = pytest.mark.gpu


def build(world, E, d, f, k, T, policy, seed=0, bias=None, activation="gelu", grad_dtype="bf16"):
    m = policy.capacity_override if policy.capacity_override is not None else E
    geom = LayerGeometry(d, f, E, k, T, world, default_slots(E, world, m), activation,
                         grad_dtype=grad_dtype)
    layout = HeapLayout()
    geom.add_regions(layout, "L0.")
    groups = emulated_group(layout, world)
    topo = F.ClusterTopology.for_nvswitch(world)
    cfg = F.ModelConfig(1, E, geom.expert_bytes, 2 * d, 1e-3, 1e-6)
    layers = []
    for r in range(world):
        ly = FssdpMoE(geom, groups[r], F.FssdpPlanner(cfg, topo, policy), 0, seed)
        if bias is not None:
            ly.gate_bias.copy_(bias)
        layers.append(ly)
    return layers


def close(out, ref, rel=2e-2, abs_=1e-3, what=""):
    out = np.asarray(out, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.abs(out - ref).max() if out.size else 0.0
    bound = rel * (np.abs(ref).max() if ref.size else 0.0) + abs_
    assert err <= bound, f"{what}: max |Δ| {err:.4g} > {bound:.4g}"


def f32(t):
    return t.float().cpu().numpy()


def zipf_bias(E, s=1.2, seed=0):
    p = 1.0 / np.arange(1, E + 1) ** s
    p = p[np.random.default_rng(seed).permutation(E)]
    return torch.tensor(np.log(p / p.sum()), dtype=torch.float32, device="cuda")


@pytest.mark.parametrize("f,activation,grad_dtype", [
    (1024, "gelu", "bf16"), (1024, "gelu", "fp32"), (384, "gelu", "bf16"), (384, "swiglu", "bf16"),
    (512, "swiglu", "fp32")])
def test_single_rank_matches_oracle(f, activation, grad_dtype):
    """GeLU and SwiGLU experts; d_ff = 384 exercises 128-wide N tiles (and, for GeLU, the
    single-CTA wgrad1: d_ff / 128 is odd); bf16 and fp32 weight gradients."""
    E, d, k, T = 8, 256, 2, 1000
    pol = F.Policy(F.PolicyKind.FSSDP, overlap_override=4, capacity_override=2)
    (ly,) = build(1, E, d, f, k, T, pol, seed=3, bias=zipf_bias(E), activation=activation,
                  grad_dtype=grad_dtype)
    assert ly.grads.dtype == (torch.bfloat16 if grad_dtype == "bf16" else torch.float32)
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    dy = (torch.randn(T, d, device="cuda", generator=g) * 0.1).bfloat16()
    y = ly.forward(x)
    dx = ly.backward(dy)
    torch.cuda.synchronize()
    idx = ly.topk_idx[:T].cpu().numpy()
    w = ly.topk_w[:T].cpu().numpy()
    experts = {e: tuple(f32(t) for t in ly.expert_weight(e)) for e in range(E)}
    ref = TO.moe_layer_fwd_bwd(f32(x), idx, w, ly.wg.cpu().numpy(), experts, f32(dy))
    close(f32(y), ref["y"], what="y")
    # g = <dy, Y_slot>: tight against the device's own expert rows (the kernel's dot
    # product), loose against the oracle (bf16 rows differ by an ulp here and there)
    pos = ly.slot_pos[:T].long().cpu()
    y_rows = ly.y_e.float().cpu()[pos]                                    # [T, k, d]
    g_dev = torch.einsum("td,tkd->tk", dy.float().cpu(), y_rows).numpy()
    close(ly.slot_grad[:T].cpu().numpy(), g_dev, rel=1e-5, abs_=1e-5, what="g (own rows)")
    close(ly.slot_grad[:T].cpu().numpy(), ref["g"], rel=5e-3, abs_=1e-4, what="g")
    close(ly.dlogit[:T].cpu().numpy(), ref["dlogit"], rel=5e-3, abs_=1e-5, what="dlogit")
    close(f32(dx), ref["dx"], what="dx")
    for e in range(E):
        grads = ly.expert_grad(e)
        close(f32(grads[0]), ref["dW1"][e], rel=1e-2, abs_=1e-5, what=f"dW1[{e}]")
        close(f32(grads[-1]), ref["dW2"][e], rel=1e-2, abs_=1e-5, what=f"dW2[{e}]")
        if activation == "swiglu":
            close(f32(grads[1]), ref["dW3"][e], rel=1e-2, abs_=1e-5, what=f"dW3[{e}]")
    close(ly.dwg.cpu().numpy(), ref["dWg"], rel=1e-3, abs_=1e-5, what="dWg")
    # padding rows of the receive buffers are zero (wgrad K blocks rely on it)
    t = ly.tables
    xr = ly.xrecv.cpu()
    for s in range(len(t.seg_start)):
        a, b = int(t.seg_start[s] + t.seg_rows[s]), int(t.seg_start[s] + t.seg_padded[s])
        assert not xr[a:b].any()


@pytest.mark.parametrize("world,E,policy_kw,f,activation,grad_dtype", [
    (4, 8, dict(overlap_override=8, capacity_override=2), 512, "gelu", "bf16"),
    (4, 8, dict(overlap_override=8, capacity_override=2), 512, "gelu", "fp32"),
    (2, 16, dict(overlap_override=4, capacity_override=3, rematerialize=True), 512, "gelu", "bf16"),
    (8, 16, dict(overlap_override=6, capacity_override=2), 512, "gelu", "bf16"),
    (4, 8, dict(kind=F.PolicyKind.EP), 512, "gelu", "bf16"),
    (4, 8, dict(overlap_override=8, capacity_override=2, rematerialize=True), 384, "swiglu",
     "bf16"),
    (8, 16, dict(overlap_override=6, capacity_override=2), 384, "gelu", "fp32"),
])
def test_multi_rank_equals_single_rank(world, E, policy_kw, f, activation, grad_dtype):
    """FSSDP over N emulated ranks == the same tokens on one rank (y, dx bit-exact;
    SpRS-reduced owner grads within the gradient dtype's tolerance: grad_excess), over 3
    iterations so history-driven adoption and calibration both act."""
    d, k, Tr = 256, 2, 384
    kind = policy_kw.pop("kind", F.PolicyKind.FSSDP)
    pol = F.Policy(kind, **policy_kw)
    bias = zipf_bias(E, 1.3, seed=world)
    multi = build(world, E, d, f, k, Tr, pol, seed=7, bias=bias, activation=activation,
                  grad_dtype=grad_dtype)
    single = build(1, E, d, f, k, Tr * world, F.Policy(F.PolicyKind.EP), seed=7, bias=bias,
                   activation=activation, grad_dtype=grad_dtype)[0]
    g = torch.Generator(device="cuda").manual_seed(11)
    replicas_seen = prefetched = 0
    for it in range(3):
        x = torch.randn(world * Tr, d, device="cuda", generator=g).bfloat16()
        dy = (torch.randn(world * Tr, d, device="cuda", generator=g) * 0.05).bfloat16()
        xs = list(x.split(Tr))
        dys = list(dy.split(Tr))
        ys = run_lockstep_forward(multi, xs)
        dxs = run_lockstep_backward(multi, dys, rematerialize=pol.rematerialize)
        for ly in multi:
            ly.planner.finish()
        y1 = single.forward(x)
        dx1 = single.backward(dy)
        single.planner.finish()
        torch.cuda.synchronize()
        dec = multi[0].decision
        replicas_seen += len(dec.target.entries) - E
        prefetched += sum(ly.pre_tables.n_spag for ly in multi if ly.pre_tables is not None)
        # every rank computed the same plan
        for ly in multi[1:]:
            assert ly.decision.target == dec.target
            assert np.array_equal(ly.decision.route, dec.route)
        assert torch.equal(torch.cat(ys), y1), "y differs from the single-rank result"
        assert torch.equal(torch.cat(dxs), dx1), "dx differs from the single-rank result"
        # owners hold the SpRS-reduced gradient of every expert
        for e in range(E):
            owner = dec.base.owner(e)
            for j, (gm, gs) in enumerate(zip(multi[owner].expert_grad(e), single.expert_grad(e))):
                assert grad_excess(gm, gs) <= 0, f"grad{j}[{e}] it{it}"
        dwg = sum(ly.dwg.double() for ly in multi)
        close(dwg.cpu().numpy(), single.dwg.double().cpu().numpy(), rel=1e-4, abs_=1e-6,
              what="dWg")
        # SpAG: every replica slot is a bit-exact copy of the owner's shard
        for r, ly in enumerate(multi):
            for e, s in ly.tables.slots.items():
                o = dec.base.owner(e)
                if o == r:
                    continue
                os_ = multi[o].tables.slots[e]
                assert torch.equal(ly.params[s], multi[o].params[os_])
    if kind == F.PolicyKind.FSSDP:
        assert replicas_seen > 0, "the skewed loads should have produced replicas"
        assert prefetched > 0, "history-driven replicas should have been fetched early"
    else:
        assert replicas_seen == 0 and prefetched == 0



@pytest.mark.parametrize("world", [1, 2])
def test_late_dots_bit_identical(world, monkeypatch):
    """The gate's <dy, Y> dots computed in the dX combine (fssdp_combine_dx_dots, the
    default wherever the gate backward follows the dX combine) equal the dispatch_grad ones
    bit for bit, and so do dlogit, dx and dWg."""
    E, d, f, k, T = 8, 256, 512, 2, 777
    pol = F.Policy(F.PolicyKind.FSSDP, overlap_override=4, capacity_override=2)
    g = torch.Generator(device="cuda").manual_seed(11)
    xs = [torch.randn(T, d, device="cuda", generator=g).bfloat16() for _ in range(world)]
    dys = [(torch.randn(T, d, device="cuda", generator=g) * 0.1).bfloat16() for _ in range(world)]
    out = {}
    for late in (False, True):
        monkeypatch.setattr(FssdpMoE, "LATE_DOTS", late)
        monkeypatch.setattr(FssdpMoE, "EARLY_GATE", False)
        layers = build(world, E, d, f, k, T, pol, seed=2, bias=zipf_bias(E))
        assert all(ly._late_dots == late for ly in layers)
        ys = run_lockstep_forward(layers, xs) if world > 1 else [layers[0].forward(xs[0])]
        dxs = (run_lockstep_backward(layers, dys) if world > 1
               else [layers[0].backward(dys[0])])
        torch.cuda.synchronize()
        out[late] = [(y.clone(), dx.clone(), ly.slot_grad[:T].clone(), ly.dlogit[:T].clone(),
                      ly.dwg.clone()) for y, dx, ly in zip(ys, dxs, layers)]
        for ly in layers:
            ly.planner.finish()
    for a, b in zip(out[False], out[True]):
        for u, v in zip(a, b):
            assert torch.equal(u, v)


@pytest.mark.parametrize("world", [2, 4])
def test_p2p_gate_reduce(world, monkeypatch):
    """dWg summed over P2P (fssdp_sum_peers after the end barrier, the default at N > 1
    in a real process group): every rank gets the same bits — the rank-order fp32 sum of
    the gate partials — and it matches the single-rank dWg of the same tokens."""
    monkeypatch.setattr(FssdpMoE, "P2P_GATE_REDUCE_EMULATED", True)
    E, d, f, k, Tr = 8, 256, 512, 2, 300
    pol = F.Policy(F.PolicyKind.FSSDP, overlap_override=4, capacity_override=2)
    bias = zipf_bias(E)
    multi = build(world, E, d, f, k, Tr, pol, seed=4, bias=bias)
    single = build(1, E, d, f, k, Tr * world, F.Policy(F.PolicyKind.EP), seed=4, bias=bias)[0]
    assert all(ly._p2p_gate_reduce for ly in multi) and not single._p2p_gate_reduce
    g = torch.Generator(device="cuda").manual_seed(3)
    for it in range(3):  # both parities of the partial buffers
        x = torch.randn(world * Tr, d, device="cuda", generator=g).bfloat16()
        dy = (torch.randn(world * Tr, d, device="cuda", generator=g) * 0.1).bfloat16()
        run_lockstep_forward(multi, list(x.split(Tr)))
        run_lockstep_backward(multi, list(dy.split(Tr)))
        for ly in multi:
            ly.planner.finish()
        single.forward(x)
        single.backward(dy)
        single.planner.finish()
        torch.cuda.synchronize()
        parts = [ly.dwg_part[ly._gpar] for ly in multi]
        ref = parts[0].clone()
        for p in parts[1:]:
            ref = ref + p
        for ly in multi:
            assert torch.equal(ly.dwg, ref), f"it{it}: rank {ly.rank}"
        close(multi[0].dwg.double().cpu().numpy(), single.dwg.double().cpu().numpy(),
              rel=1e-4, abs_=1e-6, what="dWg")
