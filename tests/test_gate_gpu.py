"""K1 gate kernel: logits within tolerance of fp32, selection/ranks/counts bit-exact
against the CPU oracle applied to the device's own logits."""

import numpy as np
import pytest
import torch

from oracle import tensor_oracle as TO

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("T,d,E,k", [(1000, 256, 8, 2), (4096, 1024, 16, 2), (777, 2048, 64, 2),
                                     (130, 512, 16, 4), (64, 128, 4, 1)])
def test_gate_topk_matches_oracle(T, d, E, k):
    from paper_2502_02581_b200 import ops

    g = torch.Generator().manual_seed(T + d + E)
    x = torch.randn(T, d, generator=g).bfloat16()
    wg = torch.randn(E, d, generator=g) / d ** 0.5
    wg[:, :] += torch.linspace(-0.5, 0.5, E)[:, None] / d  # mild skew
    idx, w, rank, tc, logits = ops.gate_topk(x.cuda(), wg.cuda(), k, want_logits=True)
    torch.cuda.synchronize()
    lg = logits.cpu().numpy()
    ref_lg = TO.gate_logits(x.float().numpy(), wg.numpy())
    assert np.abs(lg - ref_lg).max() <= 1e-4 * max(1.0, np.abs(ref_lg).max())
    o_idx, o_w, o_rank, o_tc = TO.topk_select(lg, k)
    np.testing.assert_array_equal(idx.cpu().numpy(), o_idx)
    np.testing.assert_array_equal(rank.cpu().numpy(), o_rank)
    np.testing.assert_array_equal(tc.cpu().numpy(), o_tc)
    # weights: device expf vs numpy float32 exp differ by an ulp or two, amplified by the
    # renormalisation -> stated tolerance rtol 2e-6 (selection itself is bit-exact above)
    np.testing.assert_allclose(w.cpu().numpy(), o_w, rtol=2e-6, atol=0)
    assert tc.cpu().numpy().sum() == T * k


def test_topk_ties_pick_lower_expert():
    from paper_2502_02581_b200 import ops

    T, E, k = 200, 16, 2
    lg = np.zeros((T, E), dtype=np.float32)
    lg[:, 5] = 1.0
    lg[::2, 9] = 1.0  # exact tie with expert 5 on even tokens
    idx, w, rank, tc = ops.topk_from_logits(torch.from_numpy(lg).cuda(), k)
    torch.cuda.synchronize()
    o_idx, o_w, o_rank, o_tc = TO.topk_select(lg, k)
    np.testing.assert_array_equal(idx.cpu().numpy(), o_idx)
    assert (idx.cpu().numpy()[::2] == [5, 9]).all()
    assert (idx.cpu().numpy()[1::2] == [5, 0]).all()
    np.testing.assert_array_equal(rank.cpu().numpy(), o_rank)
    np.testing.assert_array_equal(tc.cpu().numpy(), o_tc)


@pytest.mark.parametrize("T,d,E,k", [(16384, 1024, 16, 2), (1000, 256, 8, 2), (777, 2048, 64, 2),
                                     (130, 192, 16, 4)])
def test_gate_route_fused_equals_two_kernels(T, d, E, k):
    """fssdp_gate_route (gate + last-CTA scan / count all-gather) == fssdp_gate_topk followed
    by fssdp_route_scan_allgather, bit for bit, and leaves its workspace zeroed (twice)."""
    import ctypes as C

    from paper_2502_02581_b200 import _native as N
    from paper_2502_02581_b200 import ops
    from paper_2502_02581_b200.comm import HeapLayout, emulated_group
    from paper_2502_02581_b200.plan_tables import NativeTables, _layout

    g = torch.Generator().manual_seed(T + d)
    x = torch.randn(T, d, generator=g).bfloat16().cuda()
    wg = (torch.randn(E, d, generator=g) / d ** 0.5).cuda()
    bias = torch.linspace(-1, 1, E).cuda()
    layout = HeapLayout()
    layout.add("counts", 4 * E * 4)
    (grp,) = emulated_group(layout, 1)
    pb, off, flags = C.c_void_p(grp.peer_bases.data_ptr()), layout.offset("counts"), layout.offset("flags")
    table = grp.local.tensor(off, (E,), torch.int32)
    tiles = (T + ops.GATE_TILE - 1) // ops.GATE_TILE
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    idx, w, rank, tc, _ = ops.gate_topk(x, wg, k, bias=bias)
    prefix = torch.empty(tiles, E, dtype=torch.int32, device="cuda")
    N.call("fssdp_route_scan_allgather", ops._ptr(tc), tiles, E, ops._ptr(prefix), pb, off, flags,
           0, 1, -1, 0, s)
    torch.cuda.synchronize()
    want = [t.cpu().clone() for t in (idx, w, rank, tc, prefix, table)]
    ws = torch.zeros(1 + E, dtype=torch.int32, device="cuda")
    offs, nbytes = _layout(E, 1)
    blob = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    for local in (False, True):
        out = [torch.empty_like(t) for t in (idx, w, rank, tc, prefix)]
        table.zero_()
        host = torch.zeros(((E * 4 + 15) // 16 * 16) // 4 + 4, dtype=torch.int32,
                           pin_memory=True)
        flag_ptr = host.data_ptr() + (E * 4 + 15) // 16 * 16
        N.call("fssdp_gate_route", ops._ptr(x), ops._ptr(wg), ops._ptr(bias), T, d, E, k,
               *[ops._ptr(t) for t in out], ops._ptr(ws), pb, off, flags, 0, 1, -1, 0,
               ops._ptr(blob) if local else None, 512 if local and d % 256 == 0 else 0, 2, 0,
               C.c_void_p(host.data_ptr() if local else 0), (E * 4 + 15) // 16 * 16,
               C.c_void_p(flag_ptr if local else 0), C.c_uint32(7), None, 0, s)
        torch.cuda.synchronize()
        for a, b in zip(want, [t.cpu() for t in out] + [table.cpu()]):
            assert torch.equal(a, b)
        assert not ws.any()
        if local:  # the counts row pushed to the mapped host buffer, then the flag
            assert torch.equal(host[:E], want[5].reshape(-1)[:E]) and int(host[-4]) == 7
    assert int(want[5].sum()) == T * k
    # the single-rank dispatch tables the gate wrote == the host builder's for one device
    counts = want[5].numpy().astype(np.int64)
    host = NativeTables(0, np.zeros(E, np.int32), np.ones((E, 1), np.uint8), counts[None, :, None],
                        256, 256)
    dev = blob.cpu().numpy()

    def sec(name, n):
        return dev[offs[name]:offs[name] + 4 * n].view(np.int32)

    assert np.array_equal(sec("route_cum", 2 * E).reshape(E, 2), host.route_cum)
    assert np.array_equal(sec("recv_base", E).reshape(E, 1), host.recv_base)
    zr = sec("zero_rows", 2 * E).reshape(E, 2)
    assert np.array_equal(zr[zr[:, 1] > 0], host.zero_rows)
    if d % 256 == 0:  # the gate's tail wrote the GEMM tables too (local_d_ff = 512)
        ht = NativeTables(0, np.zeros(E, np.int32), np.ones((E, 1), np.uint8),
                          counts[None, :, None], d, 512)
        for name in ("fwd1", "fwd2", "dgrad2", "dgrad1", "wgrad1", "wgrad2"):
            want_g = ht.groups(name).tobytes()
            assert dev[offs[name]:offs[name] + len(want_g)].tobytes() == want_g, name
    # ... and the six grouped-GEMM tables fssdp_local_gemm_tables writes from those totals
    # == the host builder's, byte for byte (the forward GEMMs run on them before the plan)
    # (base > 0: the layer's owned slots start at that slot of a model-level region)
    for dm, dff, nm, base in ((1024, 4096, 2, 0), (2048, 1408, 3, 0), (256, 1024, 2, 0),
                              (1024, 4096, 2, 2 * E)):
        blob.zero_()
        N.call("fssdp_local_gemm_tables", pb, 0, off, E, dm, dff, nm, base, ops._ptr(blob), s)
        torch.cuda.synchronize()
        dev = blob.cpu().numpy()
        host = NativeTables(0, np.zeros(E, np.int32), np.ones((E, 1), np.uint8),
                            counts[None, :, None], dm, dff, n_mats=nm,
                            slot_layout=(base, base + E) if base else None)
        for name in ("fwd1", "fwd2", "dgrad2", "dgrad1", "wgrad1", "wgrad2"):
            want_g = host.groups(name)
            got = dev[offs[name]:offs[name] + want_g.nbytes]
            assert got.tobytes() == want_g.tobytes(), (name, dm, dff, nm)


@pytest.mark.parametrize("T,d,E,k", [(16384, 1024, 16, 2), (16384, 2048, 64, 2), (1000, 256, 8, 2),
                                     (777, 4096, 8, 2), (130, 192, 16, 4)])
def test_tensor_core_gate_route(T, d, E, k):
    """The tcgen05 gate path of fssdp_gate_route (logits = x . [hi(Wg); lo(Wg)] as one
    grouped-GEMM launch, then selection + the count tail): logits within 1e-4 of the fp64
    product, selection / weights / ranks / tile counts / prefixes bit-exact with
    fssdp_topk_from_logits applied to those same logits, totals all-gathered, workspace
    left zero."""
    import ctypes as C

    from paper_2502_02581_b200 import _native as N
    from paper_2502_02581_b200 import ops
    from paper_2502_02581_b200.comm import HeapLayout, emulated_group

    g = torch.Generator().manual_seed(T + d + E)
    x = torch.randn(T, d, generator=g).bfloat16().cuda()
    wg = (torch.randn(E, d, generator=g) / d ** 0.5).cuda()
    bias = torch.linspace(-1, 1, E).cuda()
    layout = HeapLayout()
    layout.add("counts", 4 * E * 4)
    (grp,) = emulated_group(layout, 1)
    pb, off, flags = C.c_void_p(grp.peer_bases.data_ptr()), layout.offset("counts"), layout.offset("flags")
    table = grp.local.tensor(off, (E,), torch.int32)
    tiles = (T + ops.GATE_TILE - 1) // ops.GATE_TILE
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    nbytes = int(N.LIB.fssdp_gate_gemm_ws_bytes(T, d))
    gws = torch.full((nbytes,), 0x7F, dtype=torch.uint8, device="cuda")  # garbage: no init needed
    ws = torch.zeros(1 + E, dtype=torch.int32, device="cuda")
    out = [torch.empty(T, k, dtype=torch.int32, device="cuda"),
           torch.empty(T, k, dtype=torch.float32, device="cuda"),
           torch.empty(T, k, dtype=torch.int32, device="cuda"),
           torch.empty(tiles, E, dtype=torch.int32, device="cuda"),
           torch.empty(tiles, E, dtype=torch.int32, device="cuda")]
    for _ in range(2):
        table.zero_()
        N.call("fssdp_gate_route", ops._ptr(x), ops._ptr(wg), ops._ptr(bias), T, d, E, k,
               *[ops._ptr(t) for t in out], ops._ptr(ws), pb, off, flags, 0, 1, -1, 0, None, 0,
               2, 0, None, 0, None, C.c_uint32(0), ops._ptr(gws), nbytes, s)
        torch.cuda.synchronize()
        assert not ws.any()
    # the logits the selection used: C [rows, 128] fp32 after the 1 KB header and B
    cm_off = 1024 + (128 * d * 2 + 1023) // 1024 * 1024
    cmat = gws[cm_off:cm_off + T * 128 * 4].view(torch.float32).view(T, 128)
    logits = (cmat[:, :E] + cmat[:, E:2 * E]) + bias
    ref = (x.double() @ wg.double().T) + bias.double()
    assert (logits.double() - ref).abs().max().item() <= 1e-4 * ref.abs().max().item()
    idx, w, rank, tc = ops.topk_from_logits(logits.contiguous(), k)
    assert torch.equal(out[0], idx) and torch.equal(out[1], w)
    assert torch.equal(out[2], rank) and torch.equal(out[3], tc)
    prefix = torch.cumsum(tc, 0) - tc
    assert torch.equal(out[4], prefix.int())
    assert torch.equal(table, tc.sum(0).int())


@pytest.mark.parametrize("T,d,E,k", [(1000, 256, 8, 2), (16384, 1024, 16, 2), (3000, 2048, 64, 2),
                                     (130, 512, 16, 4), (0, 256, 8, 2)])
def test_tensor_core_gate_wgrad(T, d, E, k):
    """fssdp_gate_wgrad_tc (dlogit as bf16 hi/lo, split-T tcgen05 GEMM, fixed-order reduce)
    against an fp64 sum and the SIMT fssdp_gate_wgrad; deterministic across calls."""
    import ctypes as C

    from paper_2502_02581_b200 import _native as N

    g = torch.Generator().manual_seed(T + d + E)
    x = torch.randn(max(T, 1), d, generator=g).bfloat16()[:T]
    idx = torch.stack([torch.randperm(E, generator=g)[:k] for _ in range(T)]) if T else \
        torch.zeros(0, k, dtype=torch.int64)
    dl = torch.randn(T, k, generator=g) * 0.1
    ref = torch.zeros(E, d, dtype=torch.float64)
    ref.index_add_(0, idx.reshape(-1), (dl.double()[:, :, None] * x.double()[:, None, :])
                   .reshape(-1, d))
    xd, idd, dld = x.cuda(), idx.int().cuda(), dl.float().cuda()
    ws = torch.empty(int(N.LIB.fssdp_gate_wgrad_tc_ws_bytes(T, d)), dtype=torch.uint8,
                     device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    outs = []
    for _ in range(2):
        dwg = torch.full((E, d), float("nan"), device="cuda")
        N.call("fssdp_gate_wgrad_tc", C.c_void_p(xd.data_ptr()), C.c_void_p(idd.data_ptr()),
               C.c_void_p(dld.data_ptr()), T, d, E, k, C.c_void_p(ws.data_ptr()), ws.numel(),
               C.c_void_p(dwg.data_ptr()), st)
        outs.append(dwg)
    wsimt = torch.empty(max(1, (T + 63) // 64) * E * d, device="cuda")
    simt = torch.empty(E, d, device="cuda")
    N.call("fssdp_gate_wgrad", C.c_void_p(xd.data_ptr()), C.c_void_p(idd.data_ptr()),
           C.c_void_p(dld.data_ptr()), T, d, E, k, C.c_void_p(wsimt.data_ptr()),
           C.c_void_p(simt.data_ptr()), st)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])  # deterministic
    got = outs[0].double().cpu()
    scale = max(ref.abs().max().item(), 1e-30)
    assert (got - ref).abs().max().item() <= 1e-5 * scale + 1e-7, "tensor-core dWg vs fp64"
    assert (simt.double().cpu() - got).abs().max().item() <= 2e-5 * scale + 1e-7
