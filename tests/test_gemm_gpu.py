"""tcgen05 grouped GEMM (K5/K7) against a plain PyTorch fp32 reference.

Tolerance (bf16 operands, fp32 accumulate, bf16 output): |Δ| <= 2e-2·max|ref| + 1e-3
per tensor.  fp32 outputs (wgrad) use 2e-3·max|ref| + 1e-4.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ops():
    from paper_2502_02581_b200 import ops

    return ops


def _groups(ops, rows, n_tiles, dev):
    g = np.zeros(len(rows), dtype=ops.GROUP_DTYPE)
    for i, r in enumerate(rows):
        (g["m_tiles"][i], g["a_m"][i], g["a_k"][i], g["b_n"][i], g["b_k"][i], g["k_blocks"][i],
         g["c_off"][i]) = r
    total = ops.finalize_groups(g, n_tiles)
    return torch.from_numpy(g.view(np.uint8).copy()).to(dev), len(rows), total


def _close(out, ref, rel=2e-2, abs_=1e-3):
    out = out.float()
    ref = ref.float()
    err = (out - ref).abs().max().item()
    bound = rel * ref.abs().max().item() + abs_
    assert err <= bound, f"max |Δ| {err:.4g} > {bound:.4g}"


@pytest.mark.parametrize("epi,nf", [("bf16", False), ("bf16", True), ("gelu", False),
                                    ("dgelu", False), ("dgelu", True)])
def test_kmajor_kmajor_grouped(epi, nf):
    """fwd-style: A [R,K] K-major rows per group, B [G*N, K] K-major per-group weights."""
    ops = _ops()
    dev = "cuda"
    torch.manual_seed(0)
    K, N = 320, 512
    m_tiles = [1, 3, 0, 2]
    G = len(m_tiles)
    R = sum(m_tiles) * 128
    A = torch.randn(R, K, device=dev).bfloat16()
    B = (torch.randn(G * N, K, device=dev) / K ** 0.5).bfloat16()
    C = torch.zeros(R, N, device=dev, dtype=torch.bfloat16)
    C2 = torch.zeros_like(C)
    aux = torch.randn(R, N, device=dev).bfloat16()
    rows, r0 = [], 0
    for g, mt in enumerate(m_tiles):
        rows.append((mt, r0, 0, g * N, 0, K // 64, r0 * N))
        r0 += mt * 128
    gd, ng, total = _groups(ops, rows, N // 256, dev)
    e = {"bf16": ops.EPI_BF16, "gelu": ops.EPI_GELU, "dgelu": ops.EPI_DGELU}[epi]
    ops.grouped_gemm(A, False, B, False, gd, ng, N // 256, total, C, N, epilogue=e, c2=C2, n_fastest=nf,
                     aux=aux)
    torch.cuda.synchronize()
    ref = torch.zeros(R, N, device=dev)
    r0 = 0
    for g, mt in enumerate(m_tiles):
        sl = slice(r0, r0 + mt * 128)
        ref[sl] = A[sl].float() @ B[g * N:(g + 1) * N].float().T
        r0 += mt * 128
    if epi == "bf16":
        _close(C, ref)
    elif epi == "gelu":  # C = gelu'(acc) (saved for backward), C2 = gelu(acc)
        _close(C, gelu_grad(ref))
        _close(C2, torch.nn.functional.gelu(ref, approximate="tanh"))
    else:  # C = acc * aux
        _close(C, ref * aux.float())


def gelu_grad(a):
    k0, k1 = 0.7978845608028654, 0.044715
    t = torch.tanh(k0 * (a + k1 * a ** 3))
    return 0.5 * (1 + t) + 0.5 * a * (1 - t * t) * k0 * (1 + 3 * k1 * a * a)


def test_kmajor_mnmajor_dgrad_style():
    """dgrad-style: A [R,K] K-major, B stored [G*K, N] (N contiguous) = MN-major."""
    ops = _ops()
    dev = "cuda"
    torch.manual_seed(1)
    K, N = 256, 768
    m_tiles = [2, 1, 3]
    G = len(m_tiles)
    R = sum(m_tiles) * 128
    A = torch.randn(R, K, device=dev).bfloat16()
    B = (torch.randn(G * K, N, device=dev) / K ** 0.5).bfloat16()
    C = torch.zeros(R, N, device=dev, dtype=torch.bfloat16)
    rows, r0 = [], 0
    for g, mt in enumerate(m_tiles):
        rows.append((mt, r0, 0, 0, g * K, K // 64, r0 * N))
        r0 += mt * 128
    gd, ng, total = _groups(ops, rows, N // 256, dev)
    ops.grouped_gemm(A, False, B, True, gd, ng, N // 256, total, C, N)
    torch.cuda.synchronize()
    ref = torch.zeros(R, N, device=dev)
    r0 = 0
    for g, mt in enumerate(m_tiles):
        sl = slice(r0, r0 + mt * 128)
        ref[sl] = A[sl].float() @ B[g * K:(g + 1) * K].float()
        r0 += mt * 128
    _close(C, ref)


@pytest.mark.parametrize("a_mn", [True, False])
def test_wgrad_style_token_k(a_mn):
    """wgrad-style: K = token segments (incl. an empty one), fp32 output per group."""
    ops = _ops()
    dev = "cuda"
    torch.manual_seed(2)
    M, N = 256, 512
    segs = [128, 0, 384, 64]  # tokens per group (multiples of 64)
    G = len(segs)
    Rt = sum(segs)
    Bt = torch.randn(Rt, N, device=dev).bfloat16()  # [tokens, N]  (MN-major B)
    if a_mn:
        At = torch.randn(Rt, M, device=dev).bfloat16()  # [tokens, M]  (MN-major A)
    else:
        At = torch.randn(M * G, Rt, device=dev).bfloat16()  # unused layout for K-major A
    C = torch.full((G * M, N), 7.0, device=dev)
    rows, k0 = [], 0
    for g, s in enumerate(segs):
        if a_mn:
            rows.append((M // 128, 0, k0, 0, k0, s // 64, g * M * N))
        else:
            rows.append((M // 128, g * M, k0, 0, k0, s // 64, g * M * N))
        k0 += s
    gd, ng, total = _groups(ops, rows, N // 256, dev)
    ops.grouped_gemm(At, a_mn, Bt, True, gd, ng, N // 256, total, C, N, epilogue=ops.EPI_F32)
    torch.cuda.synchronize()
    k0 = 0
    for g, s in enumerate(segs):
        if a_mn:
            a = At[k0:k0 + s].float().T
        else:
            a = At[g * M:(g + 1) * M, k0:k0 + s].float()
        ref = a @ Bt[k0:k0 + s].float()
        _close(C[g * M:(g + 1) * M], ref, rel=2e-3, abs_=1e-4)
        k0 += s


@pytest.mark.parametrize("a_mn,b_mn,epi", [(False, False, "bf16"), (False, False, "gelu"),
                                           (False, True, "dgelu"), (False, True, "bf16"),
                                           (True, True, "f32")])
@pytest.mark.parametrize("nf", [False, True])
def test_cta_pair_tiles(a_mn, b_mn, epi, nf):
    """tcgen05 cta_group::2 (256 x 256 tiles over a CTA pair): every operand major-ness and
    epilogue the layer uses, groups with even 128-row tile counts (incl. an empty group)."""
    ops = _ops()
    dev = "cuda"
    torch.manual_seed(7)
    K, N = 384, 512
    m_tiles = [2, 4, 0, 2]
    G = len(m_tiles)
    R = sum(m_tiles) * 128
    e = {"bf16": ops.EPI_BF16, "gelu": ops.EPI_GELU, "dgelu": ops.EPI_DGELU,
         "f32": ops.EPI_F32}[epi]
    if not a_mn:
        A = torch.randn(R, K, device=dev).bfloat16()                        # [M][K]
    else:
        A = torch.randn(K * G, 256, device=dev).bfloat16()                  # [K][M] per group
    if not b_mn:
        B = (torch.randn(G * N, K, device=dev) / K ** 0.5).bfloat16()       # [N][K]
    else:
        B = (torch.randn(G * K, N, device=dev) / K ** 0.5).bfloat16()       # [K][N]
    rows, refs, r0 = [], [], 0
    if a_mn:  # wgrad-like: M = 256 per group, K = per-group token rows
        C = torch.zeros(G * 256, N, device=dev)
        for g in range(G):
            kb = (K // 64) if m_tiles[g] else 0
            rows.append((2, 0, g * K, 0, g * K, kb, g * 256 * N))
            ref = A[g * K:(g + 1) * K].float().T @ B[g * K:(g + 1) * K].float()
            refs.append((slice(g * 256, (g + 1) * 256), ref if kb else torch.zeros_like(ref)))
    else:
        C = torch.zeros(R, N, device=dev, dtype=torch.bfloat16)
        for g, mt in enumerate(m_tiles):
            if b_mn:
                rows.append((mt, r0, 0, 0, g * K, K // 64, r0 * N))
                ref = A[r0:r0 + mt * 128].float() @ B[g * K:(g + 1) * K].float()
            else:
                rows.append((mt, r0, 0, g * N, 0, K // 64, r0 * N))
                ref = A[r0:r0 + mt * 128].float() @ B[g * N:(g + 1) * N].float().T
            refs.append((slice(r0, r0 + mt * 128), ref))
            r0 += mt * 128
    C2 = torch.zeros_like(C)
    aux = torch.randn(C.shape, device=dev).bfloat16() if epi == "dgelu" else None
    gd, ng, total = _groups(ops, rows, N // 256, dev)
    ops.grouped_gemm(A, a_mn, B, b_mn, gd, ng, N // 256, total, C, N, epilogue=e,
                     c2=C2 if epi == "gelu" else None, aux=aux, n_fastest=nf, cta_pair=True)
    torch.cuda.synchronize()
    for sl, ref in refs:
        if ref.numel() == 0:
            continue
        if epi == "f32":
            _close(C[sl], ref, rel=2e-3, abs_=1e-4)
        elif epi == "dgelu":
            _close(C[sl], ref * aux[sl].float())
        elif epi == "gelu":
            _close(C[sl], gelu_grad(ref))
            _close(C2[sl], torch.nn.functional.gelu(ref, approximate="tanh"))
        else:
            _close(C[sl], ref)


def test_large_square_against_torch():
    """One big group (the throughput shape family) for a sanity check of the pipeline."""
    ops = _ops()
    dev = "cuda"
    torch.manual_seed(3)
    M, K, N = 2048, 1024, 4096
    A = torch.randn(M, K, device=dev).bfloat16()
    B = (torch.randn(N, K, device=dev) / K ** 0.5).bfloat16()
    C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    gd, ng, total = _groups(ops, [(M // 128, 0, 0, 0, 0, K // 64, 0)], N // 256, dev)
    ops.grouped_gemm(A, False, B, False, gd, ng, N // 256, total, C, N)
    torch.cuda.synchronize()
    _close(C, A.float() @ B.float().T)


@pytest.mark.parametrize("pair", [False, True])
def test_wgrad_c_dest_scatter(pair):
    """Groups with c_dest > 0 store through the given tensor maps (the push-SpRS wire):
    here two extra fp32 buffers stand in for two owners' staging regions."""
    ops = _ops()
    dev = "cuda"
    torch.manual_seed(4)
    M, N = 256, 512
    segs = [256, 128, 384]
    dests = [0, 2, 1]          # group 0 -> C, group 1 -> buffer #2 slot 1, group 2 -> #1 slot 0
    slots = [0, 1, 0]
    Rt = sum(segs)
    At = torch.randn(Rt, M, device=dev).bfloat16()
    Bt = torch.randn(Rt, N, device=dev).bfloat16()
    C = torch.zeros(2 * M, N, device=dev)
    stage = [torch.full((2 * M, N), 5.0, device=dev) for _ in range(2)]
    maps = b"".join(ops.epilogue_tmap(ops.EPI_F32, s.data_ptr(), N, 2 * M) for s in stage)
    maps_dev = torch.frombuffer(bytearray(maps), dtype=torch.uint8).to(dev)
    g = np.zeros(len(segs), dtype=ops.GROUP_DTYPE)
    k0 = 0
    for i, s in enumerate(segs):
        g[i] = (M // 128, 0, 0, k0, 0, k0, s // 64, dests[i], slots[i] * M * N, 0, 0)
        k0 += s
    total = ops.finalize_groups(g, N // 256)
    gd = torch.from_numpy(g.view(np.uint8).copy()).to(dev)
    ops.grouped_gemm(At, True, Bt, True, gd, len(segs), N // 256, total, C, N,
                     epilogue=ops.EPI_F32, cta_pair=pair, c_dest_maps=maps_dev)
    torch.cuda.synchronize()
    k0 = 0
    for i, s in enumerate(segs):
        ref = At[k0:k0 + s].float().T @ Bt[k0:k0 + s].float()
        out = C if dests[i] == 0 else stage[dests[i] - 1]
        _close(out[slots[i] * M:(slots[i] + 1) * M], ref, rel=2e-3, abs_=1e-4)
        k0 += s
    assert torch.all(stage[1][:M] == 5.0)  # untouched staging slots stay
    assert torch.all(stage[0][M:] == 5.0)
    assert torch.all(C[M:] == 0.0)


def _interleave(w1, w3):
    f, k = w1.shape
    return torch.stack([w1.view(f // 128, 128, k), w3.view(f // 128, 128, k)], 1).reshape(2 * f, k)


def _deinterleave(m):
    r, f2 = m.shape
    v = m.reshape(r, f2 // 256, 2, 128)
    return v[:, :, 0].reshape(r, f2 // 2), v[:, :, 1].reshape(r, f2 // 2)


@pytest.mark.parametrize("f,pair", [(256, True), (384, True), (384, False)])
def test_swiglu_fwd1_epilogue(f, pair):
    """fwd1 of SwiGLU experts: C = bf16([a1|a3]) (block-interleaved), C2 = bf16(silu(a1)·a3)."""
    ops = _ops()
    dev = "cuda"
    torch.manual_seed(5)
    K = 256
    m_tiles = [2, 4, 2]
    G = len(m_tiles)
    R = sum(m_tiles) * 128
    A = torch.randn(R, K, device=dev).bfloat16()
    W1 = (torch.randn(G, f, K, device=dev) / K ** 0.5).bfloat16()
    W3 = (torch.randn(G, f, K, device=dev) / K ** 0.5).bfloat16()
    B = torch.cat([_interleave(W1[g], W3[g]) for g in range(G)])  # [G*2f, K]
    C = torch.zeros(R, 2 * f, device=dev, dtype=torch.bfloat16)
    H = torch.zeros(R, f, device=dev, dtype=torch.bfloat16)
    rows, r0 = [], 0
    for g, mt in enumerate(m_tiles):
        rows.append((mt, r0, 0, g * 2 * f, 0, K // 64, r0 * 2 * f))
        r0 += mt * 128
    gd, ng, total = _groups(ops, rows, 2 * f // 256, dev)
    ops.grouped_gemm(A, False, B, False, gd, ng, 2 * f // 256, total, C, 2 * f,
                     epilogue=ops.EPI_SWIGLU, c2=H, cta_pair=pair)
    torch.cuda.synchronize()
    r0 = 0
    for g, mt in enumerate(m_tiles):
        sl = slice(r0, r0 + mt * 128)
        a1 = A[sl].float() @ W1[g].float().T
        a3 = A[sl].float() @ W3[g].float().T
        c1, c3 = _deinterleave(C[sl])
        _close(c1, a1)
        _close(c3, a3)
        _close(H[sl], torch.nn.functional.silu(a1) * a3)
        r0 += mt * 128


@pytest.mark.parametrize("f,bn128", [(256, False), (512, False), (384, True), (512, True)])
def test_swiglu_dgrad2_epilogue(f, bn128):
    """dgrad2 of SwiGLU experts: acc = dH = dY·W2; with the saved [a1|a3]:
    C = bf16([dH·a3·silu'(a1) | dH·silu(a1)]) (block-interleaved)."""
    ops = _ops()
    dev = "cuda"
    torch.manual_seed(6)
    d = 256
    m_tiles = [2, 2]
    G = len(m_tiles)
    R = sum(m_tiles) * 128
    dY = torch.randn(R, d, device=dev).bfloat16()
    W2 = (torch.randn(G * d, f, device=dev) / f ** 0.5).bfloat16()  # [K=d][N=f] per group
    aux = torch.randn(R, 2 * f, device=dev).bfloat16()
    C = torch.zeros(R, 2 * f, device=dev, dtype=torch.bfloat16)
    bn = 128 if bn128 else 256
    rows, r0 = [], 0
    for g, mt in enumerate(m_tiles):
        rows.append((mt, r0, 0, 0, g * d, d // 64, r0 * 2 * f))
        r0 += mt * 128
    gd, ng, total = _groups(ops, rows, f // bn, dev)
    ops.grouped_gemm(dY, False, W2, True, gd, ng, f // bn, total, C, 2 * f,
                     epilogue=ops.EPI_DSWIGLU, aux=aux, cta_pair=True, bn128=bn128)
    torch.cuda.synchronize()
    r0 = 0
    for g, mt in enumerate(m_tiles):
        sl = slice(r0, r0 + mt * 128)
        dh = dY[sl].float() @ W2[g * d:(g + 1) * d].float()
        a1, a3 = (t.float() for t in _deinterleave(aux[sl]))
        s = torch.sigmoid(a1)
        d1, d3 = _deinterleave(C[sl])
        _close(d1, dh * a3 * s * (1 + a1 * (1 - s)))
        _close(d3, dh * a1 * s)
        r0 += mt * 128


@pytest.mark.parametrize("epi", ["bf16", "gelu", "dgelu"])
def test_bn128_kmajor(epi):
    """N = 384 (not a multiple of 256): 128-wide N tiles."""
    ops = _ops()
    dev = "cuda"
    torch.manual_seed(7)
    K, N = 256, 384
    m_tiles = [2, 2, 4]
    G = len(m_tiles)
    R = sum(m_tiles) * 128
    A = torch.randn(R, K, device=dev).bfloat16()
    b_mn = epi == "dgelu"
    B = ((torch.randn(G * K, N, device=dev) if b_mn else torch.randn(G * N, K, device=dev))
         / K ** 0.5).bfloat16()
    C = torch.zeros(R, N, device=dev, dtype=torch.bfloat16)
    C2 = torch.zeros_like(C)
    aux = torch.randn(R, N, device=dev).bfloat16()
    rows, r0 = [], 0
    for g, mt in enumerate(m_tiles):
        if b_mn:
            rows.append((mt, r0, 0, 0, g * K, K // 64, r0 * N))
        else:
            rows.append((mt, r0, 0, g * N, 0, K // 64, r0 * N))
        r0 += mt * 128
    gd, ng, total = _groups(ops, rows, N // 128, dev)
    e = {"bf16": ops.EPI_BF16, "gelu": ops.EPI_GELU, "dgelu": ops.EPI_DGELU}[epi]
    ops.grouped_gemm(A, False, B, b_mn, gd, ng, N // 128, total, C, N, epilogue=e, c2=C2,
                     aux=aux, cta_pair=True, bn128=True)
    torch.cuda.synchronize()
    r0 = 0
    for g, mt in enumerate(m_tiles):
        sl = slice(r0, r0 + mt * 128)
        if b_mn:
            acc = A[sl].float() @ B[g * K:(g + 1) * K].float()
        else:
            acc = A[sl].float() @ B[g * N:(g + 1) * N].float().T
        if epi == "bf16":
            _close(C[sl], acc)
        elif epi == "gelu":
            _close(C2[sl], torch.nn.functional.gelu(acc, approximate="tanh"))
        else:
            _close(C[sl], acc * aux[sl].float())
        r0 += mt * 128


def test_bn128_wgrad_fp32():
    """wgrad2-style fp32 output with N = 384 (128-wide N tiles), MN-major A and B."""
    ops = _ops()
    dev = "cuda"
    torch.manual_seed(8)
    M, N = 256, 384
    segs = [256, 0, 512]
    G = len(segs)
    Rt = sum(segs)
    At = torch.randn(Rt, M, device=dev).bfloat16()
    Bt = torch.randn(Rt, N, device=dev).bfloat16()
    C = torch.full((G * M, N), 3.0, device=dev)
    rows, k0 = [], 0
    for g, s_ in enumerate(segs):
        rows.append((M // 128, 0, k0, 0, k0, s_ // 64, g * M * N))
        k0 += s_
    gd, ng, total = _groups(ops, rows, N // 128, dev)
    ops.grouped_gemm(At, True, Bt, True, gd, ng, N // 128, total, C, N, epilogue=ops.EPI_F32,
                     cta_pair=True, bn128=True)
    torch.cuda.synchronize()
    k0 = 0
    for g, s_ in enumerate(segs):
        ref = At[k0:k0 + s_].float().T @ Bt[k0:k0 + s_].float()
        _close(C[g * M:(g + 1) * M], ref, rel=2e-3, abs_=1e-4)
        k0 += s_


@pytest.mark.parametrize("K,N,b_mn,pair", [(4096, 1024, False, True), (4096, 1024, True, True),
                                           (14336, 4096, False, True), (14336, 512, True, False),
                                           (2048, 1408, False, True)])
def test_long_k_against_fp32(K, N, b_mn, pair):
    """The BASELINE contraction lengths: K = d_ff 4096 (cfg2 fwd2 / dgrad1), 14 336 (cfg3),
    2048 (cfg4 d_model) with a ragged N = 1408 — bf16 out within one bf16 ulp of the fp32
    product (|Δ| <= 2^-7·|ref| + 1e-3·max|ref|)."""
    ops = _ops()
    dev = "cuda"
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.manual_seed(K + N)
    m_tiles = [2, 4]
    R = sum(m_tiles) * 128
    G = len(m_tiles)
    A = torch.randn(R, K, device=dev).bfloat16()
    B = ((torch.randn(G * K, N, device=dev) if b_mn else torch.randn(G * N, K, device=dev))
         / K ** 0.5).bfloat16()
    C = torch.zeros(R, N, device=dev, dtype=torch.bfloat16)
    bn = 128 if N % 256 else 256
    rows, r0 = [], 0
    for g, mt in enumerate(m_tiles):
        rows.append((mt, r0, 0, 0 if b_mn else g * N, g * K if b_mn else 0, K // 64, r0 * N))
        r0 += mt * 128
    n_tiles = -(-N // bn)
    gd, ng, total = _groups(ops, rows, n_tiles, dev)
    ops.grouped_gemm(A, False, B, b_mn, gd, ng, n_tiles, total, C, N, cta_pair=pair,
                     bn128=bn == 128)
    torch.cuda.synchronize()
    r0 = 0
    for g, mt in enumerate(m_tiles):
        sl = slice(r0, r0 + mt * 128)
        b = B[g * K:(g + 1) * K].float() if b_mn else B[g * N:(g + 1) * N].float().T
        ref = A[sl].float() @ b
        err = (C[sl].float() - ref).abs()
        bound = 2.0 ** -7 * ref.abs() + 1e-3 * ref.abs().max()
        assert (err <= bound).all(), f"max excess {(err - bound).max().item():.3g}"
        r0 += mt * 128


@pytest.mark.parametrize("segs,pair", [([16384, 4096], True), ([24576], True),
                                       ([11264, 0, 5120], False)])
def test_wgrad_long_token_k(segs, pair):
    """wgrad with the token axis as K at bench scale (cfg2's hottest expert holds ~11k
    rows; 24 576 = a whole rank's worth at N = 1): fp32 out vs the fp32 product,
    accumulation order only (1e-4·max|ref|: both sides sum ~24k fp32 products)."""
    ops = _ops()
    dev = "cuda"
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.manual_seed(sum(segs))
    M, N = 1024, 512
    G = len(segs)
    Rt = sum(segs)
    At = torch.randn(Rt, M, device=dev).bfloat16()
    Bt = torch.randn(Rt, N, device=dev).bfloat16()
    C = torch.full((G * M, N), 9.0, device=dev)
    rows, k0 = [], 0
    for g, s_ in enumerate(segs):
        rows.append((M // 128, 0, k0, 0, k0, s_ // 64, g * M * N))
        k0 += s_
    gd, ng, total = _groups(ops, rows, N // 256, dev)
    ops.grouped_gemm(At, True, Bt, True, gd, ng, N // 256, total, C, N, epilogue=ops.EPI_F32,
                     cta_pair=pair)
    torch.cuda.synchronize()
    k0 = 0
    for g, s_ in enumerate(segs):
        ref = At[k0:k0 + s_].float().T @ Bt[k0:k0 + s_].float()
        _close(C[g * M:(g + 1) * M], ref, rel=1e-4, abs_=0.0 if s_ else 1e-30)
        k0 += s_


@pytest.mark.parametrize("pair", [False, True])
def test_dynamic_tile_scheduler_equals_static_order(pair):
    """Tiles taken from the device counter (default) or in the static snake order: the
    same bits (each tile is computed the same way whoever takes it), and every launch
    leaves the counters zero for the next."""
    ops = _ops()
    dev = "cuda"
    torch.manual_seed(11)
    K, N = 512, 1024
    m_tiles = [2, 6, 0, 4, 2, 8]
    R = sum(m_tiles) * 128
    G = len(m_tiles)
    A = torch.randn(R, K, device=dev).bfloat16()
    B = (torch.randn(G * N, K, device=dev) / K ** 0.5).bfloat16()
    rows, r0 = [], 0
    for g, mt in enumerate(m_tiles):
        rows.append((mt, r0, 0, g * N, 0, K // 64, r0 * N))
        r0 += mt * 128
    gd, ng, total = _groups(ops, rows, N // 256, dev)
    outs = []
    for dynamic in (True, False, True):
        C = torch.zeros(R, N, device=dev, dtype=torch.bfloat16)
        ops.grouped_gemm(A, False, B, False, gd, ng, N // 256, total, C, N, cta_pair=pair,
                         dynamic=dynamic)
        torch.cuda.synchronize()
        outs.append(C)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    assert not ops._SCHED[torch.device(dev).index or 0].any()


@pytest.mark.parametrize("case", ["bf16", "gelu", "dgelu_mnB", "bf16_mnB", "swiglu", "dswiglu"])
def test_multicast_clusters_equal_pairs(case):
    """FSSDP_GEMM_MULTICAST (clusters of two CTA pairs sharing the A tile through TMA
    multicast) computes every tile the same way as the plain pair kernel: bit-identical
    outputs, over groups of different M (incl. empty ones) and an odd number of cluster
    tiles per group row."""
    ops = _ops()
    dev = "cuda"
    torch.manual_seed(13)
    K = 512
    N = 1536 if case in ("bf16", "bf16_mnB") else 1024  # 6 / 4 N tiles
    m_tiles = [2, 6, 0, 4, 2, 10]
    R = sum(m_tiles) * 128
    G = len(m_tiles)
    A = torch.randn(R, K, device=dev).bfloat16()
    b_mn = case in ("dgelu_mnB", "bf16_mnB", "dswiglu")
    if b_mn:  # B [G*K, N]: N contiguous (dgrad-style)
        B = (torch.randn(G * K, N, device=dev) / K ** 0.5).bfloat16()
    else:
        B = (torch.randn(G * N, K, device=dev) / K ** 0.5).bfloat16()
    cw = 2 * N if case == "dswiglu" else N  # dSwiGLU writes [da1 | da3] (2 x the GEMM's N)
    rows, r0 = [], 0
    for g, mt in enumerate(m_tiles):
        if b_mn:
            rows.append((mt, r0, 0, 0, g * K, K // 64, r0 * cw))
        else:
            rows.append((mt, r0, 0, g * N, 0, K // 64, r0 * cw))
        r0 += mt * 128
    gd, ng, total = _groups(ops, rows, N // 256, dev)
    epi = {"bf16": ops.EPI_BF16, "bf16_mnB": ops.EPI_BF16, "gelu": ops.EPI_GELU,
           "dgelu_mnB": ops.EPI_DGELU, "swiglu": ops.EPI_SWIGLU, "dswiglu": ops.EPI_DSWIGLU}[case]
    aux = torch.randn(R, cw, device=dev).bfloat16() if case in ("dgelu_mnB", "dswiglu") else None
    outs = []
    for mc in (False, True, True):
        C = torch.zeros(R, cw, device=dev, dtype=torch.bfloat16)
        C2 = (torch.zeros(R, N // 2 if case == "swiglu" else N, device=dev, dtype=torch.bfloat16)
              if case in ("gelu", "swiglu") else None)
        ops.grouped_gemm(A, False, B, b_mn, gd, ng, N // 256, total, C, cw, epilogue=epi, c2=C2,
                         aux=aux, n_fastest=True, cta_pair=True, multicast=mc)
        torch.cuda.synchronize()
        outs.append((C, C2))
    for C, C2 in outs[1:]:
        assert torch.equal(C, outs[0][0])
        if C2 is not None:
            assert torch.equal(C2, outs[0][1])
    assert outs[0][0].abs().sum() > 0


@pytest.mark.parametrize("case", ["bf16", "gelu", "dgelu_mnB", "bf16_mnB"])
def test_split_tail_equals_full_tiles(case):
    """FSSDP_GEMM_SPLIT_TAIL: the short last round as 256x128 half tiles gives the same bits
    as full tiles (shapes chosen so total pair tiles % pairs is in (0, pairs / 2] on a
    148-SM B200)."""
    from paper_2502_02581_b200 import _native as N

    ops = _ops()
    dev = "cuda"
    torch.manual_seed(17)
    K = 512
    N_ = 2048 if case == "gelu" else 1024
    m_tiles = [6, 8, 0, 4, 6] if case == "gelu" else [10, 14, 0, 16, 10]
    pairs = int(N.LIB.fssdp_num_sms()) // 2
    total_pairs = sum(m_tiles) // 2 * (N_ // 256)
    assert 0 < total_pairs % pairs <= pairs // 2, (total_pairs, pairs)
    R = sum(m_tiles) * 128
    G = len(m_tiles)
    A = torch.randn(R, K, device=dev).bfloat16()
    b_mn = case in ("dgelu_mnB", "bf16_mnB")
    if b_mn:
        B = (torch.randn(G * K, N_, device=dev) / K ** 0.5).bfloat16()
    else:
        B = (torch.randn(G * N_, K, device=dev) / K ** 0.5).bfloat16()
    rows, r0 = [], 0
    for g, mt in enumerate(m_tiles):
        rows.append((mt, r0, 0, 0 if b_mn else g * N_, g * K if b_mn else 0, K // 64, r0 * N_))
        r0 += mt * 128
    gd, ng, total = _groups(ops, rows, N_ // 256, dev)
    epi = {"bf16": ops.EPI_BF16, "bf16_mnB": ops.EPI_BF16, "gelu": ops.EPI_GELU,
           "dgelu_mnB": ops.EPI_DGELU}[case]
    aux = torch.randn(R, N_, device=dev).bfloat16() if case == "dgelu_mnB" else None
    outs = []
    for st in (False, True, True):
        C = torch.zeros(R, N_, device=dev, dtype=torch.bfloat16)
        C2 = torch.zeros(R, N_, device=dev, dtype=torch.bfloat16) if case == "gelu" else None
        ops.grouped_gemm(A, False, B, b_mn, gd, ng, N_ // 256, total, C, N_, epilogue=epi,
                         c2=C2, aux=aux, n_fastest=True, cta_pair=True, split_tail=st)
        torch.cuda.synchronize()
        outs.append((C, C2))
    for C, C2 in outs[1:]:
        assert torch.equal(C, outs[0][0])
        if C2 is not None:
            assert torch.equal(C2, outs[0][1])
    assert outs[0][0].abs().sum() > 0


@pytest.mark.parametrize("case", ["bf16", "bf16_mnB", "gelu", "dgelu_mnB", "dswiglu_mnB",
                                  "swiglu"])
def test_swap_tail_equals_full_tiles(case):
    """FSSDP_GEMM_SWAP_TAIL: a group's last M tile whose real rows end within 192 rows runs
    as D^T = W X^T with N' = rows rounded up to 64.  Every REAL row equals the full-tile
    result bit for bit (padding rows are not computed); rows = 1 .. 300 cover no swap,
    N' = 64 / 128 / 192 and multi-tile groups."""
    ops = _ops()
    dev = "cuda"
    torch.manual_seed(19)
    K = 512
    N_ = 1024
    rows = [1, 63, 64, 65, 130, 192, 193, 256, 300, 0, 450]
    pad = [(r + 255) // 256 * 256 for r in rows]
    R = sum(pad)
    G = len(rows)
    A = torch.zeros(R, K, device=dev).bfloat16()
    r0 = 0
    for r, p in zip(rows, pad):
        A[r0:r0 + r] = torch.randn(r, K, device=dev).bfloat16()
        r0 += p
    b_mn = case in ("dgelu_mnB", "bf16_mnB", "dswiglu_mnB")
    # dSwiGLU: N = d_ff (h space), C and aux = the interleaved [a1 | a3] layout, 2 N wide;
    # SwiGLU: N = 2 d_ff (the interleaved [a1 | a3] weight rows), C the same, C2 = h
    W = 2 * N_ if case in ("dswiglu_mnB", "swiglu") else N_
    NG = W if case == "swiglu" else N_  # the GEMM's N
    if b_mn:
        B = (torch.randn(G * K, NG, device=dev) / K ** 0.5).bfloat16()
    else:
        B = (torch.randn(G * NG, K, device=dev) / K ** 0.5).bfloat16()
    g = np.zeros(G, dtype=ops.GROUP_DTYPE)
    r0 = 0
    for i, (r, p) in enumerate(zip(rows, pad)):
        g["m_tiles"][i], g["a_m"][i], g["k_blocks"][i] = p // 128, r0, K // 64
        g["b_n"][i], g["b_k"][i] = (0, i * K) if b_mn else (i * NG, 0)
        g["c_off"][i], g["rows"][i] = r0 * W, r
        r0 += p
    total = ops.finalize_groups(g, NG // 256)
    gd = torch.from_numpy(g.view(np.uint8).copy()).to(dev)
    epi = {"bf16": ops.EPI_BF16, "bf16_mnB": ops.EPI_BF16, "gelu": ops.EPI_GELU,
           "dgelu_mnB": ops.EPI_DGELU, "dswiglu_mnB": ops.EPI_DSWIGLU,
           "swiglu": ops.EPI_SWIGLU}[case]
    aux = (torch.randn(R, W, device=dev).bfloat16()
           if case in ("dgelu_mnB", "dswiglu_mnB") else None)
    outs = []
    for st in (False, True, True):
        C = torch.full((R, W), 7.0, device=dev, dtype=torch.bfloat16)
        C2 = (torch.full((R, N_), 7.0, device=dev, dtype=torch.bfloat16)
              if case in ("gelu", "swiglu") else None)
        ops.grouped_gemm(A, False, B, b_mn, gd, G, NG // 256, total, C, W, epilogue=epi,
                         c2=C2, aux=aux, n_fastest=True, cta_pair=True, swap_tail=st)
        torch.cuda.synchronize()
        outs.append((C, C2))
    real = torch.zeros(R, dtype=torch.bool, device=dev)
    r0 = 0
    for r, p in zip(rows, pad):
        real[r0:r0 + r] = True
        r0 += p
    for C, C2 in outs[1:]:
        assert torch.equal(C[real], outs[0][0][real])
        if C2 is not None:
            assert torch.equal(C2[real], outs[0][1][real])
    # and against fp32 (the full-tile path is checked elsewhere; guard the indexing here)
    if case == "bf16":
        ref = torch.cat([A[sum(pad[:i]):sum(pad[:i]) + pad[i]].float() @
                         B[i * N_:(i + 1) * N_].float().T for i in range(G)])
        _close(outs[1][0][real], ref[real], rel=1e-2, abs_=1e-2)


@pytest.mark.parametrize("K", [64, 320, 448])
@pytest.mark.parametrize("epi", ["bf16", "dgelu"])
def test_deep_stages_odd_k_blocks(K, epi):
    """dgrad-style GEMMs (K-major A, MN-major B, bf16 / dGeLU epilogue) run 128-deep K
    stages: an odd number of 64-wide K blocks leaves the last stage's second chunk staged
    (here B's rows of the NEXT group, non-zero) but not multiplied."""
    ops = _ops()
    dev = "cuda"
    torch.manual_seed(23)
    N = 512
    m_tiles = [2, 4, 2]
    G = len(m_tiles)
    R = sum(m_tiles) * 128
    A = torch.randn(R, K, device=dev).bfloat16()
    B = (torch.randn(G * K, N, device=dev) / K ** 0.5).bfloat16()
    C = torch.zeros(R, N, device=dev, dtype=torch.bfloat16)
    aux = torch.randn(R, N, device=dev).bfloat16() if epi == "dgelu" else None
    rows, refs, r0 = [], [], 0
    for g, mt in enumerate(m_tiles):
        rows.append((mt, r0, 0, 0, g * K, K // 64, r0 * N))
        refs.append((slice(r0, r0 + mt * 128),
                     A[r0:r0 + mt * 128].float() @ B[g * K:(g + 1) * K].float()))
        r0 += mt * 128
    gd, ng, total = _groups(ops, rows, N // 256, dev)
    ops.grouped_gemm(A, False, B, True, gd, ng, N // 256, total, C, N,
                     epilogue=ops.EPI_DGELU if epi == "dgelu" else ops.EPI_BF16, aux=aux,
                     n_fastest=True, cta_pair=True)
    torch.cuda.synchronize()
    for sl, ref in refs:
        _close(C[sl], ref * aux[sl].float() if epi == "dgelu" else ref)
