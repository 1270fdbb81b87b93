"""Epilogue-cost probe: the K = d_model GEMM shapes of cfg2 (fwd1 / dgrad2: 16 groups x
2048 rows, N = d_ff = 4096, K = 1024) with each epilogue, against the K = d_ff shape (fwd2).
Run once per experiment build (FSSDP_LIB=<variant .so>) to split a tile's time between the
mainloop and the epilogue's TMEM reads, math, shared-memory staging and TMA stores."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2502_02581_b200 import ops


def groups(rows, n_tiles):
    g = np.zeros(len(rows), dtype=ops.GROUP_DTYPE)
    for i, r in enumerate(rows):
        (g["m_tiles"][i], g["a_m"][i], g["a_k"][i], g["b_n"][i], g["b_k"][i], g["k_blocks"][i],
         g["c_off"][i]) = r
    total = ops.finalize_groups(g, n_tiles)
    return torch.from_numpy(g.view(np.uint8).copy()).cuda(), len(rows), total


def timeit(fn, iters=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


G, Mg, d, f = 16, 2048, 1024, 4096
R = G * Mg
X = torch.randn(R, d, device="cuda").bfloat16()
W1 = (torch.randn(G * f, d, device="cuda") / d ** 0.5).bfloat16()
W2t = (torch.randn(G * d, f, device="cuda") / f ** 0.5).bfloat16()  # [d][f] per group
Hh = torch.randn(R, f, device="cuda").bfloat16()
A = torch.empty(R, f, device="cuda").bfloat16()
A2 = torch.empty(R, f, device="cuda").bfloat16()
Y = torch.empty(R, d, device="cuda").bfloat16()
flop = 2 * R * d * f
tag = os.environ.get("TAG", os.path.basename(os.environ.get("FSSDP_LIB", "base")))
nf = os.environ.get("NF", "1") != "0"
g1 = groups([(Mg // 128, g * Mg, 0, g * f, 0, d // 64, g * Mg * f) for g in range(G)], f // 256)
g2 = groups([(Mg // 128, g * Mg, 0, g * d, 0, f // 64, g * Mg * d) for g in range(G)], d // 256)
# dgrad2: dA[R,f] = dY[R,d] . W2[g] with W2 stored [d][f] (MN-major B), aux = gelu'
g3 = groups([(Mg // 128, g * Mg, 0, 0, g * d, d // 64, g * Mg * f) for g in range(G)], f // 256)
kw = dict(cta_pair=True, n_fastest=nf)
res = {
    "fwd1_gelu": timeit(lambda: ops.grouped_gemm(X, False, W1, False, *g1[:2], f // 256, g1[2], A, f,
                                                 ops.EPI_GELU, c2=A2, **kw)),
    "fwd1_bf16": timeit(lambda: ops.grouped_gemm(X, False, W1, False, *g1[:2], f // 256, g1[2], A, f,
                                                 ops.EPI_BF16, **kw)),
    "dgrad2_dgelu": timeit(lambda: ops.grouped_gemm(X, False, W2t, True, *g3[:2], f // 256, g3[2], A, f,
                                                    ops.EPI_DGELU, aux=Hh, **kw)),
    "dgrad2_bf16": timeit(lambda: ops.grouped_gemm(X, False, W2t, True, *g3[:2], f // 256, g3[2], A, f,
                                                   ops.EPI_BF16, **kw)),
    "fwd2": timeit(lambda: ops.grouped_gemm(Hh, False, W2t.view(G * d, f), False, *g2[:2], d // 256,
                                            g2[2], Y, d, **kw)),
}
for k, v in res.items():
    print(f"{tag:12s} {k:14s} {v * 1e3:8.1f} us {flop / (v * 1e-3) / 1e12:8.1f} TFLOP/s")
