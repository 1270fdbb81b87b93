"""A-tile multicast (clusters of two CTA pairs) vs plain CTA pairs on the cfg2 token-side
GEMM shapes (16 groups x 2048 rows, d 1024, f 4096), N-fastest tile order as the layer.

    python scripts/mc_probe.py
"""
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


def timeit(fn, iters=20):
    for _ in range(3):
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
H = torch.randn(R, f, device="cuda").bfloat16()
W2 = (torch.randn(G * d, f, device="cuda") / f ** 0.5).bfloat16()
A = torch.empty(R, f, device="cuda").bfloat16()
Hout = torch.empty(R, f, device="cuda").bfloat16()
Y = torch.empty(R, d, device="cuda").bfloat16()
flop = 2 * R * d * f
gd1 = groups([(Mg // 128, g * Mg, 0, g * f, 0, d // 64, g * Mg * f) for g in range(G)], f // 256)
gd2 = groups([(Mg // 128, g * Mg, 0, g * d, 0, f // 64, g * Mg * d) for g in range(G)], d // 256)
gd3 = groups([(Mg // 128, g * Mg, 0, 0, g * f, f // 64, g * Mg * d) for g in range(G)], d // 256)
gd5 = groups([(Mg // 128, g * Mg, 0, 0, g * d, d // 64, g * Mg * f) for g in range(G)], f // 256)
cases = {
    "fwd1_gelu": lambda mc: ops.grouped_gemm(X, False, W1, False, *gd1[:2], f // 256, gd1[2], A, f,
                                             ops.EPI_GELU, c2=Hout, n_fastest=True,
                                             cta_pair=True, multicast=mc),
    "fwd2": lambda mc: ops.grouped_gemm(H, False, W2, False, *gd2[:2], d // 256, gd2[2], Y, d,
                                        n_fastest=True, cta_pair=True, multicast=mc),
    "dgrad1": lambda mc: ops.grouped_gemm(H, False, W1, True, *gd3[:2], d // 256, gd3[2], Y, d,
                                          n_fastest=True, cta_pair=True, multicast=mc),
    "dgrad2_dgelu": lambda mc: ops.grouped_gemm(Y, False, W2.view(G * d, f), True, *gd5[:2],
                                                f // 256, gd5[2], Hout, f, ops.EPI_DGELU, aux=A,
                                                n_fastest=True, cta_pair=True, multicast=mc),
}
for rep in range(int(os.environ.get("MC_REPS", "2"))):
    for name, fn in cases.items():
        t0 = timeit(lambda: fn(False))
        t1 = timeit(lambda: fn(True))
        print(f"{name:14s} pair {t0 * 1e3:7.1f} us {flop / t0 / 1e9:7.1f} TF/s | multicast "
              f"{t1 * 1e3:7.1f} us {flop / t1 / 1e9:7.1f} TF/s", flush=True)

# wave quantization: fwd2 on the bench's Zipf-skewed, 256-padded segments (544 pair tiles =
# 7.35 waves of 74 pairs) with 256- vs 128-wide N tiles
p = 1.0 / np.arange(1, 17) ** 1.2
rows = [int(round(32768 * x / p.sum())) for x in p]
pad = [(r + 255) // 256 * 256 for r in rows]
offs = np.concatenate([[0], np.cumsum(pad)[:-1]])
Rp = int(sum(pad))
Hp = torch.randn(Rp, f, device="cuda").bfloat16()
Yp = torch.empty(Rp, d, device="cuda").bfloat16()
for bn, st in ((256, False), (256, True), (128, False)):
    gz = groups([(pd // 128, int(o), 0, g * d, 0, f // 64, int(o) * d)
                 for g, (pd, o) in enumerate(zip(pad, offs))], d // bn)
    t = timeit(lambda: ops.grouped_gemm(Hp, False, W2, False, *gz[:2], d // bn, gz[2], Yp, d,
                                        n_fastest=True, cta_pair=True, bn128=bn == 128,
                                        split_tail=st))
    print(f"fwd2 zipf-padded rows {Rp} BN {bn} split_tail {int(st)}: {t * 1e3:7.1f} us "
          f"{2 * sum(rows) * d * f / t / 1e9:7.1f} TF/s (routed)", flush=True)

# fwd1's shape (K = d = 1024, N = f = 4096) with each epilogue: what the GeLU outputs cost
if os.environ.get("EPI_PROBE"):
    for name, epi, c2 in (("bf16 (1 output)", ops.EPI_BF16, None), ("gelu (2 outputs)", ops.EPI_GELU, Hout),
                          ("f32 (1 fp32 output)", ops.EPI_F32, None)):
        Cf = torch.empty(R, f, device="cuda") if epi == ops.EPI_F32 else A
        t = timeit(lambda: ops.grouped_gemm(X, False, W1, False, *gd1[:2], f // 256, gd1[2], Cf, f,
                                            epi, c2=c2, n_fastest=True, cta_pair=True))
        print(f"fwd1 shape, epilogue {name:20s} {t * 1e3:7.1f} us {flop / t / 1e9:7.1f} TF/s",
              flush=True)
    # and fwd2's shape (K = f = 4096, N = d = 1024), bf16
    t = timeit(lambda: ops.grouped_gemm(H, False, W2, False, *gd2[:2], d // 256, gd2[2], Y, d,
                                        n_fastest=True, cta_pair=True))
    print(f"fwd2 shape, epilogue bf16 {t * 1e3:7.1f} us {flop / t / 1e9:7.1f} TF/s", flush=True)
