"""Weight-gradient GEMM probe (CUDA events): what bounds the short-K fp32-output wgrads of
cfg4 (64 experts, ~512 token rows each).  Same groups timed with the fp32 and the bf16
epilogue, with and without CTA pairs, and at longer K per group.

    python scripts/wgrad_probe.py            # FSSDP_LIB=<variant .so> for experiment builds
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


def timeit(fn, iters=10):
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


def wgrad(G, K, M, N, epi, pair, bn=256):
    """dW[g] [M x N] = A_g^T B_g, A [G*K][M] and B [G*K][N] MN-major (the layer's wgrads)."""
    a = torch.randn(G * K, M, device="cuda").bfloat16()
    b = torch.randn(G * K, N, device="cuda").bfloat16()
    out = torch.empty(G * M, N, device="cuda",
                      dtype=torch.float32 if epi == ops.EPI_F32 else torch.bfloat16)
    nt = (N + bn - 1) // bn
    gd = groups([(M // 128, 0, g * K, 0, g * K, K // 64, g * M * N) for g in range(G)], nt)
    t = timeit(lambda: ops.grouped_gemm(a, True, b, True, *gd[:2], nt, gd[2], out, N, epi,
                                        cta_pair=pair, bn128=bn == 128, dynamic=False))
    fl = 2 * G * K * M * N
    return t, fl / (t * 1e-3) / 1e12, G * M * N * out.element_size() / (t * 1e-3) / 1e9


def wgrad_ragged(Ks, M, N, epi, dynamic):
    """Groups of different token rows (descending, as the layer lists them)."""
    Ks = sorted(Ks, reverse=True)
    a = torch.randn(sum(Ks), M, device="cuda").bfloat16()
    b = torch.randn(sum(Ks), N, device="cuda").bfloat16()
    out = torch.empty(len(Ks) * M, N, device="cuda",
                      dtype=torch.float32 if epi == ops.EPI_F32 else torch.bfloat16)
    nt = N // 256
    offs = np.concatenate([[0], np.cumsum(Ks)[:-1]])
    gd = groups([(M // 128, 0, int(o), 0, int(o), k // 64, g * M * N)
                 for g, (k, o) in enumerate(zip(Ks, offs))], nt)
    t = timeit(lambda: ops.grouped_gemm(a, True, b, True, *gd[:2], nt, gd[2], out, N, epi,
                                        cta_pair=True, dynamic=dynamic))
    return t, 2 * sum(Ks) * M * N / (t * 1e-3) / 1e12


print(f"lib={os.environ.get('FSSDP_LIB', 'default')}")
if os.environ.get("RAGGED"):
    p = 1.0 / np.arange(1, 17) ** 1.2
    Ks = [max(64, int(round(32768 * x / p.sum() / 64)) * 64) for x in p]
    p4 = 1.0 / np.arange(1, 65) ** 1.2
    Ks4 = [max(64, int(round(32768 * x / p4.sum() / 64)) * 64) for x in p4]
    for cfg, M, N_, cases in (("cfg2", 4096, 1024, (("zipf", Ks), ("uniform", [2048] * 16))),
                              ("cfg4", 2816, 2048, (("zipf", Ks4), ("uniform", [512] * 64)))):
        for name, ks in cases:
            for dyn in (False, True):
                t, tf = wgrad_ragged(ks, M, N_, ops.EPI_BF16, dyn)
                print(f"{cfg} wgrad1 {name:8s} dyn={int(dyn)} {t * 1e3:8.1f} us {tf:7.1f} "
                      f"TFLOP/s rows {sum(ks)} max K {max(ks)}", flush=True)
    sys.exit(0)
for name, G, K, M, N in (("cfg4 wgrad1", 64, 512, 2816, 2048), ("cfg4 wgrad2", 64, 512, 2048, 1408),
                         ("cfg4 wgrad1 K2048", 16, 2048, 2816, 2048),
                         ("cfg2 wgrad1", 16, 2048, 4096, 1024)):
    for epi, en in ((ops.EPI_F32, "f32"), (ops.EPI_BF16, "bf16")):
        for pair in (True, False):
            if epi == ops.EPI_BF16 and not pair:
                continue
            t, tf, gbs = wgrad(G, K, M, N, epi, pair)
            print(f"{name:18s} {en:4s} pair={int(pair)} {t * 1e3:8.1f} us {tf:7.1f} TFLOP/s "
                  f"{gbs:6.0f} GB/s out", flush=True)
