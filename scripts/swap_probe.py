"""Swapped-tail probe at cfg4 shapes: 64 experts with Zipf(1.2) row counts (32768 routed
rows), d_model 2048, d_ff 1408 SwiGLU — fwd1 (SwiGLU epilogue) and dgrad2 (dSwiGLU),
swap_tail off / on, CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2502_02581_b200 import ops


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
    return s.elapsed_time(e) / iters * 1e3


G, d, f = 64, 2048, 1408
p = 1.0 / np.arange(1, G + 1) ** 1.2
rows = np.floor(p / p.sum() * 32768).astype(int)
rows[0] += 32768 - rows.sum()
pad = (rows + 255) // 256 * 256
R = int(pad.sum())
dev = "cuda"
X = torch.randn(R, d, device=dev).bfloat16()
W13 = (torch.randn(G * 2 * f, d, device=dev) / d ** 0.5).bfloat16()
W2 = (torch.randn(G * d, f, device=dev) / f ** 0.5).bfloat16()  # [d][f]: MN-major B
C = torch.empty(R, 2 * f, device=dev).bfloat16()
H = torch.empty(R, f, device=dev).bfloat16()
aux = torch.randn(R, 2 * f, device=dev).bfloat16()


def groups(n_out, b_mn, c_w):
    g = np.zeros(G, dtype=ops.GROUP_DTYPE)
    r0 = 0
    for i in range(G):
        g["m_tiles"][i], g["a_m"][i], g["k_blocks"][i] = pad[i] // 128, r0, d // 64
        g["b_n"][i], g["b_k"][i] = (0, i * d) if b_mn else (i * n_out, 0)
        g["c_off"][i], g["rows"][i] = r0 * c_w, rows[i]
        r0 += pad[i]
    total = ops.finalize_groups(g, -(-n_out // 256))
    return torch.from_numpy(g.view(np.uint8).copy()).to(dev), total


g1, t1 = groups(2 * f, False, 2 * f)
g2, t2 = groups(f, True, 2 * f)
fl = 2 * 32768 * d * 2 * f
for st in (False, True, False, True):
    a = timeit(lambda: ops.grouped_gemm(X, False, W13, False, g1, G, 2 * f // 256, t1, C, 2 * f,
                                        ops.EPI_SWIGLU, c2=H, n_fastest=True, cta_pair=True,
                                        swap_tail=st))
    b = timeit(lambda: ops.grouped_gemm(X, False, W2, True, g2, G, -(-f // 256), t2, C, 2 * f,
                                        ops.EPI_DSWIGLU, aux=aux, n_fastest=True, cta_pair=True,
                                        swap_tail=st))
    print(f"swap={int(st)} fwd1_swiglu {a:7.1f} us {fl / a / 1e6:7.1f} TF/s | "
          f"dgrad2_dswiglu {b:7.1f} us {fl / b / 1e6:7.1f} TF/s  (padded rows {R}, routed 32768)")
