"""Quick tcgen05 grouped-GEMM throughput probe (CUDA events), cfg2 fwd1/fwd2/dgrad/wgrad shapes.
DYN=1: the dynamic tile scheduler instead of the static snake order."""
import sys, os
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
dW1 = torch.empty(G * f, d, device="cuda")
flop_one = 2 * R * d * f
res = {}
DYN = os.environ.get("DYN", "0") != "0"
_gg = ops.grouped_gemm
ops.grouped_gemm = lambda *a, **k: _gg(*a, **k, dynamic=DYN)
gd = groups([(Mg // 128, g * Mg, 0, g * f, 0, d // 64, g * Mg * f) for g in range(G)], f // 256)
res["fwd1_gelu"] = timeit(lambda: ops.grouped_gemm(X, False, W1, False, *gd[:2], f // 256, gd[2], A, f, ops.EPI_GELU, c2=Hout))
gd2 = groups([(Mg // 128, g * Mg, 0, g * d, 0, f // 64, g * Mg * d) for g in range(G)], d // 256)
res["fwd2"] = timeit(lambda: ops.grouped_gemm(H, False, W2, False, *gd2[:2], d // 256, gd2[2], Y, d))
# dgrad1: dX[R,d] = dA[R,f] . W1[g] ([f][d] stored, MN-major B)
gd3 = groups([(Mg // 128, g * Mg, 0, 0, g * f, f // 64, g * Mg * d) for g in range(G)], d // 256)
res["dgrad1_mnB"] = timeit(lambda: ops.grouped_gemm(H, False, W1, True, *gd3[:2], d // 256, gd3[2], Y, d))
# wgrad1: dW1[g] [f x d] = dA_g^T X_g : A=dA [R][f] MN-major, B = X [R][d] MN-major
gd4 = groups([(f // 128, 0, g * Mg, 0, g * Mg, Mg // 64, g * f * d) for g in range(G)], d // 256)
res["wgrad1_mnA_mnB"] = timeit(lambda: ops.grouped_gemm(H, True, X, True, *gd4[:2], d // 256, gd4[2], dW1, d, ops.EPI_F32))
Xf = X.view(G, Mg, d)
W1v = W1.view(G, f, d)
res["torch_bmm_fwd1"] = timeit(lambda: torch.bmm(Xf, W1v.transpose(1, 2)))
for k, v in res.items():
    print(f"dyn={int(DYN)} {k:20s} {v*1e3:9.1f} us  {flop_one / (v * 1e-3) / 1e12:8.1f} TFLOP/s")

# cfg4-shaped wgrad1 (64 experts x 512 token rows, M = n1 = 2 x 1408, N = d = 2048, fp32 out)
G4, M4, d4, n14 = 64, 512, 2048, 2816
dA4 = torch.randn(G4 * M4, n14, device="cuda").bfloat16()
X4 = torch.randn(G4 * M4, d4, device="cuda").bfloat16()
dW4 = torch.empty(G4 * n14, d4, device="cuda")
gd5 = groups([(n14 // 128, 0, g * M4, 0, g * M4, M4 // 64, g * n14 * d4) for g in range(G4)], d4 // 256)
t4 = timeit(lambda: ops.grouped_gemm(dA4, True, X4, True, *gd5[:2], d4 // 256, gd5[2], dW4, d4,
                                     ops.EPI_F32, cta_pair=False), iters=10)
fl4 = 2 * G4 * M4 * n14 * d4
print(f"dyn={int(DYN)} cfg4_wgrad1_fp32     {t4*1e3:9.1f} us  {fl4 / (t4 * 1e-3) / 1e12:8.1f} TFLOP/s  "
      f"{G4 * n14 * d4 * 4 / (t4 * 1e-3) / 1e9:7.0f} GB/s out")
