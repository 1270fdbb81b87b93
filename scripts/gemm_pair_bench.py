import sys, os
sys.path.insert(0, "/root/repo")
exec(open("/root/repo/scripts/gemm_bench.py").read().split("G, Mg, d, f = 16, 2048, 1024, 4096")[0])
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
flop = 2 * R * d * f
for pair in (False, True):
    res = {}
    gd = groups([(Mg // 128, g * Mg, 0, g * f, 0, d // 64, g * Mg * f) for g in range(G)], f // 256)
    res["fwd1_gelu"] = timeit(lambda: ops.grouped_gemm(X, False, W1, False, *gd[:2], f // 256, gd[2], A, f, ops.EPI_GELU, c2=Hout, cta_pair=pair))
    gd2 = groups([(Mg // 128, g * Mg, 0, g * d, 0, f // 64, g * Mg * d) for g in range(G)], d // 256)
    res["fwd2"] = timeit(lambda: ops.grouped_gemm(H, False, W2, False, *gd2[:2], d // 256, gd2[2], Y, d, n_fastest=True, cta_pair=pair))
    gd3 = groups([(Mg // 128, g * Mg, 0, 0, g * f, f // 64, g * Mg * d) for g in range(G)], d // 256)
    res["dgrad1"] = timeit(lambda: ops.grouped_gemm(H, False, W1, True, *gd3[:2], d // 256, gd3[2], Y, d, n_fastest=True, cta_pair=pair))
    res["dgrad2_dgelu"] = timeit(lambda: ops.grouped_gemm(Y, False, W2.view(G * d, f), True, *groups([(Mg // 128, g * Mg, 0, 0, g * d, d // 64, g * Mg * f) for g in range(G)], f // 256)[:2], f // 256, groups([(Mg // 128, g * Mg, 0, 0, g * d, d // 64, g * Mg * f) for g in range(G)], f // 256)[2], Hout, f, ops.EPI_DGELU, aux=A, cta_pair=pair))
    gd4 = groups([(f // 128, 0, g * Mg, 0, g * Mg, Mg // 64, g * f * d) for g in range(G)], d // 256)
    res["wgrad1"] = timeit(lambda: ops.grouped_gemm(H, True, X, True, *gd4[:2], d // 256, gd4[2], dW1, d, ops.EPI_F32, cta_pair=pair))
    for k, v in res.items():
        print(f"pair={pair} {k:14s} {v*1e3:8.1f} us {flop / (v * 1e-3) / 1e12:8.1f} TFLOP/s")
