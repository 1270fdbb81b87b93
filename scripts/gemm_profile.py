"""Where each GEMM's time goes, from the diagnostic build's per-CTA role-wait counters
(python paper_2502_02581_b200/build.py --gemm-profile; diagnostics only, never the bench).

    python scripts/gemm_profile.py

Per GEMM of the cfg2 shapes (16 uniform groups of 2048 rows): fraction of the MMA issuer's
loop spent waiting for operands (full) and for a free accumulator (tempty), of the
producer's loop waiting for a free smem stage, of the epilogue's loop waiting for an
accumulator."""
import ctypes as C
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
os.environ["FSSDP_LIB"] = str(ROOT / "build" / "libfssdp_gemm_profile.so")
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_02581_b200 import _native as N  # noqa: E402
from paper_2502_02581_b200 import ops  # noqa: E402

N.LIB.fssdp_gemm_profile_read.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros((1024, 8), dtype=np.uint64)


def groups(rows, n_tiles):
    g = np.zeros(len(rows), dtype=ops.GROUP_DTYPE)
    for i, r in enumerate(rows):
        (g["m_tiles"][i], g["a_m"][i], g["a_k"][i], g["b_n"][i], g["b_k"][i], g["k_blocks"][i],
         g["c_off"][i]) = r
    total = ops.finalize_groups(g, n_tiles)
    return torch.from_numpy(g.view(np.uint8).copy()).cuda(), len(rows), total


def profile(name, fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    N.LIB.fssdp_gemm_profile_read(buf.ctypes.data, 1)
    fn()
    torch.cuda.synchronize()
    N.LIB.fssdp_gemm_profile_read(buf.ctypes.data, 1)
    live = buf[buf[:, 4] > 0]  # MMA issuers (leader CTAs)
    prod = buf[buf[:, 0] > 0]
    epi = buf[buf[:, 6] > 0]
    f = lambda a, b: float(a.sum()) / max(1.0, float(b.sum()))  # noqa: E731
    print(f"{name:14s} mma: full-wait {f(live[:, 2], live[:, 4]):5.2f} tempty-wait "
          f"{f(live[:, 3], live[:, 4]):5.2f} | producer empty-wait {f(prod[:, 1], prod[:, 0]):5.2f}"
          f" | epilogue tfull-wait {f(epi[:, 5], epi[:, 6]):5.2f} | tiles/leader "
          f"{live[:, 7].mean():.1f} (min {live[:, 7].min()}, max {live[:, 7].max()}) "
          f"| mma loop kcycles mean {live[:, 4].mean() / 1e3:.0f} max {live[:, 4].max() / 1e3:.0f}")


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
dW2 = torch.empty(G * d, f, device="cuda")
gd = groups([(Mg // 128, g * Mg, 0, g * f, 0, d // 64, g * Mg * f) for g in range(G)], f // 256)
profile("fwd1_gelu", lambda: ops.grouped_gemm(X, False, W1, False, *gd[:2], f // 256, gd[2], A, f,
                                              ops.EPI_GELU, c2=Hout, cta_pair=True))
gd2 = groups([(Mg // 128, g * Mg, 0, g * d, 0, f // 64, g * Mg * d) for g in range(G)], d // 256)
profile("fwd2", lambda: ops.grouped_gemm(H, False, W2, False, *gd2[:2], d // 256, gd2[2], Y, d,
                                         n_fastest=True, cta_pair=True))
gd3 = groups([(Mg // 128, g * Mg, 0, 0, g * f, f // 64, g * Mg * d) for g in range(G)], d // 256)
profile("dgrad1", lambda: ops.grouped_gemm(H, False, W1, True, *gd3[:2], d // 256, gd3[2], Y, d,
                                           n_fastest=True, cta_pair=True))
gd5 = groups([(Mg // 128, g * Mg, 0, 0, g * d, d // 64, g * Mg * f) for g in range(G)], f // 256)
profile("dgrad2_dgelu", lambda: ops.grouped_gemm(Y, False, W2.view(G * d, f), True, *gd5[:2],
                                                 f // 256, gd5[2], Hout, f, ops.EPI_DGELU, aux=A,
                                                 cta_pair=True))
gd4 = groups([(f // 128, 0, g * Mg, 0, g * Mg, Mg // 64, g * f * d) for g in range(G)], d // 256)
profile("wgrad1", lambda: ops.grouped_gemm(H, True, X, True, *gd4[:2], d // 256, gd4[2], dW1, d,
                                           ops.EPI_F32, cta_pair=True))
gd6 = groups([(d // 128, 0, g * Mg, 0, g * Mg, Mg // 64, g * f * d) for g in range(G)], f // 256)
profile("wgrad2", lambda: ops.grouped_gemm(Y, True, H, True, *gd6[:2], f // 256, gd6[2], dW2, f,
                                           ops.EPI_F32, cta_pair=True))

# cfg4-shaped wgrad1: 64 groups of 512 token rows (short K: 8 k-blocks per tile)
G4, M4, d4, n14 = 64, 512, 2048, 2816
dA4 = torch.randn(G4 * M4, n14, device="cuda").bfloat16()
X4 = torch.randn(G4 * M4, d4, device="cuda").bfloat16()
dW4 = torch.empty(G4 * n14, d4, device="cuda")
dW4h = torch.empty(G4 * n14, d4, device="cuda").bfloat16()
gd7 = groups([(n14 // 128, 0, g * M4, 0, g * M4, M4 // 64, g * n14 * d4) for g in range(G4)],
             d4 // 256)
profile("cfg4_wgrad1", lambda: ops.grouped_gemm(dA4, True, X4, True, *gd7[:2], d4 // 256, gd7[2],
                                                dW4, d4, ops.EPI_F32, cta_pair=True))
profile("cfg4_wgrad1_bf", lambda: ops.grouped_gemm(dA4, True, X4, True, *gd7[:2], d4 // 256,
                                                   gd7[2], dW4h, d4, ops.EPI_BF16, cta_pair=True))
