"""Plain-PyTorch fp32 references of the FSSDP tensor path on the GPU — TEST INFRASTRUCTURE.

oracle/tensor_oracle.py restates the layer in numpy; at the BASELINE.json shapes (cfg2:
32 768 routed rows x d 1024 x f 4096; cfg3: d 4096 x f 14336) numpy takes minutes, so
the full-shape parity tests use these torch fp32 restatements of the SAME math on the
GPU (fp32 matmuls with TF32 off; elementwise ops in fp32).  Two flavours:

* `layer(plain=False)` keeps the device's bf16 rounding points (the tensor oracle's contract:
  H, Y, dY_e, dA, dX_e rounded to bf16, fp32 accumulation everywhere) — differences
  against the kernels come only from accumulation order, tanh.approx / __expf, and the
  bf16 roundings they flip;
* `layer(plain=True)` drops every intermediate rounding (fp32 end to end from the same bf16
  weights and inputs) — the distance to it is the real bf16 drift of the product path.

Stage references (`stage_*`) take the device's own saved intermediates as inputs, so each
kernel is checked against one fp32 contraction and its epilogue, with no error carried in
from earlier stages.
"""

from __future__ import annotations

import torch

K0, K1 = 0.7978845608028654, 0.044715


def bf16(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.bfloat16).float()


def gelu(a):
    return 0.5 * a * (1.0 + torch.tanh(K0 * (a + K1 * a * a * a)))


def gelu_grad(a):
    t = torch.tanh(K0 * (a + K1 * a * a * a))
    return 0.5 * (1.0 + t) + 0.5 * a * (1.0 - t * t) * K0 * (1.0 + 3.0 * K1 * a * a)


def interleave(m1: torch.Tensor, m3: torch.Tensor) -> torch.Tensor:
    """Columns [a1 | a3] -> the kernels' 128-column block interleave (FSSDP_EPI_SWIGLU)."""
    r, f = m1.shape
    return torch.stack([m1.view(r, f // 128, 128), m3.view(r, f // 128, 128)], 2).reshape(r, 2 * f)


def deinterleave(m: torch.Tensor):
    r, f2 = m.shape
    v = m.reshape(r, f2 // 256, 2, 128)
    return v[:, :, 0].reshape(r, f2 // 2), v[:, :, 1].reshape(r, f2 // 2)


# ---------------------------------------------------------------- stage references
def stage_fwd1(xr, w13, swiglu):
    """-> (saved, h): GeLU saved = bf16(gelu'(A)), SwiGLU saved = bf16([a1|a3] interleaved);
    h = bf16(act(A)).  xr [n, d] (bf16 values), w13 [n1, d] (interleaved for SwiGLU)."""
    a = xr.float() @ w13.float().T
    if not swiglu:
        return bf16(gelu_grad(a)), bf16(gelu(a))
    a1, a3 = deinterleave(a)
    return bf16(a), bf16(torch.nn.functional.silu(a1) * a3)


def stage_dgrad2(dyr, w2, saved, swiglu):
    """dA from dY_e [n, d], W2 [d, f] and the saved fwd1 values (device's own)."""
    dh = dyr.float() @ w2.float()
    if not swiglu:
        return bf16(dh * saved.float())
    a1, a3 = deinterleave(saved.float())
    s = torch.sigmoid(a1)
    return interleave(bf16(dh * a3 * s * (1.0 + a1 * (1.0 - s))), bf16(dh * a1 * s))


# ---------------------------------------------------------------- whole layer
def layer(x, idx, w, wg, experts, dy, *, plain=False):
    """One rank's FSSDP layer fwd+bwd on its tokens (placement-independent math).

    x, dy [T, d] bf16 tensors; idx [T, k] int, w [T, k] fp32 (the device's routing);
    wg [E, d] fp32; experts {e: (W1 [f, d], W2 [d, f])} or {e: (W1, W3, W2)} bf16.
    plain=False: the device's bf16 rounding points; plain=True: fp32 throughout.
    Returns dict(y, dx, dW {e: tuple of fp32 grads in expert-tuple order}, dWg)."""
    rnd = (lambda t: t) if plain else bf16
    T, k = idx.shape
    d = x.shape[1]
    xf = x.float()
    dyf = dy.float()
    idx = idx.long()
    Y = torch.zeros(T, k, d, device=x.device)
    saved = {}
    for e, mats in experts.items():
        t_i, j_i = torch.nonzero(idx == e, as_tuple=True)
        if t_i.numel() == 0:
            continue
        xe = xf[t_i]
        if len(mats) == 3:
            a1 = xe @ mats[0].float().T
            a3 = xe @ mats[1].float().T
            h = rnd(torch.nn.functional.silu(a1) * a3)
            saved[e] = (t_i, j_i, (rnd(a1), rnd(a3)), h)
        else:
            a = xe @ mats[0].float().T
            h = rnd(gelu(a))
            saved[e] = (t_i, j_i, a, h)
        Y[t_i, j_i] = rnd(h @ mats[-1].float().T)
    acc = torch.zeros(T, d, device=x.device)
    for j in range(k):
        acc = acc + w[:, j:j + 1] * Y[:, j]
    y = rnd(acc)
    g = torch.einsum("td,tkd->tk", dyf, Y)
    sg = (w * g).sum(1, keepdim=True)
    dlogit = w * (g - sg)
    dXs = torch.zeros(T, k, d, device=x.device)
    dW = {}
    for e, mats in experts.items():
        if e not in saved:
            dW[e] = tuple(torch.zeros_like(m, dtype=torch.float32) for m in mats)
            continue
        t_i, j_i, sv, h = saved[e]
        dye = rnd(w[t_i, j_i][:, None] * dyf[t_i])
        dh = dye @ mats[-1].float()
        xe = xf[t_i]
        if len(mats) == 3:
            a1, a3 = sv
            s = torch.sigmoid(a1)
            da1 = rnd(dh * a3 * s * (1.0 + a1 * (1.0 - s)))
            da3 = rnd(dh * a1 * s)
            dXs[t_i, j_i] = rnd(da1 @ mats[0].float() + da3 @ mats[1].float())
            dW[e] = (da1.T @ xe, da3.T @ xe, dye.T @ h)
        else:
            da = rnd(dh * rnd(gelu_grad(sv)))  # the saved gelu'(A) is bf16 on the device
            dXs[t_i, j_i] = rnd(da @ mats[0].float())
            dW[e] = (da.T @ xe, dye.T @ h)
    dx = dXs.sum(1) + torch.einsum("tk,tkd->td", dlogit, wg[idx])
    dwg = torch.zeros_like(wg)
    for j in range(k):
        dwg.index_add_(0, idx[:, j], dlogit[:, j:j + 1] * xf)
    return dict(y=y, dx=rnd(dx), dW=dW, dWg=dwg)


def rel_err(out: torch.Tensor, ref: torch.Tensor) -> float:
    """max |out - ref| / max |ref| (0 for an all-zero pair)."""
    out, ref = out.double(), ref.double()
    den = ref.abs().max().item()
    num = (out - ref).abs().max().item()
    return num / den if den > 0 else num


def grad_excess(gm: torch.Tensor, gs: torch.Tensor) -> float:
    """A sharded run's SpRS-reduced weight gradient gm against the single-rank gs: the
    largest excess over the bound (<= 0 passes).  fp32 gradients: 1e-4·max|gs| (summation
    order only).  bf16 gradients: each holder's partial and the reduced sum are rounded to
    bf16 (one ulp = 2^-7 relative at worst), so 2 ulps of the element plus 2^-8·max|gs| for
    partials that cancel."""
    bf = gs.dtype == torch.bfloat16
    gm, gs = gm.double(), gs.double()
    peak = gs.abs().max().item()
    if bf:
        bound = 2.0 ** -6 * gs.abs() + 2.0 ** -8 * peak
    else:
        bound = torch.full_like(gs, 1e-4 * peak + 1e-6)
    return ((gm - gs).abs() - bound).max().item()
