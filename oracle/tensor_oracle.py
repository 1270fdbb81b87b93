"""numpy restatement of the FSSDP tensor path — TEST INFRASTRUCTURE (see oracle/__init__.py).

The reference moesim package models tensors as byte counts only, so this
restates the paper's semantics; parity here is UNPINNED by reference tests:

* gate: logits = x · Wgᵀ, top-k with ties to the lower expert id, GShard-style
  renormalised softmax over the selected logits;
  no capacity factor / token dropping.
* dispatch: token-slot order (t, j) ascending fills the destinations of a
  (source, expert) cell in ascending device order with the build_dispatch counts
  route[s, e, d] (dispatch.py:49-97 gives the counts; the per-token order is ours).
* expert FFN: A = X·W1ᵀ (fp32), H = bf16(gelu_tanh(A)), Y = H·W2ᵀ; the
  backward uses the saved G' = bf16(gelu_tanh'(A)): dA = bf16((dY·W2)·G').  SwiGLU experts
  (configs 3-4): H = bf16(silu(A1)·A3) from fp32 A1 = X·W1ᵀ, A3 = X·W3ᵀ; the backward uses
  the saved bf16 A1, A3: dA1 = bf16(dH·A3·silu'(A1)), dA3 = bf16(dH·silu(A1)).
* combine: y_t = Σ_j w_tj · Y_tj in fp32, j ascending, then bf16.
* SpAG: replica = owner copy; SpRS: owner = Σ replicas in ascending device order, fp32
  (PAPER.md:370-386).

Functions that the kernels reproduce bit-for-bit use explicit float32 operations in
the kernels' order (selection, ranks, positions, combine, SpAG, SpRS).
"""

from __future__ import annotations

import numpy as np

GATE_TILE = 64


# ------------------------------------------------------------------ bf16 helpers
def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> nearest bf16 (round half to even), returned as float32."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32).copy()
    nan = np.isnan(a)
    out[nan] = np.nan
    return out


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


# ------------------------------------------------------------------ gate
def gate_logits(x: np.ndarray, wg: np.ndarray) -> np.ndarray:
    """fp32 logits [T, E] (float64 accumulation; compared within tolerance)."""
    return (x.astype(np.float64) @ wg.astype(np.float64).T).astype(np.float32)


def topk_select(logits: np.ndarray, k: int):
    """Top-k selection, weights, tile-relative slot ranks and per-tile histograms.

    Mirrors K1's tail exactly: selection by repeated scan with strict '>' (ties ->
    lower expert id); e_j = exp(l_j - l_top1) in float32; s accumulated j ascending;
    w_j = e_j / s.  Ranks count earlier slots (t, j) of the same expert in the tile."""
    lg = np.asarray(logits, dtype=np.float32)
    T, E = lg.shape
    idx = np.empty((T, k), dtype=np.int32)
    for t in range(T):
        row = lg[t]
        taken = np.zeros(E, dtype=bool)
        for j in range(k):
            best, bi = np.float32(0), -1
            for e in range(E):
                if taken[e]:
                    continue
                if bi < 0 or row[e] > best:
                    best, bi = row[e], e
            taken[bi] = True
            idx[t, j] = bi
    sel = np.take_along_axis(lg, idx.astype(np.int64), axis=1)
    m = sel[:, :1]
    ex = np.exp((sel - m).astype(np.float32)).astype(np.float32)
    s = np.zeros(T, dtype=np.float32)
    for j in range(k):
        s = (s + ex[:, j]).astype(np.float32)
    w = (ex / s[:, None]).astype(np.float32)
    tiles = (T + GATE_TILE - 1) // GATE_TILE
    rank = np.empty((T, k), dtype=np.int32)
    tile_counts = np.zeros((max(tiles, 1), E), dtype=np.int32)
    for tile in range(tiles):
        cnt = np.zeros(E, dtype=np.int64)
        for t in range(tile * GATE_TILE, min(T, (tile + 1) * GATE_TILE)):
            for j in range(k):
                e = idx[t, j]
                rank[t, j] = cnt[e]
                cnt[e] += 1
        tile_counts[tile] = cnt
    return idx, w, rank, tile_counts


def expert_counts(idx: np.ndarray, E: int) -> np.ndarray:
    return np.bincount(idx.reshape(-1), minlength=E).astype(np.int64)


# ------------------------------------------------------------------ activation
def gelu_tanh(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.float32)
    k0, k1 = np.float32(0.7978845608028654), np.float32(0.044715)
    return np.float32(0.5) * x * (np.float32(1.0) + np.tanh(k0 * (x + k1 * x * x * x)))


def gelu_tanh_grad(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.float32)
    k0, k1 = np.float32(0.7978845608028654), np.float32(0.044715)
    t = np.tanh(k0 * (x + k1 * x * x * x))
    return (np.float32(0.5) * (np.float32(1.0) + t)
            + np.float32(0.5) * x * (np.float32(1.0) - t * t) * k0 * (np.float32(1.0) + np.float32(3.0) * k1 * x * x))


# ------------------------------------------------------------------ dispatch / combine
def slot_positions(idx: np.ndarray, route: np.ndarray, src: int, recv_base: np.ndarray):
    """Destination device and receive row of every token-slot of source `src`.

    route[s, e, d] (build_dispatch counts); recv_base[e, d] = first receive row of
    (src, e) on device d.  Slots of one expert are taken in (t, j) order and fill
    destinations in ascending device order."""
    T, k = idx.shape
    D = route.shape[2]
    dest = np.empty((T, k), dtype=np.int32)
    pos = np.empty((T, k), dtype=np.int32)
    seen = np.zeros(route.shape[1], dtype=np.int64)
    for t in range(T):
        for j in range(k):
            e = idx[t, j]
            r = seen[e]
            seen[e] += 1
            cum = np.concatenate([[0], np.cumsum(route[src, e])])
            d = 0
            while d + 1 < D and cum[d + 1] <= r:
                d += 1
            dest[t, j] = d
            pos[t, j] = recv_base[e, d] + (r - cum[d])
    return dest, pos


def combine(rows: np.ndarray, w: np.ndarray) -> np.ndarray:
    """rows [T, k, d] (bf16 values as float32), w [T, k] -> bf16(Σ_j w_j·rows_j), exact
    float32 order of the kernel (acc += w*y, j ascending, no FMA)."""
    T, k, d = rows.shape
    acc = np.zeros((T, d), dtype=np.float32)
    for j in range(k):
        prod = (w[:, j:j + 1].astype(np.float32) * rows[:, j, :].astype(np.float32)).astype(np.float32)
        acc = (acc + prod).astype(np.float32)
    return bf16_round(acc)


def silu(a):
    return (a / (1.0 + np.exp(-a.astype(np.float64)))).astype(np.float32)


def moe_layer_fwd_bwd(x, idx, w, wg, experts, dy):
    """Whole-layer restatement for one rank's tokens (placement-independent math).

    x [T, d] bf16-valued float32; idx/w [T, k] (the device's own routing, pinned
    bit-exactly by the gate tests); wg [E, d]; experts {e: (W1 [f, d], W2 [d, f])} (GeLU,
    PAPER.md:645) or {e: (W1, W3 [f, d], W2)} (SwiGLU: h = silu(x W1ᵀ) ⊙ (x W3ᵀ), the
    Mixtral / DeepSeek expert of configs 3-4), bf16-valued float32; dy [T, d].
    Rounding points mirror the device: fwd keeps fp32 pre-activations for h, saves bf16
    (gelu'(a) | a1, a3) for backward; dgrad2 multiplies the fp32 dH by the saved values.
    Returns dict(y, dx, g (slot <dy, Y>), dlogit, dW1 {e}, dW2 {e}, [dW3 {e}], dWg)."""
    T, k = idx.shape
    d = x.shape[1]
    swiglu = len(next(iter(experts.values()))) == 3
    Y = np.zeros((T, k, d), dtype=np.float32)
    A = {}
    H = {}
    for e, mats in experts.items():
        rows = np.argwhere(idx == e)
        if len(rows) == 0:
            continue
        xe = x[rows[:, 0]].astype(np.float32)
        W2 = mats[-1]
        if swiglu:
            a1 = (xe @ mats[0].T).astype(np.float32)
            a3 = (xe @ mats[1].T).astype(np.float32)
            h = bf16_round((silu(a1) * a3).astype(np.float32))
            A[e] = (rows, (bf16_round(a1), bf16_round(a3)))  # saved bf16 pre-activations
        else:
            a = (xe @ mats[0].T).astype(np.float32)  # fp32 pre-activation (never stored)
            h = bf16_round(gelu_tanh(a).astype(np.float32))
            A[e] = (rows, a)
        Y[rows[:, 0], rows[:, 1]] = bf16_round((h @ W2.T).astype(np.float32))
        H[e] = h
    y = combine(Y, w)
    # backward
    g = np.einsum("td,tkd->tk", dy.astype(np.float32), Y, optimize=True).astype(np.float32)
    sg = (w.astype(np.float64) * g).sum(axis=1, keepdims=True)
    dlogit = (w * (g - sg)).astype(np.float32)
    dXs = np.zeros((T, k, d), dtype=np.float32)
    dW1, dW2, dW3 = {}, {}, {}
    for e, mats in experts.items():
        W2 = mats[-1]
        if e not in A:
            dW1[e] = np.zeros_like(mats[0])
            dW2[e] = np.zeros_like(W2)
            if swiglu:
                dW3[e] = np.zeros_like(mats[1])
            continue
        rows, saved = A[e]
        dYe = bf16_round((w[rows[:, 0], rows[:, 1]][:, None] * dy[rows[:, 0]]).astype(np.float32))
        dH = (dYe @ W2).astype(np.float32)
        xe = x[rows[:, 0]].astype(np.float32)
        if swiglu:
            a1, a3 = saved
            sg1 = (1.0 / (1.0 + np.exp(-a1.astype(np.float64)))).astype(np.float32)
            dsilu = (sg1 * (1.0 + a1 * (1.0 - sg1))).astype(np.float32)
            dA1 = bf16_round((dH * a3 * dsilu).astype(np.float32))
            dA3 = bf16_round((dH * a1 * sg1).astype(np.float32))
            dXs[rows[:, 0], rows[:, 1]] = bf16_round(
                (dA1 @ mats[0] + dA3 @ mats[1]).astype(np.float32))
            dW1[e] = (dA1.T @ xe).astype(np.float32)
            dW3[e] = (dA3.T @ xe).astype(np.float32)
        else:
            gp = bf16_round(gelu_tanh_grad(saved).astype(np.float32))  # saved gelu'(a), bf16
            dA = bf16_round((dH * gp).astype(np.float32))
            dXs[rows[:, 0], rows[:, 1]] = bf16_round((dA @ mats[0]).astype(np.float32))
            dW1[e] = (dA.T @ xe).astype(np.float32)
        dW2[e] = (dYe.T @ H[e]).astype(np.float32)
    dx = dXs.sum(axis=1) + np.einsum("tk,tkd->td", dlogit, wg[idx])
    dWg = np.zeros_like(wg)
    for j in range(k):
        np.add.at(dWg, idx[:, j], dlogit[:, j:j + 1] * x)
    out = dict(y=y, dx=bf16_round(dx.astype(np.float32)), g=g, dlogit=dlogit, dW1=dW1, dW2=dW2,
               dWg=dWg)
    if swiglu:
        out["dW3"] = dW3
    return out


def sprs_sum(contribs: list[np.ndarray]) -> np.ndarray:
    """Owner's reduced gradient: float32 sum in the listed (ascending device) order."""
    acc = np.zeros_like(contribs[0], dtype=np.float32)
    for c in contribs:
        acc = (acc + c.astype(np.float32)).astype(np.float32)
    return acc
