"""Python restatement of the per-rank plan tables — TEST INFRASTRUCTURE (oracle/).

The product builds these tables in C++ (csrc/planner.cpp fssdp_build_rank_tables, reached
through paper_2502_02581_b200.plan_tables.NativeTables); this is its checker:
tests/test_plan_tables.py asserts the two produce identical bytes, and checks the
cross-rank invariants (receive positions tile every destination's segments, SpAG copies
name the owner's slot, SpRS staging indices agree between holders and owners).
Layout semantics: paper_2502_02581_b200/plan_tables.py.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2502_02581_b200.errors import InternalError
from paper_2502_02581_b200.plan_tables import (GROUP_DTYPE, ROW_ALIGN, n_tile_widths,
                                               n_tiles_f)


def slot_maps(base_owner: np.ndarray, target_mask: np.ndarray, pre_mask=None) -> list[dict]:
    """Per device: {expert: slot}.  Owned experts first (ascending), then the replicas
    fetched early (in `pre_mask`, ascending), then the other replicas (ascending)."""
    E, D = target_mask.shape
    pre = np.zeros((E, D), dtype=bool) if pre_mask is None else np.asarray(pre_mask, dtype=bool)
    maps = []
    for d in range(D):
        owned = [e for e in range(E) if base_owner[e] == d]
        reps = [e for e in range(E) if target_mask[e, d] and base_owner[e] != d]
        reps = [e for e in reps if pre[e, d]] + [e for e in reps if not pre[e, d]]
        maps.append({e: s for s, e in enumerate(owned + reps)})
    return maps


@dataclass
class RankTables:
    """Everything one rank's kernels need for one layer-iteration."""

    rank: int
    world: int
    slots: dict                  # expert -> local slot
    n_owned: int
    seg_start: np.ndarray        # [n_slots] receive row of each slot's segment
    seg_rows: np.ndarray         # [n_slots] real rows
    seg_padded: np.ndarray       # [n_slots] rows incl. padding (multiple of ROW_ALIGN)
    recv_rows: int               # total receive rows on this rank (padded)
    route_cum: np.ndarray        # [E, D+1] int32 cumulative split of this source's cells
    recv_base: np.ndarray        # [E, D] int32 first receive row on d of (this source, e)
    zero_rows: np.ndarray        # [n, 2] int32 {row, count} padding rows of this rank
    spag_copies: np.ndarray      # [n, 3] int32 {src_rank, src_slot, dst_slot}
    sprs_jobs: np.ndarray        # [n, 3] int32 {dst_slot, src_begin, src_count}
    sprs_srcs: np.ndarray        # [m, 2] int32 {rank, own slot | staging slot}, ascending rank
    sprs_pull: np.ndarray        # [m, 2] int32 {rank, grads slot on that rank} (pull transport)
    groups: dict                 # name -> (GROUP_DTYPE array, n_tiles, total_tiles)
    wgrad_split: tuple = (0, 0, 0)  # (n_shared, wgrad1_shared_tiles, wgrad2_shared_tiles)
    n_stage: int = 0             # staging slots this rank receives replica partials in


def _segments(route: np.ndarray, slots: dict, d: int):
    n = len(slots)
    rows = np.zeros(n, dtype=np.int64)
    for e, s in slots.items():
        rows[s] = int(route[:, e, d].sum())
    padded = (rows + ROW_ALIGN - 1) // ROW_ALIGN * ROW_ALIGN
    start = np.concatenate([[0], np.cumsum(padded)[:-1]]).astype(np.int64)
    return start, rows, padded


def _finalize(groups: np.ndarray, n_tiles: int):
    tiles = groups["m_tiles"].astype(np.int64) * n_tiles
    groups["tile_start"] = np.concatenate([[0], np.cumsum(tiles)[:-1]]) if len(tiles) else tiles
    return groups, n_tiles, int(tiles.sum())


def gemm_groups(seg_start, seg_padded, slot_of_seg, d_model: int, d_ff: int, shared=None,
                push=None, n_mats: int = 2, seg_rows=None, param_slots=None):
    """The six grouped-GEMM descriptor arrays of one rank (see gemm_sm100.cu).

    Slot s of the parameter region holds [W1 (f x d) | W2 (d x f)] bf16 (GeLU, n_mats 2) or
    [W13 (2f x d) | W2] (SwiGLU, n_mats 3, W13 block-interleaved); viewed as
    [(slots*n_mats*f) x d] rows for W1/W13 and, from offset n1*d, as [(slots*n_mats*d) x f]
    rows for W2 (n1 = (n_mats-1)*f, fwd1's N).  Gradient slots mirror it in fp32.

    `shared` (bool per segment): the wgrads list shared segments (experts with other
    holders — the SpRS inputs) first; the rest restart tile_start at 0 and run as a second
    launch, so SpRS can start in between.  Returns (groups, wgrad_split) with wgrad_split =
    (n_shared, wgrad1_shared_tiles, wgrad2_shared_tiles).

    `push` (per segment: None, or (owner, staging index)): a replica's wgrad writes its
    partial gradient into the owner's staging slot (c_dest = owner + 1) — the SpRS wire.

    `seg_rows` (real rows per segment): the wgrads' K stops at the first 64-row K block
    boundary past them (the zero padding beyond would only add exact zeros).

    `param_slots` (per segment, default slot_of_seg): the parameter slot B is read from
    (a model-level parameter region, fssdp_build_rank_tables slot_layout); gradient slots
    stay slot_of_seg."""
    d, f, nm = d_model, d_ff, n_mats
    n1 = (nm - 1) * f
    bn1, bnf = n_tile_widths(f, nm)
    n = len(seg_start)
    shared = [False] * n if shared is None else [bool(x) for x in shared]
    k_rows = seg_padded if seg_rows is None else (np.asarray(seg_rows, dtype=np.int64) + 63) // 64 * 64
    real = seg_padded if seg_rows is None else seg_rows  # token GEMMs: the real rows
    push = [None] * n if push is None else list(push)
    pslot = list(slot_of_seg) if param_slots is None else list(param_slots)
    out = {}
    g = np.zeros(n, dtype=GROUP_DTYPE)
    for i in range(n):
        s = pslot[i]
        st = int(seg_start[i])
        g[i] = (int(seg_padded[i] // 128), 0, st, 0, s * nm * f, 0, d // 64, 0, st * n1,
                int(real[i]), 0)
    out["fwd1"] = _finalize(g.copy(), n1 // bn1)
    for i in range(n):
        s = pslot[i]
        st = int(seg_start[i])
        g[i] = (int(seg_padded[i] // 128), 0, st, 0, s * nm * d, 0, f // 64, 0, st * d,
                int(real[i]), 0)
    out["fwd2"] = _finalize(g.copy(), d // 256)
    for i in range(n):  # dH = dY . W2  (B = W2 [K=d][N=f], MN-major)
        s = pslot[i]
        st = int(seg_start[i])
        g[i] = (int(seg_padded[i] // 128), 0, st, 0, 0, s * nm * d, d // 64, 0, st * n1,
                int(real[i]), 0)
    out["dgrad2"] = _finalize(g.copy(), n_tiles_f(f))
    for i in range(n):  # dXe = dA . W1  (B = W1 / W13 [K=n1][N=d], MN-major)
        s = pslot[i]
        st = int(seg_start[i])
        g[i] = (int(seg_padded[i] // 128), 0, st, 0, 0, s * nm * f, n1 // 64, 0, st * d,
                int(real[i]), 0)
    out["dgrad1"] = _finalize(g.copy(), d // 256)
    # each part longest-first (stable): the GEMM's snake tile order is then close to LPT
    order = (sorted([i for i in range(n) if shared[i]], key=lambda i: -int(seg_padded[i])) +
             sorted([i for i in range(n) if not shared[i]], key=lambda i: -int(seg_padded[i])))
    n_sh = sum(shared)
    split = [n_sh]
    for name, rows, n_t, extra in (("wgrad1", n1, d // 256, 0), ("wgrad2", d, n_tiles_f(f), n1 * d)):
        gw = np.zeros(n, dtype=GROUP_DTYPE)
        for j, i in enumerate(order):  # dW1 = dA^T X, dW2 = dY^T H (K = the segment's tokens)
            s = slot_of_seg[i]
            st = int(seg_start[i])
            dest, slot = (0, s) if push[i] is None else (push[i][0] + 1, push[i][1])
            gw[j] = (rows // 128, 0, 0, st, 0, st, int(k_rows[i] // 64), dest,
                     slot * nm * f * d + extra, 0, 0)
        head, _, t_sh = _finalize(gw[:n_sh], n_t)
        tail, _, t_rest = _finalize(gw[n_sh:], n_t)
        out[name] = (np.concatenate([head, tail]), n_t, t_sh + t_rest)
        split.append(t_sh)
    return out, tuple(split)


def build_rank_tables(rank: int, base_owner: np.ndarray, target_mask: np.ndarray,
                      route: np.ndarray, d_model: int, d_ff: int, pre_mask=None,
                      n_mats: int = 2, slot_layout=None) -> RankTables:
    """`pre_mask` (E, D): replicas already fetched by an earlier SpAG (same slots, no copy).
    `slot_layout` (owned_base, replica_base): parameter slots in a model-level region."""
    E, D = target_mask.shape
    if route.shape != (D, E, D):
        raise InternalError(f"route shape {route.shape} != {(D, E, D)}")
    maps = slot_maps(base_owner, target_mask, pre_mask)
    segs = [_segments(route, maps[d], d) for d in range(D)]
    slots = maps[rank]
    start, rows, padded = segs[rank]

    # where this source's rows land on every destination
    route_cum = np.zeros((E, D + 1), dtype=np.int32)
    route_cum[:, 1:] = np.cumsum(route[rank], axis=1)
    recv_base = np.zeros((E, D), dtype=np.int32)
    for e in range(E):
        for d in range(D):
            if e in maps[d]:
                s = maps[d][e]
                recv_base[e, d] = segs[d][0][s] + int(route[:rank, e, d].sum())
    zero = [(int(start[s] + rows[s]), int(padded[s] - rows[s])) for s in range(len(slots))
            if padded[s] > rows[s]]
    zero_rows = np.array(zero, dtype=np.int32).reshape(-1, 2)

    n_own = sum(1 for e in slots if int(base_owner[e]) == rank)

    def pslot(s, owned):
        if slot_layout is None:
            return s
        return slot_layout[0] + s if s < owned else slot_layout[1] + (s - owned)

    # SpAG: replicas this rank materializes, pulled from the owner's slot
    copies = []
    for e, s in sorted(slots.items(), key=lambda kv: kv[1]):
        o = int(base_owner[e])
        if o != rank and not (pre_mask is not None and pre_mask[e, rank]):
            copies.append((o, pslot(maps[o][e], E), pslot(s, n_own)))
    spag = np.array(copies, dtype=np.int32).reshape(-1, 3)

    # SpRS by push: staging index of (expert, holder) on the expert's owner — the owner's
    # experts with other holders in slot order, each followed by those holders ascending
    stage, n_stage = {}, 0
    for o in range(D):
        j = 0
        for e, s in sorted(maps[o].items(), key=lambda kv: kv[1]):
            if int(base_owner[e]) != o:
                continue
            for h in range(D):
                if h != o and target_mask[e, h]:
                    stage[(e, h)] = j
                    j += 1
        if o == rank:
            n_stage = j
    # owner side: grads[s] = sum over holders ascending of (own slot | staging slot); the
    # pull transport (fssdp_sprs_pull) reads each holder's own grads slot instead
    jobs, srcs, pull = [], [], []
    for e, s in sorted(slots.items(), key=lambda kv: kv[1]):
        if int(base_owner[e]) != rank:
            continue
        holders = [d for d in range(D) if target_mask[e, d]]
        if len(holders) <= 1:
            continue
        jobs.append((s, len(srcs), len(holders)))
        srcs.extend((h, s if h == rank else stage[(e, h)]) for h in holders)
        pull.extend((h, maps[h][e]) for h in holders)
    sprs_jobs = np.array(jobs, dtype=np.int32).reshape(-1, 3)
    sprs_srcs = np.array(srcs, dtype=np.int32).reshape(-1, 2)
    sprs_pull = np.array(pull, dtype=np.int32).reshape(-1, 2)

    order = list(range(len(slots)))  # segments are in slot order
    by_slot = {s: e for e, s in slots.items()}
    shared = [int(np.count_nonzero(target_mask[by_slot[s]])) > 1 for s in order]
    push = [None if int(base_owner[by_slot[s]]) == rank else
            (int(base_owner[by_slot[s]]), stage[(by_slot[s], rank)]) for s in order]
    groups, wgrad_split = gemm_groups(start, padded, order, d_model, d_ff, shared, push, n_mats,
                                      seg_rows=rows, param_slots=[pslot(s, n_own) for s in order])
    n_owned = sum(1 for e in slots if int(base_owner[e]) == rank)
    return RankTables(rank=rank, world=D, slots=slots, n_owned=n_owned, seg_start=start,
                      seg_rows=rows, seg_padded=padded, recv_rows=int(padded.sum()),
                      route_cum=route_cum, recv_base=recv_base, zero_rows=zero_rows,
                      spag_copies=spag, sprs_jobs=sprs_jobs, sprs_srcs=sprs_srcs,
                      sprs_pull=sprs_pull, groups=groups,
                      wgrad_split=wgrad_split, n_stage=n_stage)
