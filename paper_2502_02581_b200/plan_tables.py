"""Device plan tables: turn one layer's global plan into the flat int32 tables the
kernels consume (SURVEY.md §3.5 boundary #2).

Every rank derives every table from the same deterministic global plan (target
placement + build_dispatch route), so no table is ever exchanged between ranks.

Receive layout on device d: its local experts occupy *slots* — owned experts
(ascending id) then replicas (ascending id; replicas fetched early first); each slot's tokens form one segment of
the receive buffers, segments in slot order, each padded to a multiple of ROW_ALIGN =
256 rows (the CTA-pair GEMM M tile), so an M tile never mixes experts and wgrad K blocks see zero pad
rows.  Inside a segment, tokens are grouped by source device (ascending), and inside
a source by that source's token-slot order.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InternalError

ROW_ALIGN = 256  # = the CTA-pair GEMM M tile (two 128-row halves)
GROUP_DTYPE = np.dtype([("m_tiles", "<i4"), ("tile_start", "<i4"), ("a_m", "<i4"), ("a_k", "<i4"),
                        ("b_n", "<i4"), ("b_k", "<i4"), ("k_blocks", "<i4"), ("c_dest", "<i4"),
                        ("c_off", "<i8")])
GEMM_NAMES = ("fwd1", "fwd2", "dgrad2", "dgrad1", "wgrad1", "wgrad2")


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


def n_tile_widths(d_ff: int, n_mats: int) -> tuple:
    """(N tile of fwd1, N tile of dgrad2 / wgrad2, whose N = d_ff).  fwd1: 128 when
    d_ff % 256 != 0 (its B rows past d_ff belong to the next matrix); SwiGLU's fwd1 always
    256 (an a1|a3 block pair per tile) — fssdp_gemm_group docs.  dgrad2 / wgrad2 read B
    N-contiguous (MN-major, inner extent d_ff): always 256-wide, the last tile ragged — TMA
    zero-fills its B columns past d_ff and clips its stores there (cfg4's 1408 = 5.5 x 256)."""
    bnf = 256 if d_ff % 256 == 0 else 128
    return (256 if n_mats == 3 else bnf), 256


def n_tiles_f(d_ff: int) -> int:
    """N tiles of dgrad2 / wgrad2 (256 wide, the last one ragged)."""
    return (d_ff + 255) // 256


def gemm_groups(seg_start, seg_padded, slot_of_seg, d_model: int, d_ff: int, shared=None,
                push=None, n_mats: int = 2, seg_rows=None):
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
    boundary past them (the zero padding beyond would only add exact zeros)."""
    d, f, nm = d_model, d_ff, n_mats
    n1 = (nm - 1) * f
    bn1, bnf = n_tile_widths(f, nm)
    n = len(seg_start)
    shared = [False] * n if shared is None else [bool(x) for x in shared]
    k_rows = seg_padded if seg_rows is None else (np.asarray(seg_rows, dtype=np.int64) + 63) // 64 * 64
    push = [None] * n if push is None else list(push)
    out = {}
    g = np.zeros(n, dtype=GROUP_DTYPE)
    for i in range(n):
        s = slot_of_seg[i]
        st = int(seg_start[i])
        g[i] = (int(seg_padded[i] // 128), 0, st, 0, s * nm * f, 0, d // 64, 0, st * n1)
    out["fwd1"] = _finalize(g.copy(), n1 // bn1)
    for i in range(n):
        s = slot_of_seg[i]
        st = int(seg_start[i])
        g[i] = (int(seg_padded[i] // 128), 0, st, 0, s * nm * d, 0, f // 64, 0, st * d)
    out["fwd2"] = _finalize(g.copy(), d // 256)
    for i in range(n):  # dH = dY . W2  (B = W2 [K=d][N=f], MN-major)
        s = slot_of_seg[i]
        st = int(seg_start[i])
        g[i] = (int(seg_padded[i] // 128), 0, st, 0, 0, s * nm * d, d // 64, 0, st * n1)
    out["dgrad2"] = _finalize(g.copy(), n_tiles_f(f))
    for i in range(n):  # dXe = dA . W1  (B = W1 / W13 [K=n1][N=d], MN-major)
        s = slot_of_seg[i]
        st = int(seg_start[i])
        g[i] = (int(seg_padded[i] // 128), 0, st, 0, 0, s * nm * f, n1 // 64, 0, st * d)
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
                     slot * nm * f * d + extra)
        head, _, t_sh = _finalize(gw[:n_sh], n_t)
        tail, _, t_rest = _finalize(gw[n_sh:], n_t)
        out[name] = (np.concatenate([head, tail]), n_t, t_sh + t_rest)
        split.append(t_sh)
    return out, tuple(split)


def build_rank_tables(rank: int, base_owner: np.ndarray, target_mask: np.ndarray,
                      route: np.ndarray, d_model: int, d_ff: int, pre_mask=None,
                      n_mats: int = 2) -> RankTables:
    """`pre_mask` (E, D): replicas already fetched by an earlier SpAG (same slots, no copy)."""
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

    # SpAG: replicas this rank materializes, pulled from the owner's slot
    copies = []
    for e, s in sorted(slots.items(), key=lambda kv: kv[1]):
        o = int(base_owner[e])
        if o != rank and not (pre_mask is not None and pre_mask[e, rank]):
            copies.append((o, maps[o][e], s))
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
                                      seg_rows=rows)
    n_owned = sum(1 for e in slots if int(base_owner[e]) == rank)
    return RankTables(rank=rank, world=D, slots=slots, n_owned=n_owned, seg_start=start,
                      seg_rows=rows, seg_padded=padded, recv_rows=int(padded.sum()),
                      route_cum=route_cum, recv_base=recv_base, zero_rows=zero_rows,
                      spag_copies=spag, sprs_jobs=sprs_jobs, sprs_srcs=sprs_srcs,
                      sprs_pull=sprs_pull, groups=groups,
                      wgrad_split=wgrad_split, n_stage=n_stage)


SECTION_NAMES = ("route_cum", "recv_base", "zero_rows", "spag", "sprs_jobs", "sprs_srcs",
                 *GEMM_NAMES, "slot_expert", "seg_start", "seg_rows", "seg_padded", "sprs_pull")


_LAYOUTS: dict = {}


def _layout(E: int, D: int):
    """Section offsets of the packed tables (fssdp_tables_layout), cached per (E, D)."""
    key = (E, D)
    if key not in _LAYOUTS:
        from . import _native as N

        offs = np.zeros(len(SECTION_NAMES), dtype=np.int64)
        total = np.zeros(1, dtype=np.int64)
        N.check(N.LIB_RAW.fssdp_tables_layout(E, D, offs.ctypes.data, total.ctypes.data),
                "tables_layout")
        _LAYOUTS[key] = (dict(zip(SECTION_NAMES, offs.tolist())), int(total[0]))
    return _LAYOUTS[key]


class NativeTables:
    """The same tables built by the C++ twin (fssdp_build_rank_tables) straight into a
    pinned staging buffer — the product path; build_rank_tables above is its checker."""

    _hdr = np.zeros(29, dtype=np.int32)  # FSSDP_TAB_HEADER_INTS
    _hdr_ptr = _hdr.ctypes.data

    def __init__(self, rank, base_owner, target_mask, route, d_model, d_ff, out_bytes=None,
                 pre_mask=None, n_mats=2):
        E, D = target_mask.shape
        _, nbytes = _layout(E, D)
        blob = out_bytes if out_bytes is not None else np.zeros(nbytes, dtype=np.uint8)
        owner = np.ascontiguousarray(base_owner, dtype=np.int32)
        mask = np.ascontiguousarray(target_mask, dtype=np.uint8)
        rt = np.ascontiguousarray(route, dtype=np.int64)
        pre = None if pre_mask is None else np.ascontiguousarray(pre_mask, dtype=np.uint8)
        self._build(rank, E, D, owner.ctypes.data, mask.ctypes.data,
                    None if pre is None else pre.ctypes.data, rt.ctypes.data, d_model, d_ff,
                    blob, blob.ctypes.data, n_mats)

    @classmethod
    def from_pointers(cls, rank, E, D, owner_ptr, mask_ptr, pre_ptr, route_ptr, d_model, d_ff,
                      blob, blob_ptr, n_mats=2) -> "NativeTables":
        """Planning critical path: inputs already in place (FssdpPlanner scratch buffers),
        addresses resolved by the caller."""
        obj = cls.__new__(cls)
        obj._build(rank, E, D, owner_ptr, mask_ptr, pre_ptr, route_ptr, d_model, d_ff, blob,
                   blob_ptr, n_mats)
        return obj

    @classmethod
    def from_header(cls, E, D, blob) -> "NativeTables":
        """Tables a fused native call (fssdp_plan_layer_tables) already wrote into `blob`,
        its header in NativeTables._hdr."""
        obj = cls.__new__(cls)
        obj.E, obj.D = E, D
        obj.offsets, obj.nbytes = _layout(E, D)
        obj.blob = blob
        obj._parse_header()
        return obj

    def _parse_header(self) -> None:
        h = self._hdr.tolist()
        (self.n_slots, self.n_owned, self.recv_rows, self.n_zero, self.n_spag, self.n_sprs_jobs,
         self.n_sprs_srcs) = h[:7]
        self.gemm = {name: (h[7 + 3 * i], h[8 + 3 * i], h[9 + 3 * i])
                     for i, name in enumerate(GEMM_NAMES)}
        self.wgrad_split = (h[25], h[26], h[27])
        self.n_stage = h[28]

    def _build(self, rank, E, D, owner_ptr, mask_ptr, pre_ptr, route_ptr, d_model, d_ff, blob,
               blob_ptr, n_mats=2) -> None:
        from . import _native as N

        self.E, self.D = E, D
        self.offsets, self.nbytes = _layout(E, D)
        self.blob = blob
        if len(blob) < self.nbytes:
            raise InternalError("plan tables exceed the staging buffer")
        N.check(N.LIB_RAW.fssdp_build_rank_tables(rank, D, E, owner_ptr, mask_ptr, pre_ptr,
                                                  route_ptr, d_model, d_ff, n_mats, blob_ptr,
                                                  self.nbytes, self._hdr_ptr), "build_rank_tables")
        self._parse_header()

    def section(self, name, dtype, count):
        off = self.offsets[name]
        return self.blob[off:off + count * np.dtype(dtype).itemsize].view(dtype)

    @property
    def slot_expert(self) -> np.ndarray:
        return self.section("slot_expert", np.int32, self.n_slots)

    @property
    def slots(self) -> dict:
        return {int(e): s for s, e in enumerate(self.slot_expert)}

    @property
    def seg_start(self):
        return self.section("seg_start", np.int32, self.n_slots)

    @property
    def seg_rows(self):
        return self.section("seg_rows", np.int32, self.n_slots)

    @property
    def seg_padded(self):
        return self.section("seg_padded", np.int32, self.n_slots)

    @property
    def zero_rows(self):
        return self.section("zero_rows", np.int32, 2 * self.n_zero).reshape(-1, 2)

    @property
    def spag_copies(self):
        return self.section("spag", np.int32, 3 * self.n_spag).reshape(-1, 3)

    @property
    def sprs_jobs(self):
        return self.section("sprs_jobs", np.int32, 3 * self.n_sprs_jobs).reshape(-1, 3)

    @property
    def sprs_srcs(self):
        return self.section("sprs_srcs", np.int32, 2 * self.n_sprs_srcs).reshape(-1, 2)

    @property
    def sprs_pull(self):
        return self.section("sprs_pull", np.int32, 2 * self.n_sprs_srcs).reshape(-1, 2)

    @property
    def route_cum(self):
        return self.section("route_cum", np.int32, self.E * (self.D + 1)).reshape(self.E, self.D + 1)

    @property
    def recv_base(self):
        return self.section("recv_base", np.int32, self.E * self.D).reshape(self.E, self.D)

    def groups(self, name) -> np.ndarray:
        return self.section(name, GROUP_DTYPE, self.gemm[name][0])
