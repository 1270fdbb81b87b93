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

import numpy as np

from .errors import InternalError

ROW_ALIGN = 256  # = the CTA-pair GEMM M tile (two 128-row halves)
GROUP_DTYPE = np.dtype([("m_tiles", "<i4"), ("tile_start", "<i4"), ("a_m", "<i4"), ("a_k", "<i4"),
                        ("b_n", "<i4"), ("b_k", "<i4"), ("k_blocks", "<i4"), ("c_dest", "<i4"),
                        ("c_off", "<i8"), ("rows", "<i4"), ("reserved", "<i4")])
GEMM_NAMES = ("fwd1", "fwd2", "dgrad2", "dgrad1", "wgrad1", "wgrad2")


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
    pinned staging buffer — the product path; oracle/plan_tables_oracle.py is its checker."""

    _hdr = np.zeros(29, dtype=np.int32)  # FSSDP_TAB_HEADER_INTS
    _hdr_ptr = _hdr.ctypes.data

    def __init__(self, rank, base_owner, target_mask, route, d_model, d_ff, out_bytes=None,
                 pre_mask=None, n_mats=2, slot_layout=None):
        E, D = target_mask.shape
        _, nbytes = _layout(E, D)
        blob = out_bytes if out_bytes is not None else np.zeros(nbytes, dtype=np.uint8)
        owner = np.ascontiguousarray(base_owner, dtype=np.int32)
        mask = np.ascontiguousarray(target_mask, dtype=np.uint8)
        rt = np.ascontiguousarray(route, dtype=np.int64)
        pre = None if pre_mask is None else np.ascontiguousarray(pre_mask, dtype=np.uint8)
        lay = None if slot_layout is None else np.ascontiguousarray(slot_layout, dtype=np.int64)
        self._build(rank, E, D, owner.ctypes.data, mask.ctypes.data,
                    None if pre is None else pre.ctypes.data, rt.ctypes.data, d_model, d_ff,
                    blob, blob.ctypes.data, n_mats, None if lay is None else lay.ctypes.data)

    @classmethod
    def from_pointers(cls, rank, E, D, owner_ptr, mask_ptr, pre_ptr, route_ptr, d_model, d_ff,
                      blob, blob_ptr, n_mats=2, layout_ptr=None) -> "NativeTables":
        """Planning critical path: inputs already in place (FssdpPlanner scratch buffers),
        addresses resolved by the caller."""
        obj = cls.__new__(cls)
        obj._build(rank, E, D, owner_ptr, mask_ptr, pre_ptr, route_ptr, d_model, d_ff, blob,
                   blob_ptr, n_mats, layout_ptr)
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
               blob_ptr, n_mats=2, layout_ptr=None) -> None:
        from . import _native as N

        self.E, self.D = E, D
        self.offsets, self.nbytes = _layout(E, D)
        self.blob = blob
        if len(blob) < self.nbytes:
            raise InternalError("plan tables exceed the staging buffer")
        N.check(N.LIB_RAW.fssdp_build_rank_tables(rank, D, E, owner_ptr, mask_ptr, pre_ptr,
                                                  route_ptr, d_model, d_ff, n_mats, layout_ptr,
                                                  blob_ptr, self.nbytes, self._hdr_ptr),
                "build_rank_tables")
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
