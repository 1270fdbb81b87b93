"""FssdpMoE — one FSSDP MoE layer executed on B200s (the hot path of BASELINE.json).

Forward (per rank):  K1 gate -> K2 counts all-gather -> host plan (FssdpPlanner, bit-exact
with moesim; plan + device tables + upload in one native call) -> K4 dispatch -> K3 SpAG of
the replicas this rank materializes (those the history-based candidate already implied
were pulled early, on a side stream, from the count all-gather on) -> K5 grouped FFN
(tcgen05) -> K6 combine.
Backward:  K7 token-side A2A (w·dy to the experts, <dy, Y> for the gate) -> optional
re-materialization SpAG -> dgrad2 and the weight grads of the SpRS-input slots (replica
partials are stored straight into their owners' staging slots by the GEMM epilogue) ->
K8 SpRS owner-side reduction on a side stream, beside dgrad1 and the remaining wgrads ->
dX combine + gate backward.

All heavy work is sm_100a kernels in libfssdp.so; PyTorch only owns memory and streams.
Execution is split into phases so a driver can run several logical ranks in lockstep
on one GPU (PeerGroup mode "emulated") — the multi-rank parity tests do that.
"""

from __future__ import annotations

import contextlib
import os
import ctypes as C
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import ops
from .comm import HeapLayout, PeerGroup
from .engine import FssdpPlanner, PolicyKind
from .errors import DimensionError, InternalError
from .plan_tables import NativeTables, _layout, n_tile_widths

WG_TILE = 64  # FSSDP_WG_TILE (include/fssdp.h)
GROUP_BYTES = N.C.sizeof(N.GemmGroup)  # fssdp_gemm_group

# barrier slots (flag pads) used by one layer; layer i uses base + 8*i
BAR_COUNTS, BAR_DISPATCH, BAR_Y, BAR_DGRAD, BAR_DX, BAR_END, BAR_RESHARD, BAR_SPRS = range(8)
EPOCH_SLOT0 = 72  # + layer index: the owner-update epoch of the layer (comm.FLAG_SLOTS)


@dataclass(frozen=True)
class LayerGeometry:
    d_model: int
    d_ff: int
    num_experts: int
    top_k: int
    max_tokens: int      # per rank per step
    world: int
    slots: int           # local expert slot capacity (owned + replicas)
    activation: str = "gelu"  # "gelu": [W1 | W2];  "swiglu": [W13 | W2] (Mixtral/DeepSeek)
    owned_max: int = 0        # max experts of this layer a rank owns (0: ceil(E / world))
    reshard: bool = False     # heterogeneous re-sharding enabled: a staging region for moves
    optimizer: bool = False   # AdamW state (fp32 master, m, v) of the owned shards in the heap
    # model-level parameter region (model_regions): this layer's owned slots start at
    # owned_base, its replica slots at replica_base (shared by every layer under
    # re-materialization); -1: the layer's own contiguous [owned | replica] region
    owned_base: int = -1
    replica_base: int = -1
    param_slots_total: int = 0  # slots of the model-level region (its TMA extent)
    # weight-gradient buffers (grads, SpRS staging): "bf16" — the reference's memory and
    # traffic model (grad_bytes = param bytes, engine.py:223; SpRS priced at expert_bytes,
    # engine.py:536-538): the wgrad GEMMs accumulate in fp32 (TMEM) and round once on store,
    # the SpRS sums the holders' partials in fp32 and rounds once — or "fp32"
    grad_dtype: str = "bf16"

    @property
    def n_mats(self) -> int:  # expert matrices per slot
        return 3 if self.activation == "swiglu" else 2

    @property
    def n1(self) -> int:  # fwd1's output width: a (GeLU) or the interleaved [a1|a3] (SwiGLU)
        return (self.n_mats - 1) * self.d_ff

    @property
    def recv_cap(self) -> int:
        rows = self.world * self.max_tokens * self.top_k + self.slots * 255  # 256-row padding
        return (rows + 127) // 128 * 128

    @property
    def slot_param_bytes(self) -> int:      # [W1 f×d | W2 d×f] or [W13 2f×d | W2] bf16
        return 2 * self.n_mats * self.d_model * self.d_ff

    @property
    def slot_grad_elems(self) -> int:       # the same matrices (grad_dtype elements)
        return self.n_mats * self.d_model * self.d_ff

    @property
    def grad_elem_bytes(self) -> int:
        return 2 if self.grad_dtype == "bf16" else 4

    @property
    def expert_bytes(self) -> int:
        return self.slot_param_bytes

    @property
    def split(self) -> bool:
        return self.owned_base >= 0

    @property
    def replica_cap(self) -> int:
        """Replica slots this layer may fill in one iteration."""
        return max(0, self.slots - self.owned_cap)

    @property
    def owned_cap(self) -> int:
        """Most experts of this layer one rank can own (optimizer-state slots)."""
        return self.owned_max or -(-self.num_experts // self.world)

    @property
    def stage_slots(self) -> int:
        """Staging slots for replica partial gradients pushed to this rank as an owner:
        at most (world-1) holders per owned expert, and at most every other rank's replica
        slots in total."""
        if self.world <= 1:
            return 0
        if self.owned_max:  # heterogeneous sharding: per-rank ownership varies
            return (self.world - 1) * self.owned_max
        owned_max = -(-self.num_experts // self.world)
        owned_min = self.num_experts // self.world
        return min((self.world - 1) * owned_max,
                   (self.world - 1) * max(0, self.slots - owned_min))

    def validate(self) -> None:
        if self.d_model % 256 or self.d_ff % 128:
            raise DimensionError("d_model must be a multiple of 256 and d_ff of 128 (GEMM tiles)")
        if self.grad_dtype not in ("bf16", "fp32"):
            raise DimensionError(f"grad_dtype must be 'bf16' or 'fp32', not {self.grad_dtype!r}")
        if self.activation not in ("gelu", "swiglu"):
            raise DimensionError(f"unknown expert activation {self.activation!r}")
        if not 1 <= self.top_k <= min(8, self.num_experts) or self.num_experts > 64:
            raise DimensionError("need 1 <= top_k <= 8 and num_experts <= 64")

    def add_regions(self, layout: HeapLayout, prefix: str) -> None:
        d, R = self.d_model, self.recv_cap
        if not self.split:
            layout.add(prefix + "params", self.slots * self.slot_param_bytes)
        # gradients: a replica's partial goes straight to its owner's staging slot (the
        # wgrad epilogue's c_dest stores), so the split layout keeps owned slots only
        grad_slots = self.owned_cap if self.split and self.world > 1 else self.slots
        layout.add(prefix + "grads", grad_slots * self.slot_grad_elems * self.grad_elem_bytes)
        layout.add(prefix + "xrecv", R * d * 2)
        layout.add(prefix + "y", R * d * 2)
        layout.add(prefix + "dyrecv", R * d * 2)
        layout.add(prefix + "dxe", R * d * 2)
        layout.add(prefix + "counts", (self.world * self.num_experts * 4 + 15) // 16 * 16)
        # the gate's dWg partials (two, by step parity), summed over P2P after the end barrier
        layout.add(prefix + "dwgp", 2 * self.num_experts * d * 4)
        layout.add(prefix + "stage",
                   max(1, self.stage_slots) * self.slot_grad_elems * self.grad_elem_bytes)
        # re-shard staging: the old owned shards, pulled by their new owners
        layout.add(prefix + "reshard", (self.slots if self.reshard else 1) * self.slot_param_bytes)
        if self.optimizer:  # fp32 master / exp_avg / exp_avg_sq of the owned slots (+ staging)
            n = self.owned_cap * self.slot_grad_elems * 4
            for k in ("opt_master", "opt_m", "opt_v"):
                layout.add(prefix + k, n)
            layout.add(prefix + "reshard_opt", 3 * n if self.reshard else 16)


def default_slots(num_experts: int, world: int, m: int) -> int:
    return min(num_experts, -(-num_experts // world) + max(0, m))


def model_regions(layout: HeapLayout, geoms: list, rematerialize: bool,
                  prefix: str = "L{}.") -> list:
    """The model-level parameter region plus every layer's own regions; returns the
    geometries with their slot bases.  Owned slots of every layer persist (they ARE the
    shards); replica slots follow moesim's memory model (memory_report, engine.py:188-226):
    retain = each layer keeps its replicas from forward to backward (Σ over layers),
    rematerialize = ONE replica region shared by every layer (max over layers) — a layer's
    backward re-gathers its replicas (FssdpMoE.backward, phase_spag(refetch_early=True))."""
    from dataclasses import replace

    if not geoms:
        return []
    sb = {g.slot_param_bytes for g in geoms}
    if len(sb) != 1:
        raise DimensionError("layers of one model need equal expert shapes")
    owned_bases, ob = [], 0
    for g in geoms:
        owned_bases.append(ob)
        ob += g.owned_cap
    rep_bases, rb = [], ob
    for g in geoms:
        rep_bases.append(ob if rematerialize else rb)
        rb += 0 if rematerialize else g.replica_cap
    total = ob + (max(g.replica_cap for g in geoms) if rematerialize else rb - ob)
    layout.add("params", max(1, total) * sb.pop())
    out = []
    for li, g in enumerate(geoms):
        ng = replace(g, owned_base=owned_bases[li], replica_base=rep_bases[li],
                     param_slots_total=total)
        ng.add_regions(layout, prefix.format(li))
        out.append(ng)
    return out


def replica_region_bytes(geoms: list) -> int:
    """Bytes of replica parameter slots the heap holds for these (split) geometries."""
    if not geoms or not geoms[0].split:
        return sum(g.replica_cap * g.slot_param_bytes for g in geoms)
    bases = {g.replica_base for g in geoms}
    if len(bases) == 1 and len(geoms) > 1:  # shared (re-materialization)
        return max(g.replica_cap for g in geoms) * geoms[0].slot_param_bytes
    return sum(g.replica_cap for g in geoms) * geoms[0].slot_param_bytes


class FssdpMoE:
    """One FSSDP MoE layer on one (logical) rank.

    Parameters live in the rank's symmetric heap: the owned expert shards (slots
    [0, n_owned)) and the SpAG replica slots after them; gradients likewise (fp32)."""

    def __init__(self, geom: LayerGeometry, group: PeerGroup, planner: FssdpPlanner,
                 layer_index: int = 0, seed: int = 0, prefix: str = "L0."):
        geom.validate()
        self.g = geom
        self.group = group
        self.planner = planner
        self.layer = layer_index
        self.rank = group.rank
        self.world = group.world
        self.dev = group.device
        self.seed = seed
        self.bar_base = 8 * layer_index
        L = group.layout
        heap = group.local
        d, f, E, R = geom.d_model, geom.d_ff, geom.num_experts, geom.recv_cap
        self.off = {k: L.offset(prefix + k) for k in
                    ("grads", "xrecv", "y", "dyrecv", "dxe", "counts", "stage", "reshard",
                     "dwgp")}
        # parameter slots: "params" = the region the plan tables' slot indices address
        # (model-level in the split layout), "owned" = this layer's first owned slot
        sb = geom.slot_param_bytes
        if geom.split:
            self.off["params"] = L.offset("params")
            self.off["owned"] = self.off["params"] + geom.owned_base * sb
            n_param_slots = geom.param_slots_total
        else:
            self.off["params"] = self.off["owned"] = L.offset(prefix + "params")
            n_param_slots = geom.slots
        self.opt_state = None  # {"master", "m", "v"}: [owned_cap, slot elems] fp32 heap views
        if geom.optimizer:
            for k in ("opt_master", "opt_m", "opt_v", "reshard_opt"):
                self.off[k] = L.offset(prefix + k)
            self.opt_state = {k: heap.tensor(self.off["opt_" + k],
                                             (geom.owned_cap, geom.n_mats * d * f), torch.float32)
                              for k in ("master", "m", "v")}
        self.epoch_slot = EPOCH_SLOT0 + layer_index
        self._fwd_epoch = 0
        self.flags_off = L.offset("flags")
        # params: this layer's slots from its first owned one — in the split layout only the
        # owned slots (replicas: self.replicas, see slot_params)
        self.param_region = heap.tensor(self.off["params"], (n_param_slots, geom.n_mats * d * f),
                                        torch.bfloat16)
        if geom.split:
            self.params = self.param_region[geom.owned_base:geom.owned_base + geom.owned_cap]
            self.replicas = self.param_region[geom.replica_base:
                                              geom.replica_base + geom.replica_cap]
        else:
            self.params = self.param_region
            self.replicas = None
        grad_slots = geom.owned_cap if geom.split and self.world > 1 else geom.slots
        self.grads = heap.tensor(self.off["grads"], (grad_slots, geom.n_mats * d * f),
                                 torch.bfloat16 if geom.grad_dtype == "bf16" else torch.float32)
        self.epi_wgrad = ops.EPI_BF16 if geom.grad_dtype == "bf16" else ops.EPI_F32
        self.xrecv = heap.tensor(self.off["xrecv"], (R, d), torch.bfloat16)
        self.y_e = heap.tensor(self.off["y"], (R, d), torch.bfloat16)
        self.dyrecv = heap.tensor(self.off["dyrecv"], (R, d), torch.bfloat16)
        self.dxe = heap.tensor(self.off["dxe"], (R, d), torch.bfloat16)
        self.counts_table = heap.tensor(self.off["counts"], (self.world, E), torch.int32)
        # counts readback through mapped pinned memory (SM-pushed, flag-signalled): the copy
        # engines may be busy with the caller's bulk input/output transfers
        self.counts_nbytes = (self.world * E * 4 + 15) // 16 * 16
        self.counts_host_raw = torch.zeros(self.counts_nbytes // 4 + 4, dtype=torch.int32,
                                           pin_memory=True)
        self.counts_host = self.counts_host_raw[:self.world * E].view(self.world, E)
        self.counts_host_np = self.counts_host.numpy()
        self.counts_host_ptr = self.counts_host.data_ptr()
        self.counts_flag_ptr = self.counts_host_raw.data_ptr() + self.counts_nbytes
        self.counts_dev_ptr = self.counts_table.data_ptr()
        self._counts_epoch = 0
        # wgrad destinations for replica partials: every rank's staging region, as the
        # epilogue tensor maps of wgrad1 (ldc d) and wgrad2 (ldc f); built once
        stage_elems = max(1, geom.stage_slots) * geom.slot_grad_elems
        self.dest_maps = {}
        for name, ldc in (("wgrad1", d), ("wgrad2", f)):
            blob = b"".join(ops.epilogue_tmap(self.epi_wgrad, base + self.off["stage"], ldc,
                                              stage_elems // ldc) for base in group.bases)
            self.dest_maps[name] = torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(self.dev)
        # 2-D TMA views of the parameter region (nm = matrices per slot, n1 = (nm-1) f)
        nm, n1 = geom.n_mats, geom.n1
        flat = self.param_region.view(-1)
        self.w1_view = flat.view(n_param_slots * nm * f, d)           # W1/W13 of slot s: rows s*nm*f..
        self.w2_view = flat[n1 * d:].view(n_param_slots * nm * d - (nm - 1) * d, f)  # W2: rows s*nm*d..
        # local activations (capacity-sized once, so plans never reallocate): fwd1 saves
        # gelu'(a) (GeLU) or the pre-activations [a1|a3] (SwiGLU) for dgrad2's epilogue
        self.gprime = torch.empty(R, n1, dtype=torch.bfloat16, device=self.dev)
        self.h = torch.empty(R, f, dtype=torch.bfloat16, device=self.dev)
        self.da = torch.empty(R, n1, dtype=torch.bfloat16, device=self.dev)
        self.epi_fwd1 = ops.EPI_SWIGLU if geom.activation == "swiglu" else ops.EPI_GELU
        self.epi_dgrad2 = ops.EPI_DSWIGLU if geom.activation == "swiglu" else ops.EPI_DGELU
        # per GEMM: 128-wide N tiles where N = d_ff is not a multiple of 256; CTA pairs where
        # every group has an even number of 128-row tiles (wgrad1: M = n1)
        bn1, bnf = n_tile_widths(f, nm)
        bn = {"fwd1": bn1, "fwd2": 256, "dgrad2": bnf, "dgrad1": 256, "wgrad1": 256,
              "wgrad2": bnf}
        pair = {k: self.CTA_PAIR for k in bn}
        pair["wgrad1"] = self.CTA_PAIR and (n1 // 128) % 2 == 0
        self._bn = bn
        self._gemm_flags = {k: (ops.GEMM_BN128 if bn[k] == 128 else 0) |
                               (ops.GEMM_CTA_PAIR if pair[k] else 0) for k in bn}
        Tc = geom.max_tokens
        k = geom.top_k
        tiles = (Tc + ops.GATE_TILE - 1) // ops.GATE_TILE
        self.wg = torch.empty(E, d, dtype=torch.float32, device=self.dev)
        # the gate logits on tcgen05 (one grouped-GEMM launch + selection): its workspace
        self._gate_gemm_bytes = 0
        self.gate_gemm_ws = None
        # default: only where the mma.sync gate cannot stage its split weights in shared
        # memory (E x (4 d + 16) > 80 KB, e.g. cfg4's 64 x 2048: 126 us there); at cfg2 the
        # staged mma.sync gate is as fast in isolation and 0.3 % faster per step
        gate_gemm = (self.GATE_GEMM if self.GATE_GEMM is not None
                     else E * (4 * d + 16) > 80 * 1024)
        if gate_gemm and E <= 64 and d % 64 == 0:
            self._gate_gemm_bytes = int(N.LIB.fssdp_gate_gemm_ws_bytes(geom.max_tokens, d))
            self.gate_gemm_ws = torch.empty(self._gate_gemm_bytes, dtype=torch.uint8,
                                            device=self.dev)
        self.gate_bias = torch.zeros(E, dtype=torch.float32, device=self.dev)
        self.dwg = torch.zeros(E, d, dtype=torch.float32, device=self.dev)
        self.dwg_part = [heap.tensor(self.off["dwgp"] + i * E * d * 4, (E, d), torch.float32)
                         for i in range(2)]
        self._gpar = 0  # parity of the dWg partial the last gate backward wrote
        self.topk_idx = torch.empty(Tc, k, dtype=torch.int32, device=self.dev)
        self.topk_w = torch.empty(Tc, k, dtype=torch.float32, device=self.dev)
        self.slot_rank = torch.empty(Tc, k, dtype=torch.int32, device=self.dev)
        self.tile_counts = torch.empty(max(tiles, 1), E, dtype=torch.int32, device=self.dev)
        self.tile_prefix = torch.empty_like(self.tile_counts)
        self.slot_dest = torch.empty(Tc, k, dtype=torch.int32, device=self.dev)
        self.slot_pos = torch.empty(Tc, k, dtype=torch.int32, device=self.dev)
        self.slot_grad = torch.empty(Tc, k, dtype=torch.float32, device=self.dev)
        self.dlogit = torch.empty(Tc, k, dtype=torch.float32, device=self.dev)
        # token-local copy of the K gathered expert rows (combine -> dispatch_grad's <dy, Y>):
        # the backward then pulls nothing over NVLink; one rank reads its own heap anyway
        self.y_slots = (torch.empty(Tc * k, d, dtype=torch.bfloat16, device=self.dev)
                        if self.world > 1 and self.KEEP_Y_SLOTS else None)
        # the gate backward: on the tensor cores (fssdp_gate_wgrad_tc) unless FSSDP_GATE_WGRAD_TC=0
        self._wg_tc = self.GATE_WGRAD_TC and E <= 64 and d % 256 == 0
        if self._wg_tc:
            self.wg_ws = torch.empty(int(N.LIB.fssdp_gate_wgrad_tc_ws_bytes(Tc, d)),
                                     dtype=torch.uint8, device=self.dev)
        else:
            wg_tiles = max(1, (Tc + WG_TILE - 1) // WG_TILE)
            self.wg_ws = torch.empty(wg_tiles * E * d, dtype=torch.float32, device=self.dev)
        self.grid_counter = torch.zeros(4, dtype=torch.int32, device=self.dev)
        # dynamic tile scheduler counters of this layer's GEMMs (all on the main stream, in
        # order; each launch leaves them zero) — used with FSSDP_GEMM_DYN=1
        self.gemm_sched = torch.zeros(2, dtype=torch.int32, device=self.dev)
        self._gemm_sched_ptr = C.c_void_p(self.gemm_sched.data_ptr())
        self.gate_ws = torch.zeros(1 + E, dtype=torch.int32, device=self.dev)  # ticket, totals
        self.blob_host = torch.empty(1 << 20, dtype=torch.uint8, pin_memory=True)
        self.blob_host_np = self.blob_host.numpy()
        self.blob_host_ptr = self.blob_host_np.ctypes.data
        self.blob_dev = torch.empty(1 << 20, dtype=torch.uint8, device=self.dev)
        self.blob_dev_ptr = self.blob_dev.data_ptr()
        # tables of the early (estimate-based) SpAG, staged separately from the final ones
        self.pre_host = torch.empty(1 << 20, dtype=torch.uint8, pin_memory=True)
        self.pre_host_np = self.pre_host.numpy()
        self.pre_dev = torch.empty(1 << 20, dtype=torch.uint8, device=self.dev)
        self.pre_mask = None      # (E, D) replicas fetched early this iteration, or None
        self.pre_mask_ptr = None
        self.pre_tables = None
        self._pre_done = None     # event on the side stream after the early SpAG (W1 parts)
        self._pre_w2 = None       # ... and after its W2 parts (fwd2 waits for it)
        self._pre_staged = None   # event after the H2D of pre_host (before it is rewritten)
        self.decision = None
        self.tables = None
        self._cs = None  # launching stream during forward()/backward()
        self._plan_pending = False
        # plan capacity limits + the parameter slot layout (fssdp_plan_layer_tables)
        self._slot_layout = (geom.owned_base, geom.replica_base) if geom.split else None
        self._limits = np.array(
            [geom.owned_cap if geom.split else geom.slots, geom.recv_cap, geom.stage_slots,
             geom.owned_base if geom.split else -1, geom.replica_base, geom.replica_cap],
            dtype=np.int64)
        self._limits_ptr = self._limits.ctypes.data
        self._tab_ptrs = None
        self._dispatch_args = None
        self._dispatched = False
        self._pb_c = C.c_void_p(self.group.peer_bases.data_ptr())
        self.T = 0
        self.x = None
        self._owned_expert_ids = None
        self._base_owner = None      # owner per expert of the partition the params follow
        self._reshard_pending = None  # device copy list of a re-shard gather, or None
        self.reset_plan_stats()
        self.init_parameters(seed)

    def reset_plan_stats(self) -> None:
        """Counters of the early (estimate-based) SpAG against the final plan, per forward."""
        self.plan_stats = {"plans": 0, "early": 0, "early_hit": 0, "early_extended": 0,
                           "early_fallback": 0, "late_copies": 0}

    # ------------------------------------------------------------ parameters
    def owned_experts(self) -> list:
        base = self.planner.shards.per_layer[self.layer]
        return sorted(base.chunks_on(self.rank))

    def init_parameters(self, seed: int) -> None:
        """Deterministic per-expert init (independent of ownership): W1 (W3) ~ N(0, 1/d),
        W2 ~ N(0, 1/f), Wg ~ N(0, 1/d) (replicated)."""
        d, f, E = self.g.d_model, self.g.d_ff, self.g.num_experts
        gen = torch.Generator(device=self.dev)
        gen.manual_seed(seed * 7919 + 17 + 1_000_033 * self.layer)
        self.wg.copy_(torch.randn(E, d, generator=gen, device=self.dev) / d ** 0.5)
        n1 = self.g.n1
        for s, e in enumerate(self.owned_experts()):
            mats = self.make_expert(e, seed)
            self.params[s, : n1 * d].copy_(self.pack_w13(mats[:-1]).reshape(-1))
            self.params[s, n1 * d:].copy_(mats[-1].reshape(-1))
        self._owned_expert_ids = self.owned_experts()
        self._n_owned = len(self._owned_expert_ids)
        self._base_owner = np.asarray(self.planner.shards.per_layer[self.layer].owners())

    def make_expert(self, e: int, seed: int):
        """(W1 [f,d], W2 [d,f]) or, for SwiGLU, (W1, W3 [f,d], W2) — bf16, seeded per expert."""
        d, f = self.g.d_model, self.g.d_ff
        gen = torch.Generator(device=self.dev)
        gen.manual_seed(seed * 1_000_003 + 31 * e + 1 + 100_003 * self.layer)
        w1 = (torch.randn(f, d, generator=gen, device=self.dev) / d ** 0.5).bfloat16()
        w2 = (torch.randn(d, f, generator=gen, device=self.dev) / f ** 0.5).bfloat16()
        if self.g.activation != "swiglu":
            return w1, w2
        w3 = (torch.randn(f, d, generator=gen, device=self.dev) / d ** 0.5).bfloat16()
        return w1, w3, w2

    @staticmethod
    def pack_w13(mats):
        """[W1] or the block-interleaved [W1; W3] (128-row blocks, FSSDP_EPI_SWIGLU)."""
        if len(mats) == 1:
            return mats[0]
        w1, w3 = mats
        f, d = w1.shape
        return torch.stack([w1.view(f // 128, 128, d), w3.view(f // 128, 128, d)], 1).reshape(2 * f, d)

    @staticmethod
    def unpack_w13(w13):
        """Inverse of pack_w13 for an interleaved [2f, d] tensor: (W1, W3)."""
        f2, d = w13.shape
        v = w13.reshape(f2 // 256, 2, 128, d)
        return v[:, 0].reshape(f2 // 2, d), v[:, 1].reshape(f2 // 2, d)

    def _slot_mats(self, buf, e):
        s = self._owned_expert_ids.index(e)
        d, f, n1 = self.g.d_model, self.g.d_ff, self.g.n1
        w2 = buf[s, n1 * d:].view(d, f)
        if self.g.activation != "swiglu":
            return buf[s, : f * d].view(f, d), w2
        w1, w3 = self.unpack_w13(buf[s, : n1 * d].view(n1, d))
        return w1, w3, w2

    def slot_params(self, s: int) -> torch.Tensor:
        """Parameters of local slot s of the current plan (owned slots first, then the
        replicas SpAG materialized) — a view into the parameter region."""
        n_owned = self.tables.n_owned if self.tables is not None else self._n_owned
        if self.replicas is None or s < n_owned:
            return self.params[s]
        return self.replicas[s - n_owned]

    def expert_weight(self, e: int):
        """(W1 [f,d], W2 [d,f]) of an owned expert (views into the heap); SwiGLU: (W1, W3,
        W2), W1/W3 de-interleaved copies."""
        return self._slot_mats(self.params, e)

    def expert_grad(self, e: int):
        """(dW1, dW2) [SwiGLU: (dW1, dW3, dW2)] of an owned expert after backward
        (SpRS-reduced; grad_dtype)."""
        return self._slot_mats(self.grads, e)

    # ------------------------------------------------------------ helpers
    def _stream(self):
        """The launching stream (resolved once per forward / backward call: looking up
        torch's current stream costs microseconds on the planning critical path)."""
        cs = self._cs
        if cs is None:
            cs = C.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)
        return cs

    def _bar(self, which: int):
        slot, epoch = self.group.barrier_args(self.bar_base + which)
        return slot, epoch

    def _tab(self, name: str) -> C.c_void_p:
        """Device address of a table section (the layout is fixed per (E, D))."""
        ptrs = self._tab_ptrs
        if ptrs is None:
            offs, _ = _layout(self.g.num_experts, self.world)
            ptrs = self._tab_ptrs = {k: C.c_void_p(self.blob_dev_ptr + v) for k, v in offs.items()}
        return ptrs[name]

    def _pb(self) -> C.c_void_p:
        return self._pb_c

    # ------------------------------------------------------------ forward phases
    # Early SpAG: the estimate-based candidate (engine.py:497-501) depends only on the
    # load history, so its replicas are pulled on a side stream while the gate, the
    # count all-gather and the host planner run; the final plan (a superset after
    # calibration, or the bare partition after fallback) then copies only the rest.
    # Peers read an owner's shards early, before any barrier of the step: every forward
    # first publishes an owner-update epoch (phase_publish, after the caller's optimizer
    # step in stream order) and the early copies wait for every owner's (_ce_copies).
    PREFETCH = os.environ.get("FSSDP_PREFETCH", "1") != "0"

    # FSSDP_EPOCHS=0 drops the owner-update epochs (negative control of
    # scripts/dist_train_check.py: the early copies then race the owners' optimizer step)
    EPOCHS = os.environ.get("FSSDP_EPOCHS", "1") != "0"

    def _epochs_live(self) -> bool:
        """Owner-update epochs guard the early copy-engine SpAG between processes (emulated
        ranks run in lockstep on one stream: nothing to guard)."""
        return (self.EPOCHS and self.group.mode == "dist" and self.world > 1 and self.PREFETCH
                and self.PRE_W1_CE)

    def phase_publish(self) -> None:
        """Owner-update epoch: this rank's owned shards are final for forward #e — stream-
        ordered after whatever the caller ran before this forward (its optimizer step), so
        a peer's early SpAG (which starts before any barrier of the step) may read them."""
        self._fwd_epoch += 1
        if self._epochs_live():
            self._call("fssdp_publish_epoch", self._pb(), self.flags_off, self.epoch_slot,
                       self.rank, C.c_uint32(self._fwd_epoch & 0xFFFFFFFF), self._stream())

    def phase_prefetch(self) -> None:
        self.pre_mask, self.pre_mask_ptr, self.pre_tables, self._pre_done = None, None, None, None
        self._pre_w2 = None
        self._pre_launch = False
        self._pre_w2_pending = False
        if not self.PREFETCH:
            return
        if self._base_owner is not None and not np.array_equal(
                self._base_owner, self.planner._owners(self.layer)):
            return  # a re-shard of this layer is pending: its owners' slots are not in place
        pre = self.planner.candidate(self.layer)
        if pre is None:
            return
        if self._pre_staged is not None:
            self._pre_staged.synchronize()  # last iteration's H2D of pre_host has landed
        base_owner = self.planner._owners(self.layer)
        E, D = pre.shape
        tables = NativeTables(self.rank, base_owner, pre, np.zeros((D, E, D), dtype=np.int64),
                              self.g.d_model, self.g.d_ff, out_bytes=self.pre_host_np,
                              n_mats=self.g.n_mats, slot_layout=self._slot_layout)
        n_rep, rep_cap = tables.n_slots - tables.n_owned, self.g.slots - self.g.owned_cap
        if tables.n_slots > self.g.slots or (self.g.split and n_rep > rep_cap):
            raise InternalError(f"early plan needs {tables.n_slots} slots > capacity {self.g.slots}")
        self.pre_mask, self.pre_mask_ptr, self.pre_tables = pre, pre.ctypes.data, tables
        if tables.n_spag == 0:
            return
        main = torch.cuda.current_stream(self.dev)
        side = self._side_stream()
        side.wait_stream(main)  # previous users of the replica slots are done
        with torch.cuda.stream(side):
            nb = tables.nbytes
            self.pre_dev[:nb].copy_(self.pre_host[:nb], non_blocking=True)
            self._pre_staged = torch.cuda.Event()
            self._pre_staged.record(side)
        self._pre_launch = True  # the copies themselves start at PREFETCH_AT
        if self.PREFETCH_AT == "gate" or self.PRE_W1_CE:
            self._launch_prefetch()

    def _launch_prefetch(self) -> None:
        """Early SpAG on the side stream, ordered after the gate and the count all-gather:
        it then runs in the host-planning gap instead of slowing the gate (measured)."""
        if not getattr(self, "_pre_launch", False):
            return
        self._pre_launch = False
        if self.PRE_W1_CE:
            self._pre_done = self._ce_copies(0, self.g.n1 * self.g.d_model * 2)
        else:
            self._launch_prefetch_w1()
        self._pre_w2_pending = True
        if not (self.PRE_W2_AFTER_DISPATCH or self.PRE_W2_CE):
            self._launch_prefetch_w2()

    # the early SpAG's W1 parts by the copy engines too, started with the gate (an SM copy
    # kernel there slowed the gate; the copy engines take no SMs) — N=4, interleaved A/B:
    # 1.794 -> 1.787 ms.  FSSDP_PRE_W1_CE=0: the bounded-grid SM kernel at PREFETCH_AT
    PRE_W1_CE = os.environ.get("FSSDP_PRE_W1_CE", "1") != "0"

    def _launch_prefetch_w1(self) -> None:
        main = torch.cuda.current_stream(self.dev)
        side = self._side_stream()
        side.wait_stream(main)
        with torch.cuda.stream(side):
            # fwd1 reads only W1 (W13) of a replica: that part first, its own event, then
            # W2 — which crosses NVLink while fwd1 runs (fwd2 waits for it)
            n1b = self.g.n1 * self.g.d_model * 2
            self._spag_launch("spag_pre", self.pre_dev, self.pre_tables, side, 0, n1b)
            self._pre_done = torch.cuda.Event()
            self._pre_done.record(side)

    # experiment (off): start the early SpAG's W2 part once the dispatch is done.  The
    # dispatch then has NVLink to itself (N=4: 105 -> 48 us) but the step is not faster
    # (1.792 vs 1.800 ms, interleaved A/B): W2 then lands during fwd1, which it slows
    PRE_W2_AFTER_DISPATCH = os.environ.get("FSSDP_PRE_W2_AFTER_DISPATCH", "0") == "1"

    # the early SpAG's W2 parts by the copy engines, once the dispatch is done: they cross
    # NVLink beside fwd1 without taking its SMs (an SM copy kernel cannot co-reside with the
    # GEMM's 227 KB CTAs and delays them), and the dispatch has NVLink to itself
    # (N=4, interleaved A/B: dispatch 103 -> 48 us, step 1.799 -> 1.756 ms)
    PRE_W2_CE = os.environ.get("FSSDP_PRE_W2_CE", "1") != "0"

    def _launch_prefetch_w2_ce(self, after=None) -> None:
        n1b = self.g.n1 * self.g.d_model * 2
        self._pre_w2 = self._ce_copies(n1b, self.g.slot_param_bytes - n1b, after)

    def _ce_copies(self, part_off: int, part_bytes: int, after=None) -> torch.cuda.Event:
        """The early SpAG's copies of one part of every slot, by the copy engines on their
        own stream (after the current stream's work, or after the event `after`); returns
        their completion event.  The W1 part starts before any barrier of the step: it
        first waits until every owner published this forward's epoch (its shards are final
        — phase_publish)."""
        ce = getattr(self, "_ce", None)
        if ce is None:
            ce = self._ce = torch.cuda.Stream(device=self.dev)
        if after is not None:
            ce.wait_event(after)
        else:
            ce.wait_stream(torch.cuda.current_stream(self.dev))
        if part_off == 0 and self._epochs_live():
            N.call_raw("fssdp_wait_epochs", self._pb(), self.flags_off, self.epoch_slot,
                       self.world, C.c_uint32(self._fwd_epoch & 0xFFFFFFFF),
                       C.c_void_p(ce.cuda_stream))
        sb = self.g.slot_param_bytes
        off = self.off["params"] + part_off
        bases = self.group.bases
        s = C.c_void_p(ce.cuda_stream)
        copies = self.pre_tables.spag_copies.tolist()
        if self.timers is not None and copies:  # bench: the copies' window on their stream
            t0, t1 = N.NativeEvent(), N.NativeEvent()
            t0.record(ce)
        for src_rank, src_slot, dst_slot in copies:
            N.call_raw("fssdp_copy_async", C.c_void_p(bases[self.rank] + off + dst_slot * sb),
                       C.c_void_p(bases[src_rank] + off + src_slot * sb), part_bytes, s)
        if self.timers is not None and copies:
            t1.record(ce)
            self.timers.setdefault("spag_pre", []).append((t0, t1))
        ev = torch.cuda.Event()
        ev.record(ce)
        return ev

    def _launch_prefetch_w2(self, after=None) -> None:
        if not getattr(self, "_pre_w2_pending", False):
            return
        self._pre_w2_pending = False
        if self.PRE_W2_CE:
            self._launch_prefetch_w2_ce(after)
            return
        side = self._side_stream()
        if self.PRE_W2_AFTER_DISPATCH:
            side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):
            n1b = self.g.n1 * self.g.d_model * 2
            self._spag_launch("spag_pre", self.pre_dev, self.pre_tables, side, n1b,
                              self.g.slot_param_bytes - n1b)
            self._pre_w2 = torch.cuda.Event()
            self._pre_w2.record(side)

    # the early SpAG runs beside the count readback, the host planning and the table upload:
    # a bounded grid (one CTA per SM by default, FSSDP_SPAG_PRE_CTAS; 0 = full width) keeps
    # those small transfers from stalling behind it (N=4: the table upload went from ~90 to
    # ~20 us, the step from 1.874 to 1.844 ms; N=2 unchanged — profiles/r1_spag_pre_ctas.txt)
    SPAG_PRE_CTAS = int(os.environ.get("FSSDP_SPAG_PRE_CTAS", "-1"))

    def _spag_launch(self, key, blob_dev, tables, stream, part_off=0, part_bytes=0) -> None:
        """SpAG copies of `tables`; part_off / part_bytes (0 = whole slot) select a part of
        every slot (W1 or W2)."""
        spag = C.c_void_p(blob_dev.data_ptr() + tables.offsets["spag"])
        off = self.off["params"] + part_off
        cap = 0
        if key == "spag_pre":
            cap = self.SPAG_PRE_CTAS if self.SPAG_PRE_CTAS >= 0 else N.LIB.fssdp_num_sms()
        self._timed(key, lambda: N.call(
            "fssdp_gather_slots", self._pb(), self.rank, off, off, self.g.slot_param_bytes,
            part_bytes, spag, tables.n_spag, cap, C.c_void_p(stream.cuda_stream)))

    def phase_gate(self, x: torch.Tensor) -> None:
        if x.dtype != torch.bfloat16 or x.dim() != 2 or x.shape[1] != self.g.d_model:
            raise DimensionError(f"x must be [T, {self.g.d_model}] bf16, got {tuple(x.shape)} {x.dtype}")
        T = x.shape[0]
        if T > self.g.max_tokens:
            raise DimensionError(f"{T} tokens exceed max_tokens={self.g.max_tokens}")
        self.x = x.contiguous()
        self.T = T
        E, k = self.g.num_experts, self.g.top_k
        # K1 + K2 fused: the gate's last CTA scans the tile counts, all-gathers this rank's
        # totals and joins the count barrier
        slot, epoch = self._bar(BAR_COUNTS)
        # host boundary #1 inside the same launch (after the count barrier the table is
        # complete) — not under lockstep emulation, whose ranks' gates run one after another
        fused = self.FUSED_PUSH and (self.group.mode == "dist" or self.world == 1)
        self._pushed_with_gate = fused
        if fused:
            self._counts_epoch = (self._counts_epoch + 1) & 0xFFFFFFFF
        self._call("fssdp_gate_route", ops._ptr(self.x), ops._ptr(self.wg),
                   ops._ptr(self.gate_bias), T, self.g.d_model, E, k, ops._ptr(self.topk_idx),
                   ops._ptr(self.topk_w), ops._ptr(self.slot_rank), ops._ptr(self.tile_counts),
                   ops._ptr(self.tile_prefix), ops._ptr(self.gate_ws), self._pb(),
                   self.off["counts"], self.flags_off, self.rank, self.world, slot, epoch,
                   C.c_void_p(self.blob_dev_ptr) if self.LOCAL_DISPATCH and self.world == 1
                   else None,
                   self.g.d_ff if self._local_gemm else 0, self.g.n_mats,
                   max(0, self.g.owned_base),
                   C.c_void_p(self.counts_host_ptr if fused else 0), self.counts_nbytes,
                   C.c_void_p(self.counts_flag_ptr if fused else 0),
                   C.c_uint32(self._counts_epoch),
                   ops._ptr(self.gate_gemm_ws), self._gate_gemm_bytes, self._stream())
        if self.gate_gemm_ws is not None:
            N.launch_count += 2  # + the weight-split and GEMM launches

    def phase_counts(self) -> None:
        """The counts are all-gathered by the gate launch; the early SpAG may start now."""
        if self.PREFETCH_AT == "counts":
            self._launch_prefetch()

    # the gate launch also pushes the counts to the host (FSSDP_FUSED_PUSH=0: a separate
    # push_host kernel after it)
    FUSED_PUSH = os.environ.get("FSSDP_FUSED_PUSH", "1") != "0"
    _pushed_with_gate = False

    # where the early SpAG starts: with the gate ("gate"), after the count all-gather
    # ("counts"), or once the counts readback has left ("push")
    PREFETCH_AT = os.environ.get("FSSDP_PREFETCH_AT", "counts")

    def _push_counts(self) -> None:
        """Host boundary #1: the all-gathered counts to mapped pinned memory + a flag, by the
        SMs (a copy-engine transfer would queue behind the caller's bulk copies)."""
        self._mark("readback")
        if not self._pushed_with_gate:
            self._counts_epoch = (self._counts_epoch + 1) & 0xFFFFFFFF
            self._timed("push_host", lambda: N.check(N.LIB_RAW.fssdp_push_host(
                self.counts_dev_ptr, self.counts_host_ptr, self.counts_nbytes,
                self.counts_flag_ptr, self._counts_epoch, self._stream()), "counts readback"))
        if self.PREFETCH_AT == "push":
            self._launch_prefetch()

    def phase_plan(self, dispatch: bool = False, pushed: bool = False) -> None:
        """Counts readback, host plan, table upload; with dispatch=True the dispatch is
        launched right after the upload, before any Python bookkeeping of the plan."""
        if not pushed:
            self._push_counts()
        N.check(N.LIB_RAW.fssdp_host_wait(self.counts_flag_ptr, self._counts_epoch, 60.0),
                "counts readback")
        t_host = time.perf_counter()
        self._mark("synced")
        self._plan_tables(self.counts_host_np, dispatch)
        if self.timers is not None:
            self.timers.setdefault("host_plan_s", []).append(time.perf_counter() - t_host)

    # N > 1: counts wait, plan, tables, upload and the dispatch launch in ONE native call
    # with its arguments built before the counts arrive (no Python on the critical path).
    # The instrumented passes (phase timers, gap probe) keep the separate calls.
    FUSED_PLAN = os.environ.get("FSSDP_FUSED_PLAN", "1") != "0"

    def _fused_plan_ok(self) -> bool:
        return (self.FUSED_PLAN and self.timers is None and self.gap_events is None and
                self.planner.policy.reshard_interval == 0 and self._reshard_pending is None)

    def phase_plan_dispatch(self) -> None:
        self._push_counts()
        E, D = self.g.num_experts, self.world
        args = self.planner.plan_call_args(
            self.layer, (D, E), self.counts_host_ptr, self.rank, self.pre_mask_ptr,
            self.g.d_model, self.g.d_ff, self.blob_host_np, self.blob_host_ptr,
            NativeTables._hdr_ptr, self.blob_dev_ptr, self._stream(), self._limits_ptr,
            self.g.n_mats)
        dl = self._dispatch_launch
        if dl is None:
            dl = self._dispatch_launch = N.DispatchLaunch(
                0, self.topk_idx.data_ptr(), self.slot_rank.data_ptr(),
                self.tile_prefix.data_ptr(), 0, self.g.d_model, E, self.g.top_k, self.world,
                self.slot_dest.data_ptr(), self.slot_pos.data_ptr(), self.group.peer_bases.data_ptr(),
                self.off["xrecv"], self.flags_off, self.rank, 0, 0, self.grid_counter.data_ptr())
        dl.x = self.x.data_ptr()
        dl.T = self.T
        dl.bar_slot, dl.epoch = self._bar(BAR_DISPATCH)
        N.check(N.LIB_RAW.fssdp_plan_layer_dispatch(
            self.counts_flag_ptr, self._counts_epoch, 60.0, *args, C.byref(dl)),
            "plan_layer_dispatch")
        N.launch_count += N.KERNELS_PER_CALL["fssdp_plan_layer_dispatch"]
        self._mark("dispatch_issued")
        self.planner.plan_counts(self.layer, self.counts_host_np)
        self._dispatched = True
        tables = NativeTables.from_header(E, D, self.blob_host_np)
        self.tables = self.packed = tables
        self.gemm = tables.gemm
        self._plan_pending = True

    _dispatch_launch = None

    def _plan_tables(self, counts, dispatch: bool = False) -> None:
        # plan + this rank's tables + their upload (boundary #2), capacity-checked: one native
        # call; the Python-side decision object is built after the dispatch is launched
        E, D = self.g.num_experts, self.world
        # (timed as "pull_host": the native window covers only the table upload kernel)
        # single rank with device-written tables (the gate's tail): the device blob already
        # holds every section the kernels read, byte-equal — no upload
        dev_blob = None if self._local_gemm else self.blob_dev_ptr
        self._timed("pull_host", lambda: self.planner.plan_with_tables(
            self.layer, counts, self.counts_host_ptr, self.rank, self.pre_mask_ptr,
            self.g.d_model, self.g.d_ff, self.blob_host_np, self.blob_host_ptr,
            NativeTables._hdr_ptr, dev_blob, self._stream(), self._limits_ptr,
            decide=False, n_mats=self.g.n_mats))
        self._mark("planned")
        if self.gap_events is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            self.gap_events[-1] = (self.gap_events[-1][0], e1)
        self._dispatched = False
        if dispatch and not self.planner.last_reshard_moves:
            self.phase_dispatch(n_zero=int(NativeTables._hdr[3]))  # header: n_zero
            self._dispatched = True
        if self.planner.last_reshard_moves:
            self._reshard_stage()
        tables = NativeTables.from_header(E, D, self.blob_host_np)
        self.tables = self.packed = tables
        self.gemm = tables.gemm
        self._plan_pending = True

    def _finish_plan(self) -> None:
        """Decision object and consistency checks, off the planning critical path."""
        if not self._plan_pending:
            return
        self._plan_pending = False
        dec = self.planner.last_decision(self.layer)
        tables = self.tables
        target = dec.target.mask  # 0/1 uint8, like pre_mask
        pre = self.pre_mask
        if pre is not None and np.any(pre > target):
            # the final plan dropped a prefetched replica: it can only be the bare
            # partition (fallback), which has no replica slots — keep the layout check honest
            if np.any(target > dec.base.mask):
                raise InternalError("final placement is neither a superset of the early one "
                                    "nor the bare partition")
        st = self.plan_stats
        st["plans"] += 1
        st["late_copies"] += int(tables.n_spag)
        if pre is not None:
            st["early"] += 1
            if np.array_equal(pre, target):
                st["early_hit"] += 1          # the final plan is exactly the early one
            elif not np.any(target > dec.base.mask):
                st["early_fallback"] += 1     # dropped: the bare partition (fallback)
            else:
                st["early_extended"] += 1     # calibration added replicas (late SpAG)
        if tables.n_owned != self._n_owned or (
                self.planner.last_reshard_moves and
                list(tables.slot_expert[:tables.n_owned]) != self._owned_expert_ids):
            raise InternalError("ownership changed without a re-shard data move")
        self.decision = dec

    def phase_spag(self, refetch_early: bool = False) -> None:
        """The SpAG of the final plan's replicas not fetched early; the main stream then
        waits for the early SpAG.  `refetch_early` (rematerialization in backward) also
        re-pulls the early replicas."""
        if self._pre_done is None and not self.tables.n_spag and not refetch_early:
            return
        main = torch.cuda.current_stream(self.dev)
        if self._pre_done is not None:
            main.wait_event(self._pre_done)
            self._pre_done = None
        if refetch_early and self.pre_tables is not None and self.pre_tables.n_spag:
            if self._pre_staged is not None:  # pre_dev was uploaded on the side stream
                main.wait_event(self._pre_staged)
            self._spag_launch("spag_pre", self.pre_dev, self.pre_tables, main)
        if self.tables.n_spag:
            self._spag_launch("spag", self.blob_dev, self.tables, main)

    # ------------------------------------------------------------ re-sharding
    # When the planner's re-shard trigger (engine.py:470-487) adopts a new ShardPlan, the
    # owned shards follow it: every rank copies its old owned slots into its staging region
    # (planning phase), then — after a device barrier — every rank pulls its new owned
    # experts, in slot order, from their old owners' staging (dispatch phase, before the
    # dispatch's own barrier, so no replica is pulled from a shard still in flight).  With
    # an optimizer (geometry optimizer=True) its fp32 master and both moments move the same
    # way: params + 6x state = the 7x expert_bytes per moved expert the reference prices
    # (engine.py:233, 444-453).
    def _reshard_stage(self) -> None:
        new_owner = np.asarray(self.planner.shards.per_layer[self.layer].owners())
        if np.array_equal(new_owner, self._base_owner):
            return  # this layer's partition did not change
        if not self.g.reshard:
            raise InternalError("re-sharding needs a layer built with reshard=True "
                                "(policy.reshard_interval > 0)")
        nb = self._n_owned * self.g.slot_param_bytes
        if nb:
            stage = self.group.local.tensor(self.off["reshard"], (nb,), torch.uint8)
            stage.copy_(self.params.view(torch.uint8).view(-1)[:nb])
        if self.opt_state is not None and self._n_owned:  # the Adam state moves with them
            ost = self.group.local.tensor(self.off["reshard_opt"],
                                          (3, self.g.owned_cap, self.g.slot_grad_elems),
                                          torch.float32)
            for i, k in enumerate(("master", "m", "v")):
                ost[i, :self._n_owned].copy_(self.opt_state[k][:self._n_owned])
        old_owner = self._base_owner
        old_slots = {r: sorted(int(e) for e in np.flatnonzero(old_owner == r))
                     for r in range(self.world)}
        new_owned = sorted(int(e) for e in np.flatnonzero(new_owner == self.rank))
        copies = np.array([(int(old_owner[e]), old_slots[int(old_owner[e])].index(e), s)
                           for s, e in enumerate(new_owned)], dtype=np.int32).reshape(-1, 3)
        self._reshard_pending = torch.from_numpy(copies).to(self.dev)
        self._owned_expert_ids = new_owned
        self._n_owned = len(new_owned)
        self._base_owner = new_owner

    def _reshard_gather(self) -> None:
        copies = self._reshard_pending
        if copies is None:
            return
        self._reshard_pending = None
        self.phase_barrier(BAR_RESHARD)  # every old owner has staged its shards
        self._call("fssdp_gather_slots", self._pb(), self.rank, self.off["reshard"],
                   self.off["owned"], self.g.slot_param_bytes, 0, ops._ptr(copies),
                   copies.shape[0], 0, self._stream())
        if self.opt_state is not None:  # fp32 master / exp_avg / exp_avg_sq: 6x expert_bytes
            sb = self.g.slot_grad_elems * 4
            for i, k in enumerate(("opt_master", "opt_m", "opt_v")):
                self._call("fssdp_gather_slots", self._pb(), self.rank,
                           self.off["reshard_opt"] + i * self.g.owned_cap * sb, self.off[k], sb,
                           0, ops._ptr(copies), copies.shape[0], 0, self._stream())

    def phase_dispatch(self, n_zero: int | None = None) -> None:
        """K4 — first launch after the host plan: its arguments are mostly prebuilt (the
        Python between the table upload and this launch is GPU idle time)."""
        self._reshard_gather()
        slot, epoch = self._bar(BAR_DISPATCH)
        a = self._dispatch_args
        if a is None:
            a = self._dispatch_args = (
                ops._ptr(self.topk_idx), ops._ptr(self.slot_rank), ops._ptr(self.tile_prefix),
                ops._ptr(self.slot_dest), ops._ptr(self.slot_pos), self._pb(),
                C.c_void_p(self.grid_counter.data_ptr()))
        idx, rank_, prefix, dest, pos, pb, counter = a
        self._call("fssdp_dispatch", C.c_void_p(self.x.data_ptr()), idx, rank_, prefix, self.T,
                   self.g.d_model, self.g.num_experts, self.g.top_k, self.world,
                   self._tab("route_cum"), self._tab("recv_base"), dest, pos, pb,
                   self.off["xrecv"], self._tab("zero_rows"),
                   self.tables.n_zero if n_zero is None else n_zero,
                   self.flags_off, self.rank, slot, epoch, counter, self._stream())
        self._mark("dispatch_issued")

    # CUDA-event instrumentation (bench.py): name -> list of (start, end) events recorded on
    # the launching stream around each kernel launch; None disables it.
    timers = None

    def _mark(self, name: str) -> None:
        """Host timestamp of a planning-path point (bench.py's host breakdown)."""
        if self.timers is not None:
            self.timers.setdefault("marks", []).append((name, time.perf_counter()))

    def _timed(self, key, fn):
        """fn (one device entry point), inside a native launch-timing window when profiling:
        the events sit right around its kernels, so host time spent issuing the launch
        never counts as kernel time (torch events around the call would hold it whenever
        the GPU is waiting for this launch)."""
        if self.timers is None:
            fn()
        else:
            N.timed_launch(self.timers, key, fn)

    # tile order per GEMM: N-fastest (neighbouring CTAs share the A tile: the activation
    # rows) for the forward / dgrad GEMMs, M-fastest (sharing the B tile) for the wgrads
    # (fwd1 / dgrad2 N-fastest too: 0.4 % per step, interleaved A/B at N = 1)
    N_FASTEST = {"fwd2": True, "dgrad1": True, "fwd1": True, "dgrad2": True}
    for _k in os.environ.get("FSSDP_NFAST", "").split(","):  # experiments: extra N-fastest GEMMs
        if _k:
            N_FASTEST[_k] = True
    KEEP_Y_SLOTS = os.environ.get("FSSDP_KEEP_Y", "1") != "0"
    # N > 1: dispatch_grad writes the gate's dlogit (whole tokens per 4-slot warp batch), so
    # the gate backward runs on its own stream beside the expert GEMMs instead of after the
    # dX combine at the end of the step (N=4: 1.816 -> 1.805 ms).  One rank keeps it beside
    # the last wgrads (interleaved A/B at N=1: 0.3-0.5 % faster there, cfg2 and cfg4)
    EARLY_GATE = os.environ.get("FSSDP_EARLY_GATE", "1") != "0"

    # experiment: where the dX combine and (N = 1) the gate backward run — "overlap" (dx
    # stream beside the remaining wgrads), "gate_end" (gate backward after them on the main
    # stream), "serial" (both after them), "dx_first" (the dX combine on the main stream
    # before them, the gate backward beside them)
    DX_MODE = os.environ.get("FSSDP_DX_MODE", "overlap")
    GATE_WGRAD_TC = os.environ.get("FSSDP_GATE_WGRAD_TC", "1") == "1"
    # experiment (FSSDP_LATE_DOTS=1): the gate's <dy, Y> dots in the dX combine (beside
    # the wgrads) instead of in dispatch_grad, which then only scatters w * dy on the
    # critical path — where the gate backward follows the dX combine anyway (no early
    # gate).  Bit-identical (test); measured 0.5 % SLOWER per step at N=1 (interleaved
    # A/B: the 100 MB of extra reads slow the wgrads they run beside more than
    # dispatch_grad gains), so off by default
    LATE_DOTS = os.environ.get("FSSDP_LATE_DOTS", "0") == "1"

    @property
    def _late_dots(self) -> bool:
        return self.LATE_DOTS and not self._early_gate

    @property
    def _early_gate(self) -> bool:
        return self.EARLY_GATE and 4 % self.g.top_k == 0 and self.world > 1
    CTA_PAIR = True  # tcgen05 cta_group::2 256x256 tiles (segments are 256-row aligned)
    # the gate logits as a tcgen05 GEMM: FSSDP_GATE_GEMM=1 always, =0 never, unset: where
    # the mma.sync gate cannot stage its weights (see __init__)
    GATE_GEMM = {"0": False, "1": True}.get(os.environ.get("FSSDP_GATE_GEMM", ""))
    # dynamic tile scheduling of the grouped GEMMs (FSSDP_GEMM_DYN=1): measured neutral in
    # isolation (cfg2 shapes within +-1.5 %) and 1.7 % slower per step than the static snake
    # order (interleaved A/B, N=1), so off by default
    # (FSSDP_GEMM_DYN=name,name: only those GEMMs)
    _dyn = os.environ.get("FSSDP_GEMM_DYN", "0")
    GEMM_DYN = (set(("fwd1", "fwd2", "dgrad2", "dgrad1", "wgrad1", "wgrad2")) if _dyn == "1"
                else set() if _dyn == "0" else set(_dyn.split(",")))
    # A-tile multicast across two CTA pairs (FSSDP_GEMM_MULTICAST): these GEMMs, where
    # eligible (N-fastest, CTA pairs, 256-wide N tiles, even n_tiles)
    GEMM_MC = set(x for x in os.environ.get("FSSDP_GEMM_MC", "").split(",") if x)
    # short last rounds as half tiles (FSSDP_GEMM_SPLIT_TAIL; the kernel applies it only
    # where eligible and useful)
    SPLIT_TAIL = set(x for x in os.environ.get("FSSDP_SPLIT_TAIL", "").split(",") if x)
    # swapped-operand tail tiles of the token GEMMs (the kernel applies them where eligible:
    # bf16 / GeLU / dGeLU epilogues, 256-wide N tiles): +0.3 % cfg2, +1.2 % cfg4 per step
    # (interleaved A/B); FSSDP_SWAP_TAIL=name,name or "0" overrides
    _swap = os.environ.get("FSSDP_SWAP_TAIL")
    SWAP_TAIL = (set(("fwd1", "fwd2", "dgrad2", "dgrad1")) if _swap is None
                 else set(x for x in _swap.split(",") if x and x != "0"))

    def _call(self, name, *args):
        """One device entry point, CUDA-event-timed under its own name when profiling."""
        if self.timers is None:
            N.call_raw(name, *args)
        else:
            self._timed(name[6:], lambda: N.call_raw(name, *args))

    def _gemm(self, name, a, a_mn, b, b_mn, c, ldc, epi, c2=None, aux=None, part=None):
        """One grouped GEMM of the plan; `part` "shared" / "rest" launches the wgrad prefix
        of SpRS-input slots / the remaining groups (tables: wgrad_split)."""
        ng, n_tiles, total = self.gemm[name]
        tab = self._tab(name)
        if part is not None:
            n_sh = self.tables.wgrad_split[0]
            t_sh = self.tables.wgrad_split[1 if name == "wgrad1" else 2]
            if part == "shared":
                ng, total = n_sh, t_sh
            else:
                ng, total = ng - n_sh, total - t_sh
                tab = C.c_void_p(tab.value + n_sh * GROUP_BYTES)
        if total == 0:
            return
        flags = (1 if self.N_FASTEST.get(name, False) else 0) | self._gemm_flags[name]
        if name in self.SPLIT_TAIL:
            flags |= ops.GEMM_SPLIT_TAIL
        if name in self.SWAP_TAIL:
            flags |= ops.GEMM_SWAP_TAIL
        if name in self.GEMM_MC and flags & 1 and flags & ops.GEMM_CTA_PAIR and \
                not flags & ops.GEMM_BN128 and n_tiles % 2 == 0 and name not in self.GEMM_DYN:
            flags |= ops.GEMM_MULTICAST
        maps = ops._ptr(self.dest_maps.get(name))
        self._timed("gemm." + name, lambda: N.call(
            "fssdp_grouped_gemm", int(a_mn), int(b_mn), epi, ops._ptr(a), a.shape[1], a.shape[0],
            ops._ptr(b), b.shape[1], b.shape[0], tab, ng, n_tiles, total, ops._ptr(c),
            ops._ptr(c2), ops._ptr(aux), maps, ldc, c.numel() // ldc, flags,
            self._gemm_sched_ptr if name in self.GEMM_DYN else None, self._stream()))

    # fwd1 is launched before the host issues the early SpAG's W2 copies (they still start
    # after the dispatch: an event recorded before fwd1): issuing the copies first delayed
    # fwd1's launch by the host time of the copy calls (N=4: a ~30 us GPU gap)
    W2_AFTER_FWD1_LAUNCH = os.environ.get("FSSDP_W2_AFTER_FWD1_LAUNCH", "1") != "0"

    def phase_experts_fwd(self) -> None:
        f, d, n1 = self.g.d_ff, self.g.d_model, self.g.n1
        late = (self.W2_AFTER_FWD1_LAUNCH and self.PRE_W2_CE and
                getattr(self, "_pre_w2_pending", False))
        if late:
            after = torch.cuda.Event()
            after.record(torch.cuda.current_stream(self.dev))  # the dispatch (+ late SpAG)
        else:
            self._launch_prefetch_w2()  # after the dispatch (and any late SpAG) in stream order
        self._gemm("fwd1", self.xrecv, False, self.w1_view, False, self.gprime, n1, self.epi_fwd1,
                   c2=self.h)
        if late:
            self._launch_prefetch_w2(after)
        if self._pre_w2 is not None:  # the early replicas' W2 parts
            torch.cuda.current_stream(self.dev).wait_event(self._pre_w2)
            self._pre_w2 = None
        self._gemm("fwd2", self.h, False, self.w2_view, False, self.y_e, d, ops.EPI_BF16)

    def phase_barrier(self, which: int) -> None:
        slot, epoch = self._bar(which)
        if slot < 0:
            return
        self._call("fssdp_barrier", self._pb(), self.flags_off, self.rank, self.world, slot,
               C.c_uint32(epoch), self._stream())

    def phase_combine(self) -> torch.Tensor:
        y = torch.empty(self.T, self.g.d_model, dtype=torch.bfloat16, device=self.dev)
        self._call("fssdp_combine", ops._ptr(self.slot_dest), ops._ptr(self.slot_pos),
               ops._ptr(self.topk_w), self.T, self.g.d_model, self.g.top_k, self._pb(),
               self.off["y"], ops._ptr(y), ops._ptr(self.y_slots), self._stream())
        return y

    # ------------------------------------------------------------ backward phases
    def phase_dispatch_grad(self, dy: torch.Tensor) -> None:
        if dy.shape != (self.T, self.g.d_model) or dy.dtype != torch.bfloat16:
            raise DimensionError("dy must match the forward output ([T, d] bf16)")
        self.dy = dy.contiguous()
        t = self.tables
        slot, epoch = self._bar(BAR_DGRAD)
        self._call("fssdp_dispatch_grad", ops._ptr(self.dy), ops._ptr(self.slot_dest),
               ops._ptr(self.slot_pos), ops._ptr(self.topk_w), self.T, self.g.d_model,
               self.g.top_k, self._pb(), self.off["y"], ops._ptr(self.y_slots),
               self.off["dyrecv"],
               ops._ptr(None if self._late_dots else self.slot_grad),
               ops._ptr(self.dlogit if self._early_gate else None),
               self._tab("zero_rows"), self.g.num_experts if self._local_gemm else t.n_zero,
               self.flags_off, self.rank, self.world, slot, C.c_uint32(epoch),
               C.c_void_p(self.grid_counter.data_ptr() + 4), self._stream())

    def phase_experts_bwd(self) -> None:
        self.phase_bwd_shared()
        self.phase_bwd_rest()

    def phase_bwd_shared(self) -> None:
        """dH -> dA (all slots), then the weight grads of the slots SpRS reduces."""
        f, d, n1 = self.g.d_ff, self.g.d_model, self.g.n1
        self._gemm("dgrad2", self.dyrecv, False, self.w2_view, True, self.da, n1, self.epi_dgrad2,
                   aux=self.gprime)
        grads2d = self.grads.view(-1)
        self._gemm("wgrad1", self.da, True, self.xrecv, True, grads2d, d, self.epi_wgrad,
                   part="shared")
        self._gemm("wgrad2", self.dyrecv, True, self.h, True, grads2d, f, self.epi_wgrad,
                   part="shared")

    def phase_bwd_rest(self) -> None:
        """dXe and the weight grads of the slots no other rank holds."""
        self.phase_dgrad1()
        self.phase_wgrad_rest()

    def phase_dgrad1(self) -> None:
        self._gemm("dgrad1", self.da, False, self.w1_view, True, self.dxe, self.g.d_model,
                   ops.EPI_BF16)

    def phase_wgrad_rest(self) -> None:
        f, d = self.g.d_ff, self.g.d_model
        grads2d = self.grads.view(-1)
        self._gemm("wgrad1", self.da, True, self.xrecv, True, grads2d, d, self.epi_wgrad,
                   part="rest")
        self._gemm("wgrad2", self.dyrecv, True, self.h, True, grads2d, f, self.epi_wgrad,
                   part="rest")

    # dx_event: recorded right after the dX combine on the stream that ran it — dx is final
    # there, well before backward() returns (the remaining wgrads, SpRS and the end barrier
    # follow): a caller can stream dx out (or into the previous layer's backward) from it
    dx_event = None

    def phase_combine_dx(self, dx: torch.Tensor | None = None) -> torch.Tensor:
        dx = self._combine_dx(dx)
        if self.dx_event is None:
            self.dx_event = torch.cuda.Event()
        self.dx_event.record(torch.cuda.current_stream(self.dev))
        return dx

    def _combine_dx(self, dx: torch.Tensor | None = None) -> torch.Tensor:
        if dx is None:
            dx = torch.empty(self.T, self.g.d_model, dtype=torch.bfloat16, device=self.dev)
        if self._late_dots:
            self._call("fssdp_combine_dx_dots", ops._ptr(self.slot_dest), ops._ptr(self.slot_pos),
                       ops._ptr(self.topk_idx), ops._ptr(self.topk_w), ops._ptr(self.dy),
                       ops._ptr(self.y_slots), self.off["y"], ops._ptr(self.wg), self.T,
                       self.g.d_model, self.g.num_experts, self.g.top_k, self._pb(),
                       self.off["dxe"], ops._ptr(self.slot_grad), ops._ptr(self.dlogit),
                       ops._ptr(dx), self._stream())
            return dx
        self._call("fssdp_combine_dx", ops._ptr(self.slot_dest), ops._ptr(self.slot_pos),
               ops._ptr(self.topk_idx), ops._ptr(self.topk_w), ops._ptr(self.slot_grad),
               ops._ptr(self.wg), self.T, self.g.d_model, self.g.num_experts, self.g.top_k,
               self._pb(), self.off["dxe"], ops._ptr(None if self._early_gate else self.dlogit),
               ops._ptr(dx), self._stream())
        return dx

    # dWg all-reduce (the gate is replicated, its gradient data-parallel): the partials in
    # the heap, summed in rank order over P2P right after the step's end barrier
    # (fssdp_sum_peers: bit-identical on every rank, no NCCL call in the step).
    # FSSDP_P2P_GATE_REDUCE=0: the NCCL all-reduce in reduce_gate_grad() instead
    P2P_GATE_REDUCE = os.environ.get("FSSDP_P2P_GATE_REDUCE", "1") != "0"
    P2P_GATE_REDUCE_EMULATED = False  # tests: the same over emulated ranks (lockstep)

    @property
    def _p2p_gate_reduce(self) -> bool:
        return self.P2P_GATE_REDUCE and self.world > 1 and (
            self.group.mode == "dist" or self.P2P_GATE_REDUCE_EMULATED)

    def phase_gate_wgrad(self) -> None:
        out = self.dwg
        if self._p2p_gate_reduce:
            self._gpar ^= 1
            out = self.dwg_part[self._gpar]
        if self._wg_tc:
            self._call("fssdp_gate_wgrad_tc", ops._ptr(self.x), ops._ptr(self.topk_idx),
                       ops._ptr(self.dlogit), self.T, self.g.d_model, self.g.num_experts,
                       self.g.top_k, ops._ptr(self.wg_ws), self.wg_ws.numel(),
                       ops._ptr(out), self._stream())
            return
        self._call("fssdp_gate_wgrad", ops._ptr(self.x), ops._ptr(self.topk_idx),
               ops._ptr(self.dlogit), self.T, self.g.d_model, self.g.num_experts, self.g.top_k,
               ops._ptr(self.wg_ws), ops._ptr(out), self._stream())

    def phase_gate_reduce(self) -> None:
        """dWg = sum over ranks of the partials (after a barrier that every rank's gate
        backward precedes).  The parity double buffer keeps a fast rank's next partial off
        the one its peers may still be reading."""
        if not self._p2p_gate_reduce:
            return
        E, d = self.g.num_experts, self.g.d_model
        self._call("fssdp_sum_peers", self._pb(), self.world,
                   self.off["dwgp"] + self._gpar * E * d * 4, E * d, ops._ptr(self.dwg),
                   self._stream())

    def phase_sprs(self) -> None:
        n = self.tables.n_sprs_jobs
        if n == 0:
            return
        self._timed("sprs", lambda: N.call(
            "fssdp_sprs", self._pb(), self.rank, self.off["grads"], self.off["stage"],
            self.g.slot_grad_elems, self.g.grad_elem_bytes, self._tab("sprs_jobs"), n,
            self._tab("sprs_srcs"),
            self._stream()))

    # ------------------------------------------------------------ one rank per process
    def forward(self, x: torch.Tensor) -> torch.Tensor:
        self._cs = C.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)
        try:
            return self._forward(x)
        finally:
            self._cs = None

    # planning-gap probe (bench.py): two CUDA events per step around the host planning
    # gap, from the end of the count all-gather to the start of the dispatch
    gap_events = None

    # single rank: the gate writes the dispatch tables itself (the placement cannot change),
    # so the dispatch runs while the host plans (FSSDP_LOCAL_DISPATCH=0 disables)
    LOCAL_DISPATCH = os.environ.get("FSSDP_LOCAL_DISPATCH", "1") != "0"
    # single rank: the gate's last CTA also writes the six GEMM tables from its totals
    # (byte-equal to the host builder's), so fwd1/fwd2 are queued before the host plan
    # instead of waiting for it (device timeline: fwd1 started 34 us after the dispatch,
    # waiting for the plan's table upload; as a separate single-thread kernel the tables
    # themselves took 17 us).  FSSDP_LOCAL_GEMM=0: the GEMMs wait for the host tables
    LOCAL_GEMM_TABLES = os.environ.get("FSSDP_LOCAL_GEMM", "1") != "0"

    @property
    def _local_gemm(self) -> bool:
        return self.LOCAL_GEMM_TABLES and self.LOCAL_DISPATCH and self.world == 1

    def _forward(self, x: torch.Tensor) -> torch.Tensor:
        self.phase_publish()
        self.phase_prefetch()
        self.phase_gate(x)
        self.phase_counts()
        if self.gap_events is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
            self.gap_events.append((e0, None))  # closed after the table upload
        fwd_queued = False
        if self.LOCAL_DISPATCH and self.world == 1:
            self._push_counts()
            self.phase_dispatch(n_zero=self.g.num_experts)  # one {row, count} per expert
            if self._local_gemm:
                # the GEMM tables too came from the device (the gate wrote them): the forward
                # GEMMs are queued before the host plan (which then overlaps them)
                E = self.g.num_experts
                self.gemm = dict(getattr(self, "gemm", None) or {})
                self.gemm["fwd1"] = (E, self.g.n1 // self._bn["fwd1"], -1)
                self.gemm["fwd2"] = (E, self.g.d_model // 256, -1)
                self.phase_experts_fwd()
                fwd_queued = True
            self.phase_plan(pushed=True)
        elif self._fused_plan_ok():
            self.phase_plan_dispatch()
        else:
            self.phase_plan(dispatch=True)
            if not self._dispatched:
                self.phase_dispatch()
        self._mark("dispatch_launched")
        if not fwd_queued:
            self.phase_spag()  # only fwd1 reads the replicas: the dispatch overlaps the early SpAG
            self.phase_experts_fwd()
        self._finish_plan()  # Python bookkeeping of the plan, once the GEMMs are queued
        self.phase_barrier(BAR_Y)
        return self.phase_combine()

    def backward(self, dy: torch.Tensor, rematerialize: bool | None = None) -> torch.Tensor:
        self._cs = C.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)
        try:
            return self._backward(dy, rematerialize)
        finally:
            self._cs = None

    def _backward(self, dy: torch.Tensor, rematerialize: bool | None) -> torch.Tensor:
        self.phase_dispatch_grad(dy)
        main = torch.cuda.current_stream(self.dev)
        if self._early_gate:
            gs = self._gate_stream()
            gs.wait_stream(main)
            with self._on(gs):
                self.phase_gate_wgrad()
        remat = self.planner.policy.rematerialize if rematerialize is None else rematerialize
        if remat:
            self.phase_spag(refetch_early=True)
        # Three streams.  main: dgrad2, the shared-slot wgrads, dgrad1, the remaining
        # wgrads.  side (replicas only): SpRS as soon as every rank has the weight grads of
        # its shared slots.  dx: the dX combine and the gate backward as soon as every rank
        # has its dXe rows — both HBM/NVLink-bound, they run beside the tensor-bound wgrads
        # (disjoint buffers).  The decision is global (same plan on every rank), so every
        # rank joins the same barriers.
        replicas = self.decision.target != self.decision.base
        self.phase_bwd_shared()
        if replicas:
            side = self._side_stream()
            side.wait_stream(main)
            with self._on(side):
                self.phase_barrier(BAR_SPRS)
                self.phase_sprs()
        self.phase_dgrad1()
        dx = torch.empty(self.T, self.g.d_model, dtype=torch.bfloat16, device=self.dev)
        dxs = self._dx_stream()
        dxs.wait_stream(main)
        mode = self.DX_MODE
        if mode == "dx_first":  # dX combine on the main stream, the gate backward beside
            self.phase_barrier(BAR_DX)
            self.phase_combine_dx(dx)
            if not self._early_gate:
                dxs.wait_stream(main)
                with self._on(dxs):
                    self.phase_gate_wgrad()
        elif mode != "serial":
            with self._on(dxs):
                self.phase_barrier(BAR_DX)
                self.phase_combine_dx(dx)
                if not self._early_gate and mode != "gate_end":
                    self.phase_gate_wgrad()
        self.phase_wgrad_rest()
        if mode == "serial":
            self.phase_barrier(BAR_DX)
            self.phase_combine_dx(dx)
        if not self._early_gate and mode in ("serial", "gate_end"):
            self.phase_gate_wgrad()
        main.wait_stream(dxs)
        if self._early_gate:
            main.wait_stream(self._gate_stream())
        if replicas:
            main.wait_stream(side)
        self.phase_barrier(BAR_END)
        self.phase_gate_reduce()
        return dx

    @contextlib.contextmanager
    def _on(self, stream: torch.cuda.Stream):
        """Launch the enclosed phases on `stream` (torch's current stream and _stream())."""
        prev = self._cs
        self._cs = C.c_void_p(stream.cuda_stream)
        try:
            with torch.cuda.stream(stream):
                yield
        finally:
            self._cs = prev

    def _dx_stream(self) -> torch.cuda.Stream:
        if getattr(self, "_dxs", None) is None:
            self._dxs = torch.cuda.Stream(device=self.dev)
        return self._dxs

    def _gate_stream(self) -> torch.cuda.Stream:
        if getattr(self, "_gs", None) is None:
            self._gs = torch.cuda.Stream(device=self.dev)
        return self._gs

    def _side_stream(self) -> torch.cuda.Stream:
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=self.dev)
        return self._side

    def reduce_gate_grad(self, pg=None) -> None:
        """dWg is data-parallel (the gate is replicated).  By default the backward already
        summed it over P2P (phase_gate_reduce); else one small NCCL all-reduce."""
        if self.world > 1 and self.group.mode == "dist" and not self._p2p_gate_reduce:
            import torch.distributed as dist

            dist.all_reduce(self.dwg, group=pg)


def create_layer(d_model: int, d_ff: int, num_experts: int, top_k: int, max_tokens: int,
                 policy, *, rank: int = 0, world: int = 1, device="cuda", seed: int = 0,
                 peer_bw: float = 770e9, attn_fwd_time: float = 1e-3,
                 per_token_expert_time: float | None = None, pg=None,
                 activation: str = "gelu", record_trace: bool = False,
                 optimizer: bool = False, grad_dtype: str = "bf16") -> FssdpMoE:
    """One rank per process: heap layout, IPC peer group (world > 1), planner, layer.
    optimizer=True reserves the owned shards' AdamW state in the heap (optim.FssdpAdam);
    grad_dtype "bf16" / "fp32" weight-gradient buffers (LayerGeometry.grad_dtype)."""
    (layer,) = create_model(1, d_model, d_ff, num_experts, top_k, max_tokens, policy, rank=rank,
                            world=world, device=device, seed=seed, peer_bw=peer_bw,
                            attn_fwd_time=attn_fwd_time,
                            per_token_expert_time=per_token_expert_time, pg=pg,
                            activation=activation, record_trace=record_trace,
                            optimizer=optimizer, grad_dtype=grad_dtype)
    return layer


def replica_slots(planner: FssdpPlanner) -> int:
    """Replica slots per layer and rank: the planner's m (capacity_override, else
    free_bytes_per_device // expert_bytes, else every expert — engine.py:389-402); none for
    EP or when nothing can be fetched (t or m <= 0: FSSDP degenerates to EP)."""
    if planner.policy.kind != PolicyKind.FSSDP or planner.t <= 0 or planner.m <= 0:
        return 0
    return int(planner.m)


def layer_geometries(planner: FssdpPlanner, d_model: int, d_ff: int, top_k: int,
                     max_tokens: int, m: int, activation: str = "gelu",
                     optimizer: bool = False, grad_dtype: str = "bf16") -> list:
    """Per-layer geometry under the planner's current ShardPlan (even or heterogeneous):
    slot capacity = the most experts any rank owns in that layer + m replica slots.  With
    re-sharding on, a layer may later own up to a device's whole share across layers
    (ShardPlan slot totals, placement.py:240-250): the capacity covers that."""
    geoms = []
    reshard = planner.policy.reshard_interval > 0
    for base in planner.shards.per_layer:
        D, E = base.num_devices, base.num_chunks
        owned_max = max(len(base.chunks_on(d)) for d in range(D))
        if reshard:
            owned_max = min(E, max(owned_max, -(-(E * len(planner.shards.per_layer)) // D)))
        geoms.append(LayerGeometry(d_model, d_ff, E, top_k, max_tokens, D,
                                   min(E, owned_max + max(0, m)), activation, owned_max, reshard,
                                   optimizer, grad_dtype=grad_dtype))
    return geoms


def create_model(num_layers: int, d_model: int, d_ff: int, num_experts: int, top_k: int,
                 max_tokens: int, policy, *, rank: int = 0, world: int = 1, device="cuda",
                 seed: int = 0, peer_bw: float = 770e9, attn_fwd_time: float = 1e-3,
                 per_token_expert_time: float | None = None, pg=None,
                 activation: str = "gelu", load_profile=None, record_trace: bool = False,
                 optimizer: bool = False, grad_dtype: str = "bf16") -> list:
    """num_layers FSSDP MoE layers sharing one planner (one iteration = every layer's
    forward, then backward in reverse, then planner.finish()) and one symmetric heap.
    grad_dtype: "bf16" (default; the reference's grad_bytes = param bytes) or "fp32".
    load_profile [L, E] (expected per-expert loads): the initial ShardPlan comes from
    heterogeneous_sharding (Alg. 2, planner.py:302-385) instead of the even split."""
    from .engine import ModelConfig
    from .planner import GlobalLoadProfile, heterogeneous_sharding
    from .topology import ClusterTopology

    nm = 3 if activation == "swiglu" else 2
    topo = ClusterTopology.for_nvswitch(world, peer_bw)
    if per_token_expert_time is None:
        per_token_expert_time = 2.0 * nm * d_model * d_ff / 1381.7e12
    cfg = ModelConfig(num_layers, num_experts, 2 * nm * d_model * d_ff, 2 * d_model,
                      attn_fwd_time, per_token_expert_time)
    if not 1 <= num_layers <= 8:
        raise DimensionError("1 <= num_layers <= 8 (8 barrier slots per layer in the flag pad)")
    planner = FssdpPlanner(cfg, topo, policy, record_trace)
    if load_profile is not None:
        planner.shards = heterogeneous_sharding(
            GlobalLoadProfile(np.asarray(load_profile, dtype=np.float64)), planner.t, topo)
    geoms = layer_geometries(planner, d_model, d_ff, top_k, max_tokens, replica_slots(planner),
                             activation, optimizer, grad_dtype)
    layout = HeapLayout()
    # owned slots per layer; replica slots per layer (retain) or one shared set (remat)
    geoms = model_regions(layout, geoms, policy.rematerialize)
    group = PeerGroup(layout, rank, world, device, "dist", pg=pg)
    return [FssdpMoE(geom, group, planner, li, seed, prefix=f"L{li}.")
            for li, geom in enumerate(geoms)]


class FssdpMoEFunction(torch.autograd.Function):
    """autograd wrapper: y = layer(x); expert grads land in the layer's heap (SpRS-reduced
    on their owners), the gate grad in layer.dwg."""

    @staticmethod
    def forward(ctx, x, layer):
        ctx.layer = layer
        return layer.forward(x)

    @staticmethod
    def backward(ctx, dy):
        dx = ctx.layer.backward(dy.to(torch.bfloat16).contiguous())
        ctx.layer.planner.finish()
        return dx, None


def run_lockstep_forward(layers: list, xs: list) -> list:
    """Emulated multi-rank forward: every phase on every logical rank before the next."""
    for ly in layers:
        ly.phase_publish()
    for ly in layers:
        ly.phase_prefetch()
    for ly, x in zip(layers, xs):
        ly.phase_gate(x)
    for ly in layers:
        ly.phase_counts()
    for ly in layers:
        ly.phase_plan()
    for ly in layers:
        ly.phase_dispatch()
        ly._finish_plan()
    for ly in layers:
        ly.phase_spag()
    for ly in layers:
        ly.phase_experts_fwd()
    return [ly.phase_combine() for ly in layers]


def run_lockstep_backward(layers: list, dys: list, rematerialize: bool = False) -> list:
    for ly, dy in zip(layers, dys):
        ly.phase_dispatch_grad(dy)
    if rematerialize:
        for ly in layers:
            ly.phase_spag(refetch_early=True)
    for ly in layers:
        ly.phase_bwd_shared()
    for ly in layers:
        ly.phase_bwd_rest()
    dxs = [ly.phase_combine_dx() for ly in layers]
    for ly in layers:
        ly.phase_gate_wgrad()
    for ly in layers:
        ly.phase_gate_reduce()
    for ly in layers:
        ly.phase_sprs()
    return dxs
