"""AdamW for FSSDP layers: each rank updates the expert shards it OWNS (after SpRS their
grads slots hold the fully reduced gradient) plus its replica of the dense gate.

The owned shards' fp32 master weights and both moments live in the symmetric heap next to
the parameters (LayerGeometry.optimizer), so a re-shard moves them with the parameters
(params + 6x state: the 7x expert_bytes per moved expert of moesim engine.py:233, 444-453)
and the memory follows memory_report's `optimizer_bytes = 6 x param` (engine.py:188-226).
One fused kernel per layer (fssdp_adam_step) rewrites the bf16 working copy from the
master; the next forward publishes the owner-update epoch peers' early SpAG waits for.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from .errors import ConfigError


class FssdpAdam:
    """AdamW over the owned expert shards of `layers` (one rank's FssdpMoE list) and their
    gate weights.  Call step() after backward (and the gate-gradient all-reduce)."""

    def __init__(self, layers, lr: float = 1e-4, betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 0.0, gate: bool = True):
        self.layers = list(layers)
        for ly in self.layers:
            if ly.opt_state is None:
                raise ConfigError("FssdpAdam needs layers built with optimizer=True "
                                  "(create_layer / create_model)")
        self.lr, self.betas, self.eps, self.weight_decay = lr, betas, eps, weight_decay
        self.step_count = 0
        self.gate = gate
        self._gate_state = {}
        for ly in self.layers:
            n = ly._n_owned
            st = ly.opt_state
            st["master"][:n].copy_(ly.params[:n].float())
            st["m"][:n].zero_()
            st["v"][:n].zero_()
            if gate:
                self._gate_state[id(ly)] = (torch.zeros_like(ly.wg), torch.zeros_like(ly.wg))

    def _adam(self, params, master, m, v, grads, n, stream) -> None:
        b1, b2 = self.betas
        N.call("fssdp_adam_step", C.c_void_p(0 if params is None else params.data_ptr()),
               C.c_void_p(master.data_ptr()), C.c_void_p(m.data_ptr()),
               C.c_void_p(v.data_ptr()), C.c_void_p(grads.data_ptr()),
               int(grads.dtype == torch.bfloat16), n, self.lr, b1, b2,
               self.eps, self.weight_decay, self.step_count, stream)

    @torch.no_grad()
    def step(self) -> None:
        self.step_count += 1
        for ly in self.layers:
            stream = C.c_void_p(torch.cuda.current_stream(ly.dev).cuda_stream)
            n = ly._n_owned  # owned slots are [0, n): after any re-shard of this iteration
            if n:
                st = ly.opt_state
                self._adam(ly.params, st["master"], st["m"], st["v"], ly.grads,
                           n * ly.g.slot_grad_elems, stream)
            if self.gate:
                gm, gv = self._gate_state[id(ly)]
                self._adam(None, ly.wg, gm, gv, ly.dwg, ly.wg.numel(), stream)

    def state_of(self, ly, expert: int) -> dict:
        """fp32 master / m / v of an expert this rank owns (views)."""
        s = ly._owned_expert_ids.index(expert)
        return {k: ly.opt_state[k][s] for k in ("master", "m", "v")}
