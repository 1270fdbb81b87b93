"""The cfg2 FSSDP layer on N real GPUs driven from ONE process, phase by phase — for ncu's
per-kernel NVLink counters (ncu must not wrap a multi-rank torchrun command; here every
kernel is an ordinary launch of one process, replayable).

    python scripts/nvlink_layer.py [--gpus N] [--iters 4]
    ncu --metrics gpu__time_duration.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum \
        -k regex:"dispatch|combine|spag|sprs|gather" python scripts/nvlink_layer.py

Rank r's symmetric heap lives on GPU r (peer access enabled, peer table of raw device
pointers — the same addressing the IPC-mapped multi-process path uses), so every P2P
kernel moves its bytes over NVLink.  Device barriers are disabled (PeerGroup "emulated");
instead every phase of every rank finishes (all devices synchronized) before the next
phase starts, so the data dependencies the barriers enforce hold.  The early SpAG runs on
the SM copy kernel here (FSSDP_PRE_W1_CE=0 / FSSDP_PRE_W2_CE=0): copy-engine transfers are
not kernels and carry no ncu counters.  Prints one JSON line with each rank's plan and
the algorithmic bytes the counters are compared against (bench.py a2a_stats / spag_traffic).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("FSSDP_PRE_W1_CE", "0")
os.environ.setdefault("FSSDP_PRE_W2_CE", "0")

import numpy as np  # noqa: E402
import torch  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))

import paper_2502_02581_b200 as F  # noqa: E402
from paper_2502_02581_b200.comm import Heap, HeapLayout, PeerGroup  # noqa: E402
from paper_2502_02581_b200.layer import FssdpMoE, LayerGeometry, default_slots  # noqa: E402
from nvlink_probe import enable_peers  # noqa: E402


def sync_all(n):
    for d in range(n):
        torch.cuda.synchronize(d)


def each(layers, fn, n):
    out = []
    for ly in layers:
        with torch.cuda.device(ly.dev):
            out.append(fn(ly))
    sync_all(n)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=torch.cuda.device_count())
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--tokens", type=int, default=16384)
    args = ap.parse_args()
    n = args.gpus
    enable_peers(n)
    E, d, f, k, T = 16, 1024, 4096, 2, args.tokens
    pol = F.Policy(F.PolicyKind.FSSDP, overlap_override=8, capacity_override=4)
    geom = LayerGeometry(d, f, E, k, T, n, default_slots(E, n, 4), "gelu")
    layout = HeapLayout()
    geom.add_regions(layout, "L0.")
    heaps = [Heap(layout.size, f"cuda:{r}") for r in range(n)]
    groups = [PeerGroup(layout, r, n, f"cuda:{r}", "emulated", heaps=heaps) for r in range(n)]
    topo = F.ClusterTopology.for_nvswitch(n, 774e9)
    cfg = F.ModelConfig(1, E, geom.expert_bytes, 2 * d, 1e-3, 2.0 * 2 * d * f / 1381.7e12)
    p = 1.0 / np.arange(1, E + 1) ** 1.2
    p = p[np.random.default_rng(42).permutation(E)]
    layers = []
    for r in range(n):
        with torch.cuda.device(r):
            ly = FssdpMoE(geom, groups[r], F.FssdpPlanner(cfg, topo, pol), 0, 1234)
            ly.gate_bias.copy_(torch.tensor(np.log(p / p.sum()), dtype=torch.float32))
            layers.append(ly)
    xs, dys = [], []
    for r in range(n):
        g = torch.Generator(device=f"cuda:{r}").manual_seed(1000 + r)
        xs.append(torch.randn(T, d, device=f"cuda:{r}", generator=g).bfloat16())
        dys.append((torch.randn(T, d, device=f"cuda:{r}", generator=g) * 0.05).bfloat16())
    for _ in range(args.iters):
        each(layers, lambda ly: ly.phase_prefetch(), n)
        each(layers, lambda ly: ly.phase_gate(xs[ly.rank]), n)
        each(layers, lambda ly: ly.phase_counts(), n)
        each(layers, lambda ly: ly.phase_plan(), n)
        each(layers, lambda ly: (ly.phase_dispatch(), ly._finish_plan()), n)
        each(layers, lambda ly: ly.phase_spag(), n)
        each(layers, lambda ly: ly._launch_prefetch_w2(), n)
        each(layers, lambda ly: ly.phase_experts_fwd(), n)
        each(layers, lambda ly: ly.phase_combine(), n)
        each(layers, lambda ly: ly.phase_dispatch_grad(dys[ly.rank]), n)
        each(layers, lambda ly: ly.phase_bwd_shared(), n)
        each(layers, lambda ly: ly.phase_sprs(), n)
        each(layers, lambda ly: ly.phase_bwd_rest(), n)
        each(layers, lambda ly: ly.phase_combine_dx(), n)
        for ly in layers:
            ly.planner.finish()
    dec = layers[0].decision
    B = 2 * d
    r_ = np.asarray(dec.route, dtype=np.float64)
    mat = r_.sum(axis=1) * B
    np.fill_diagonal(mat, 0.0)
    tr, rep = F.spag_traffic(dec.base, dec.target, geom.expert_bytes)
    out = {"n_gpus": n, "config": "cfg2 (E 16, d 1024, f 4096, T 16384/GPU, t 8, m 4)",
           "replicas": len(dec.target.entries) - E,
           "a2a_bytes_out_per_rank": mat.sum(axis=1).tolist(),
           "a2a_bytes_in_per_rank": mat.sum(axis=0).tolist(),
           "spag_bytes_in_per_rank": tr.data.sum(axis=0).tolist(),
           "spag_bottleneck_bytes": rep.bottleneck_bytes,
           "sprs_bytes_fp32_in_per_rank": (2 * tr.data.sum(axis=0)).tolist(),
           "early_copies": [int(ly.pre_tables.n_spag) if ly.pre_tables is not None else 0
                            for ly in layers],
           "late_copies": [int(ly.tables.n_spag) for ly in layers]}
    print("NVLINK_LAYER " + json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
