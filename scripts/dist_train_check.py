"""Multi-process training-loop check of the owner-update epochs (one rank per GPU):

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/dist_train_check.py

Every iteration: forward, backward, gate all-reduce, AdamW step on the owned shards
(FssdpAdam).  Rank 1 delays its optimizer step (a device sleep before it), so the other
ranks start their next forward — and their early copy-engine SpAG of rank 1's shards —
while rank 1 is still updating them.  After every forward, every replica slot must be a
byte-exact copy of its owner's CURRENT (updated) shard: the early copies waited for the
owner's published epoch.  Prints "TRAIN OK".  FSSDP_EPOCHS=0 (negative control) drops the
epochs; the check then reports torn/stale replicas."""

import hashlib
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2502_02581_b200 as F  # noqa: E402
from paper_2502_02581_b200.layer import create_layer  # noqa: E402


def digest(t: torch.Tensor) -> str:
    return hashlib.sha256(t.contiguous().view(torch.uint8).cpu().numpy().tobytes()).hexdigest()


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    E, d, f, k, T = 16, 1024, 4096, 2, 16384
    pol = F.Policy(F.PolicyKind.FSSDP, overlap_override=8, capacity_override=4,
                   reshard_interval=0)
    layer = create_layer(d, f, E, k, T, pol, rank=rank, world=world, device=dev, seed=9,
                         optimizer=True)
    p = 1.0 / np.arange(1, E + 1) ** (1.2 if world > 2 else 1.6)  # replicas at N=2 too
    layer.gate_bias.copy_(torch.tensor(np.log(p[np.random.default_rng(3).permutation(E)] / p.sum()),
                                       dtype=torch.float32))
    opt = F.FssdpAdam([layer], lr=1e-3)
    bad = checked = early = 0
    for it in range(12):
        g = torch.Generator(device=dev).manual_seed(50 + 7 * it + rank)
        x = torch.randn(T, d, device=dev, generator=g).bfloat16()
        dy = (torch.randn(T, d, device=dev, generator=g) * 0.05).bfloat16()
        layer.forward(x)
        torch.cuda.synchronize()
        early += layer.pre_tables.n_spag if layer.pre_tables is not None else 0
        # every replica slot vs its owner's current shard
        t = layer.tables
        mine = {int(e): digest(layer.slot_params(s)) for s, e in enumerate(t.slot_expert)}
        allm = [None] * world
        dist.all_gather_object(allm, mine)
        dec = layer.decision
        for e, h in mine.items():
            o = dec.base.owner(e)
            if o != rank:
                checked += 1
                bad += int(allm[o][e] != h)
        layer.backward(dy)
        layer.reduce_gate_grad()
        layer.planner.finish()
        if rank == 1:
            torch.cuda._sleep(200_000_000)  # ~0.1 s: the owner's update runs late
        opt.step()
    tot = torch.tensor([bad, checked, early], device=dev)
    dist.all_reduce(tot)
    if rank == 0:
        ok = tot[0].item() == 0 and tot[1].item() > 0 and tot[2].item() > 0
        print(f"replica checks {tot[1].item()}, early copy-engine copies {tot[2].item()}, "
              f"stale/torn {tot[0].item()}", flush=True)
        print("TRAIN OK" if ok else "TRAIN FAIL", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    if tot[0].item():
        sys.exit(1)


if __name__ == "__main__":
    main()
