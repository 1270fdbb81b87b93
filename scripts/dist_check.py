"""Multi-process FSSDP parity check (one rank per GPU, CUDA-IPC peer heaps, device barriers).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/dist_check.py

Every rank runs the FSSDP layer on its token shard for a few iterations; rank 0 re-runs
all tokens through a single-rank layer and checks y/dx bit-exactly and every owner's
SpRS-reduced expert gradient within fp32 tolerance.  Prints "DIST OK" on success.
"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2502_02581_b200 as F  # noqa: E402
from paper_2502_02581_b200.layer import create_layer  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    E, d, f, k, Tr = 16, 512, 1024, 2, 1024
    pol = F.Policy(F.PolicyKind.FSSDP, overlap_override=6, capacity_override=2,
                   reshard_interval=0)
    layer = create_layer(d, f, E, k, Tr, pol, rank=rank, world=world, device=dev, seed=5,
                         per_token_expert_time=1e-6)
    p = 1.0 / np.arange(1, E + 1) ** 1.3
    bias = torch.tensor(np.log(p[np.random.default_rng(1).permutation(E)] / p.sum()),
                        dtype=torch.float32, device=dev)
    layer.gate_bias.copy_(bias)
    single = None
    if rank == 0:
        single = create_layer(d, f, E, k, Tr * world, F.Policy(F.PolicyKind.EP), rank=0, world=1,
                              device=dev, seed=5)
        single.gate_bias.copy_(bias)
    ok = True
    replicas = 0
    for it in range(4):
        g = torch.Generator(device=dev).manual_seed(100 + it)
        x = torch.randn(world * Tr, d, device=dev, generator=g).bfloat16()
        dy = (torch.randn(world * Tr, d, device=dev, generator=g) * 0.05).bfloat16()
        xs, dys = x[rank * Tr:(rank + 1) * Tr], dy[rank * Tr:(rank + 1) * Tr]
        y = layer.forward(xs.contiguous())
        dx = layer.backward(dys.contiguous())
        layer.reduce_gate_grad()
        layer.planner.finish()
        torch.cuda.synchronize()
        replicas += len(layer.decision.target.entries) - E
        ys = [torch.empty_like(y) for _ in range(world)]
        dxs = [torch.empty_like(dx) for _ in range(world)]
        dist.all_gather(ys, y)
        dist.all_gather(dxs, dx)
        # owners' reduced grads -> rank 0
        grads = {}
        for e in range(E):
            owner = layer.decision.base.owner(e)
            buf = torch.empty(2 * d * f, device=dev, dtype=torch.float32)
            if rank == owner:
                g1, g2 = layer.expert_grad(e)
                buf.copy_(torch.cat([g1.reshape(-1), g2.reshape(-1)]))
            dist.broadcast(buf, src=owner)
            grads[e] = buf
        if rank == 0:
            y1 = single.forward(x)
            dx1 = single.backward(dy)
            single.planner.finish()
            torch.cuda.synchronize()
            same_y = torch.equal(torch.cat(ys), y1)
            same_dx = torch.equal(torch.cat(dxs), dx1)
            worst, grads_ok = 0.0, True
            for e in range(E):
                g1, g2 = single.expert_grad(e)
                ref = torch.cat([g1.reshape(-1), g2.reshape(-1)]).float()
                diff = (grads[e] - ref).abs()
                err = diff.max().item() / (ref.abs().max().item() + 1e-12)
                worst = max(worst, err)
                if g1.dtype == torch.bfloat16:  # partials and sum rounded (tests/_torch_ref)
                    bound = 2.0 ** -6 * ref.abs() + 2.0 ** -8 * ref.abs().max()
                    grads_ok = grads_ok and bool((diff <= bound).all())
                else:
                    grads_ok = grads_ok and err < 1e-4
            dwg_ok = torch.allclose(layer.dwg, single.dwg, rtol=1e-4, atol=1e-6)
            print(f"iter {it}: y bit-exact {same_y}, dx bit-exact {same_dx}, worst grad rel err "
                  f"{worst:.2e}, dWg ok {dwg_ok}, replicas {len(layer.decision.target.entries) - E}",
                  flush=True)
            ok = ok and same_y and same_dx and grads_ok and dwg_ok
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.broadcast(flag, src=0)
    if rank == 0:
        print("DIST OK" if flag.item() and replicas > 0 else f"DIST FAIL (replicas={replicas})",
              flush=True)
    dist.barrier()
    dist.destroy_process_group()
    if not flag.item():
        sys.exit(1)


if __name__ == "__main__":
    main()
