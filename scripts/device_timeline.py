"""Device-side kernel timeline of the bench workload (torch.profiler / CUPTI activity
records: GPU timestamps of every kernel, no CUDA events in the stream).

    python scripts/device_timeline.py [--config cfg2] [--steps 3] [--out gpurun_out/tl.json]

Prints, for the last profiled step, every kernel (start/end relative to the step's first
kernel, µs) and the GPU idle gaps on the critical stream, plus totals."""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--e2e", action="store_true",
                    help="host inputs: x, dy H2D one step ahead, y and dx D2H (bench e2e)")
    args = ap.parse_args()
    bench.select_config(args.config)
    import paper_2502_02581_b200 as F
    from paper_2502_02581_b200.layer import create_layer

    C = bench.CFG2
    T = C["tokens_per_gpu"]
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    if world > 1:  # torchrun: one rank per GPU, each profiles its own device
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    layer = create_layer(C["d_model"], C["d_ff"], C["num_experts"], C["top_k"], T,
                         F.Policy(F.PolicyKind.FSSDP, **bench.POLICY), rank=rank, world=world,
                         device=dev, seed=1234, activation=C["activation"])
    E = C["num_experts"]
    p = 1.0 / np.arange(1, E + 1) ** bench.ZIPF_S
    p = p[np.random.default_rng(42).permutation(E)]
    layer.gate_bias.copy_(torch.tensor(np.log(p / p.sum()), dtype=torch.float32))
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    xs = [torch.randn(T, C["d_model"], device=dev, generator=g).bfloat16() for _ in range(4)]
    dys = [(torch.randn(T, C["d_model"], device=dev, generator=g) * 0.05).bfloat16()
           for _ in range(4)]

    def step(i):
        layer.forward(xs[i % 4])
        layer.backward(dys[i % 4])
        layer.reduce_gate_grad()
        layer.planner.finish()

    if args.e2e:  # the bench's e2e pipeline (bench.py run_ours, e2e section)
        xh = [x.cpu().pin_memory() for x in xs[:2]]
        dyh = [t.cpu().pin_memory() for t in dys[:2]]
        yh = [torch.empty_like(xh[0]).pin_memory() for _ in range(2)]
        dxh = [torch.empty_like(xh[0]).pin_memory() for _ in range(2)]
        xb = [torch.empty_like(xs[0]) for _ in range(2)]
        dyb = [torch.empty_like(dys[0]) for _ in range(2)]
        cs, ds = torch.cuda.Stream(), torch.cuda.Stream()
        main = torch.cuda.current_stream()
        in_ev = [torch.cuda.Event() for _ in range(2)]
        done_ev = [torch.cuda.Event() for _ in range(2)]
        fwd_ev = [torch.cuda.Event() for _ in range(2)]
        for ev in done_ev:
            ev.record(main)
        state = {"prev": None}

        def prefetch(i):
            b = i % 2
            with torch.cuda.stream(cs):
                cs.wait_event(done_ev[b])
                xb[b].copy_(xh[i % 2], non_blocking=True)
                dyb[b].copy_(dyh[i % 2], non_blocking=True)
                in_ev[b].record(cs)

        def d2h(t, host, ev):
            with torch.cuda.stream(ds):
                ds.wait_event(ev)
                host.copy_(t, non_blocking=True)
                t.record_stream(ds)

        prefetch(0)

        def step(i):  # noqa: F811
            b = i % 2
            main.wait_event(in_ev[b])
            y = layer.forward(xb[b])
            fwd_ev[b].record(main)
            prefetch(i + 1)
            if state["prev"] is not None:
                d2h(*state["prev"])
            d2h(y, yh[b], fwd_ev[b])
            dx = layer.backward(dyb[b])
            layer.planner.finish()
            done_ev[b].record(main)
            state["prev"] = (dx, dxh[b], done_ev[b])

    for i in range(5):
        step(i)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(args.steps):
            step(i)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    # memcpy records carry "Memcpy" names; kernels the rest
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda t: t[0])
    # split into steps at each gate launch
    starts = [i for i, k in enumerate(ks) if "gate_topk" in k[2]]
    last = ks[starts[-1]:] if starts else ks
    t0 = last[0][0]
    rows = [(round(a - t0, 2), round(b - t0, 2), n[:70]) for a, b, n in last]
    busy_end, gaps = rows[0][0], 0.0
    for a, b, n in rows:
        if a > busy_end:
            gaps += a - busy_end
        busy_end = max(busy_end, b)
    step_us = (ks[starts[-1]][0] - ks[starts[-2]][0]) if len(starts) > 1 else None
    lines = [f"{a:9.2f} {b:9.2f} {b - a:8.2f}  {n}" for a, b, n in rows]
    lines.append(json.dumps({"rank": rank, "step_us": step_us, "idle_gaps_us": round(gaps, 2),
                             "kernels": len(rows)}))
    if world == 1:
        print("\n".join(lines))
    else:  # one file per rank (gpurun_out/tl_dev_n{world}_r{rank}.txt)
        with open(f"gpurun_out/tl_dev_n{world}_r{rank}.txt", "w") as fh:
            fh.write("\n".join(lines) + "\n")
    if args.out:
        with open(args.out, "w") as fh:
            json.dump({"rows": rows, "step_us": step_us, "idle_gaps_us": gaps}, fh)


if __name__ == "__main__":
    main()
