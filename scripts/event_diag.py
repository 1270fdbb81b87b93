"""Why do per-kernel CUDA events (bench.py's instrumented pass) read longer than the
uninstrumented step?  Alternates plain and instrumented passes of the cfg2 N=1 step,
timing each pass as a whole and sampling SM clocks during it.

    python scripts/event_diag.py [--steps 20]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2502_02581_b200 as F  # noqa: E402
from paper_2502_02581_b200.layer import create_layer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    bench.select_config("cfg2")
    C2, T = bench.CFG2, 16384
    dev = torch.device("cuda", 0)
    pol = F.Policy(F.PolicyKind.FSSDP, **bench.POLICY)
    layer = create_layer(C2["d_model"], C2["d_ff"], C2["num_experts"], C2["top_k"], T, pol,
                         rank=0, world=1, device=dev, seed=1234)
    E = C2["num_experts"]
    p = 1.0 / np.arange(1, E + 1) ** bench.ZIPF_S
    p = p[np.random.default_rng(42).permutation(E)]
    layer.gate_bias.copy_(torch.tensor(np.log(p / p.sum()), dtype=torch.float32))
    gen = torch.Generator(device=dev).manual_seed(1000)
    x = torch.randn(T, C2["d_model"], device=dev, generator=gen).bfloat16()
    dy = (torch.randn(T, C2["d_model"], device=dev, generator=gen) * 0.05).bfloat16()

    def step():
        layer.forward(x)
        layer.backward(dy)
        layer.planner.finish()

    for _ in range(5):
        step()
    torch.cuda.synchronize()

    def run(mode):
        layer.timers = {} if mode != "plain" else None
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        with bench.ClockSampler(0) as clk:
            torch.cuda.synchronize()
            s.record()
            for _ in range(args.steps):
                step()
                if mode == "inst_sync":
                    torch.cuda.synchronize()
            e.record()
            torch.cuda.synchronize()
        out = {"mode": mode, "ms_per_step": round(s.elapsed_time(e) / args.steps, 4),
               "clocks": clk.summary()}
        if layer.timers:
            tm = layer.timers
            tm.pop("marks", None)
            tm.pop("host_plan_s", None)
            per = {k: round(sum(a.elapsed_time(b) for a, b in v) / args.steps, 4) for k, v in tm.items()}
            out["gemm_ms"] = round(sum(v for k, v in per.items() if k.startswith("gemm.")), 4)
            out["kernels_ms"] = round(sum(per.values()), 4)
            out["per"] = per
        layer.timers = None
        print(out, flush=True)

    for mode in ("plain", "inst", "plain", "inst", "inst_sync", "plain"):
        run(mode)


if __name__ == "__main__":
    main()
