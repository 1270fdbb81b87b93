#!/usr/bin/env python
"""FSSDP MoE layer fwd+bwd throughput on B200 (BASELINE.json metric), one rank per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (configs[1], "cfg2"): a GPT-MoE layer — 16 experts, top-2, d_model 1024,
d_ff 4096 (GeLU), 16384 tokens per GPU, bf16 — under seeded Zipf(1.2)-skewed gate
loads, FSSDP policy (t=8 replicable experts, m=4 replica slots, calibration on).  A step
is one FSSDP layer fwd+bwd: early SpAG of the history-based candidate (side stream), gate,
counts all-gather, host plan (bit-exact moesim planner), SpAG of the rest, token dispatch, grouped FFN (tcgen05), combine; backward A2A, dgrad/wgrad,
dX combine + gate backward, SpRS.  Weak scaling: tokens per GPU are fixed.

Prints ONE JSON line (rank 0).  `value` = all ranks' tokens / max-over-ranks device
time with inputs resident in HBM; `e2e` = the same through FssdpMoE.forward/backward
with pinned-host inputs copied in and dx copied out inside the timed region.
`--impl reference` times the CPU oracle port of the same path (oracle/, numpy) on a
bounded token sample with all host threads.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MoE fwd+bwd tokens/s at 1/2/4/8 B200; sparse AG/RS GB/s vs NVLink peak"
# BASELINE.json configs.  cfg2 is the metric's configuration (the default bench line); the
# others are available with --config for reference measurements (one MoE layer of that
# shape; cfg3's heterogeneous sharding over 4 layers is covered by tests/test_configs_gpu.py).
# FSSDP knobs (engine.py:88-121) for cfg2: t = 8 replicable experts, m = 4 replica slots per
# GPU — chosen offline with the bit-exact planner for the lowest max/mean device load at N = 4/8.
CONFIGS = {
    "cfg1": dict(num_experts=8, top_k=2, d_model=256, d_ff=1024, tokens_per_gpu=1024,
                 activation="gelu", zipf_s=1.2,
                 policy=dict(overlap_override=4, capacity_override=2, calibration=True,
                             rematerialize=False, reshard_interval=0),
                 workload="cfg1: toy MoE layer, 8 experts top-2, d_model 256, d_ff 1024 GeLU, "
                          "1024 tokens/GPU"),
    "cfg2": dict(num_experts=16, top_k=2, d_model=1024, d_ff=4096, tokens_per_gpu=16384,
                 activation="gelu", zipf_s=1.2,
                 policy=dict(overlap_override=8, capacity_override=4, calibration=True,
                             rematerialize=False, reshard_interval=0),
                 workload="cfg2: single GPT-MoE layer fwd+bwd (FSSDP), 16 experts top-2, "
                          "d_model 1024, d_ff 4096 GeLU, 16K tokens/GPU, Zipf(1.2) gate skew"),
    "cfg3": dict(num_experts=8, top_k=2, d_model=4096, d_ff=14336, tokens_per_gpu=8192,
                 activation="swiglu", zipf_s=1.0,
                 policy=dict(overlap_override=2, capacity_override=1, calibration=True,
                             rematerialize=False, reshard_interval=0),
                 workload="cfg3: Mixtral-8x7B-shaped MoE layer, 8 SwiGLU experts top-2, "
                          "d_model 4096, d_ff 14336, 8K tokens/GPU"),
    "cfg4": dict(num_experts=64, top_k=2, d_model=2048, d_ff=1408, tokens_per_gpu=16384,
                 activation="swiglu", zipf_s=1.2,
                 policy=dict(overlap_override=16, capacity_override=4, calibration=True,
                             rematerialize=True, reshard_interval=0),
                 workload="cfg4: 64 fine-grained SwiGLU experts top-2, d_model 2048, d_ff 1408, "
                          "16K tokens/GPU, Zipf(1.2), re-materialization"),
}
CFG = CONFIGS["cfg2"]
CFG2 = CFG  # the metric's configuration
POLICY = CFG["policy"]
ZIPF_S = CFG["zipf_s"]
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def _nvlink_peak():
    """Per-direction NVLink peak measured on this pool's B200s by scripts/nvlink_probe.py
    (inbound user bytes of one GPU pulling from every peer, best of SM kernel / copy
    engines), committed under profiles/; else B200_PROFILING.md's 770 GB/s peer copy."""
    f = ROOT / "profiles" / "r2_nvlink_peak_n4.json"
    if f.exists():
        try:
            return float(json.loads(f.read_text())["nvlink_gbs"]), f"measured ({f.name})"
        except (KeyError, ValueError):
            pass
    return 770.0, "fallback (B200_PROFILING.md peer copy)"


NVLINK_PEER_GBS, NVLINK_PEAK_SRC = _nvlink_peak()
INPUT_POOL = 8  # distinct (x, dy) batches cycled through the steps: routing varies per step


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--tokens", type=int, default=None, help="tokens per GPU (default: config)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--grad-dtype", default="bf16", choices=["bf16", "fp32"],
                    help="weight-gradient buffers (bf16: the reference's grad bytes = param bytes)")
    return ap.parse_args()


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured (MEASURED_PEAKS.json)"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------- clocks sampling
class ClockSampler:
    """SM clock + throttle reasons sampled every 10 ms through NVML during the timed region
    (nvidia-smi's own process start is too slow for a region this short)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self.max_mhz = None
        self.err = None

    def _sample(self):
        nv = self._nv
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        self.samples.append((sm, reasons))

    def _run(self):
        try:
            while not self._stop.wait(0.01):
                self._sample()
        except Exception as exc:  # pragma: no cover - NVML failure mid-run
            self.err = repr(exc)

    def __enter__(self):
        try:  # NVML opened and sampled once synchronously: every region gets >= 2 samples
            import pynvml as nv

            nv.nvmlInit()
            self._nv = nv
            self._h = nv.nvmlDeviceGetHandleByIndex(self.idx)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._sample()
            self._t.start()
        except Exception as exc:  # pragma: no cover - NVML missing
            self.err = repr(exc)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t.is_alive():
            self._t.join(timeout=10)
        if self.err is None and self.max_mhz is not None:
            try:
                self._sample()
            except Exception as exc:  # pragma: no cover
                self.err = repr(exc)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz,
                    "reasons": ["unsampled" if self.err is None else "nvml: " + self.err],
                    "samples": 0}
        sm = sorted(s[0] for s in self.samples)
        reasons = sorted({name for _, r in self.samples for name, bit in self.REASONS.items()
                          if r & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples)}


# ----------------------------------------------------------------- CPU oracle leg
class OracleWorkload:
    """The cfg2 step restated by the CPU oracle port (oracle/: numpy gate + planner port +
    fwd/bwd restatement) on a bounded token sample — the CPU baseline, never the product."""

    def __init__(self, sample_tokens: int, seed: int = 0):
        import numpy as np

        from oracle import planner_oracle as PO
        from oracle import tensor_oracle as TO

        self.np, self.PO, self.TO = np, PO, TO
        E, d, f = CFG2["num_experts"], CFG2["d_model"], CFG2["d_ff"]
        rng = np.random.default_rng(seed)
        self.sample = sample_tokens
        self.x = TO.bf16_round(rng.standard_normal((sample_tokens, d)).astype(np.float32))
        self.wg = (rng.standard_normal((E, d)) / np.sqrt(d)).astype(np.float32)
        p = 1.0 / np.arange(1, E + 1) ** ZIPF_S
        self.bias = np.log(p[rng.permutation(E)] / p.sum()).astype(np.float32)
        nm = 3 if CFG["activation"] == "swiglu" else 2

        def mat(rows, cols, fan_in):
            return TO.bf16_round((rng.standard_normal((rows, cols)) / np.sqrt(fan_in))
                                 .astype(np.float32))
        self.experts = {e: tuple([mat(f, d, d) for _ in range(nm - 1)] + [mat(d, f, f)])
                        for e in range(E)}
        self.dy = TO.bf16_round((0.05 * rng.standard_normal((sample_tokens, d))).astype(np.float32))
        self.topo = PO.Topo(1, 1, NVLINK_PEER_GBS * 1e9, NVLINK_PEER_GBS * 1e9)
        self.knobs = dict(t=POLICY["overlap_override"], m=POLICY["capacity_override"],
                          calibration=True, rematerialize=False, expert_bytes=2 * nm * d * f,
                          token_bytes=2 * d, attn_fwd_time=1e-3, ptt=2.0 * nm * d * f / 1381.7e12)

    def step(self) -> float:
        np, PO, TO = self.np, self.PO, self.TO
        E, k = CFG2["num_experts"], CFG2["top_k"]
        t0 = time.perf_counter()
        logits = TO.gate_logits(self.x, self.wg) + self.bias
        idx, w, _, _ = TO.topk_select(logits, k)
        counts = np.bincount(idx.reshape(-1), minlength=E)[None, :]
        PO.plan_layer([0] * E, counts.astype(np.float64), counts, self.topo, self.knobs)
        TO.moe_layer_fwd_bwd(self.x, idx, w, self.wg, self.experts, self.dy)
        return time.perf_counter() - t0

    @staticmethod
    def threads() -> int:
        n = os.cpu_count() or 1
        try:
            from threadpoolctl import threadpool_info

            n = max((i.get("num_threads", 1) for i in threadpool_info()), default=n)
        except Exception:
            pass
        return n


def planner_compare(devices: int = 8, reps: int = 20) -> dict:
    """One layer-iteration of FSSDP decisions (adoption gate, calibration, fallback,
    build_dispatch; engine.py:491-553) at `devices` GPUs on this config's skewed counts:
    the Python restatement (oracle/, the reference's own algorithm) vs the native planner."""
    import numpy as np

    import paper_2502_02581_b200 as F
    from oracle import planner_oracle as PO

    E, T, k = CFG["num_experts"], CFG["tokens_per_gpu"], CFG["top_k"]
    nm = 3 if CFG["activation"] == "swiglu" else 2
    rng = np.random.default_rng(7)
    p = 1.0 / np.arange(1, E + 1) ** ZIPF_S
    p = p[rng.permutation(E)] / p.sum()
    hist = [rng.multinomial(T * k, p, size=devices).astype(np.int64) for _ in range(5)]
    actual = rng.multinomial(T * k, p, size=devices).astype(np.int64)
    est = np.mean(np.stack(hist), axis=0)
    d, f = CFG["d_model"], CFG["d_ff"]
    knobs = dict(t=POLICY["overlap_override"], m=POLICY["capacity_override"], calibration=True,
                 rematerialize=False, expert_bytes=2 * nm * d * f, token_bytes=2 * d,
                 attn_fwd_time=1e-3, ptt=2.0 * nm * d * f / 1381.7e12)
    topo = PO.Topo(1, devices, NVLINK_PEER_GBS * 1e9, NVLINK_PEER_GBS * 1e9)
    owner = [e * devices // E for e in range(E)]
    t0 = time.perf_counter()
    for _ in range(reps):
        PO.plan_layer(owner, est, actual, topo, knobs)
    oracle_ms = (time.perf_counter() - t0) * 1e3 / reps
    cfg = F.ModelConfig(1, E, knobs["expert_bytes"], 2 * d, 1e-3, knobs["ptt"])
    pl = F.FssdpPlanner(cfg, F.ClusterTopology.for_nvswitch(devices, NVLINK_PEER_GBS * 1e9),
                        F.Policy(F.PolicyKind.FSSDP, **POLICY))
    for h in hist:
        pl.history[0].append(h)
    t0 = time.perf_counter()
    for _ in range(reps):
        pl.plan_layer(0, actual)
    native_ms = (time.perf_counter() - t0) * 1e3 / reps
    return {"devices": devices, "oracle_port_python": round(oracle_ms, 3),
            "native_cpp_via_python": round(native_ms, 4),
            "note": "planning decisions only; bit-identical outputs (tests/test_planner_native.py)"}


def cpu_sample_tokens(at_cfg2: int) -> int:
    """The CPU sample, scaled so a step costs about what `at_cfg2` tokens cost at cfg2."""
    nm = 3 if CFG["activation"] == "swiglu" else 2
    scale = (2 * 1024 * 4096) / (nm * CFG["d_model"] * CFG["d_ff"])
    return int(max(64, min(at_cfg2 * scale, CFG["tokens_per_gpu"])))


def cpu_oracle_rate(sample_tokens: int, budget_s: float):
    wl = OracleWorkload(sample_tokens)
    wl.step()  # warm-up
    steps, spent = 0, 0.0
    while steps == 0 or spent < budget_s:
        spent += wl.step()
        steps += 1
    return steps * sample_tokens / spent, {"steps": steps, "seconds": spent,
                                           "threads": OracleWorkload.threads()}


_THREAD_LIMITS = None


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # every host core (torchrun sets OMP_NUM_THREADS=1 for each rank; the BLAS pool of the
    # numpy port is raised back here)
    global _THREAD_LIMITS
    try:
        import numpy  # noqa: F401  (the BLAS library must be loaded to be re-limited)
        from threadpoolctl import threadpool_limits

        _THREAD_LIMITS = threadpool_limits(limits=os.cpu_count() or 1)
    except Exception:
        pass
    sample = cpu_sample_tokens(2048)
    wl = OracleWorkload(sample)
    for _ in range(args.warmup):
        wl.step()
    total = sum(wl.step() for _ in range(args.steps))
    value = args.steps * sample / total
    det = {"threads": OracleWorkload.threads()}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": _config(args, args.gpus),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": det["threads"],
                         "kind": "port",
                         "sample": f"{sample} tokens of {args.config} per step through oracle/ (numpy "
                                   f"fwd+bwd restatement + planner port), scaled to tokens/s"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config(args, world):
    return {"workload": CFG["workload"], "activation": CFG["activation"],
            "experts": CFG2["num_experts"], "top_k": CFG2["top_k"], "d_model": CFG2["d_model"],
            "d_ff": CFG2["d_ff"], "tokens_per_gpu": args.tokens,
            "global_batch_tokens": args.tokens * world, "parallelism": f"fssdp{world}",
            "policy": POLICY, "zipf_s": ZIPF_S, "grad_dtype": args.grad_dtype,
            "l2": "per-step working set > 1 GB exceeds the 126 MB L2 (no explicit flush)"}


def a2a_stats(dec, allp, keys, world):
    """Token A2A against its roofline: bytes = dispatch_traffic(route, B),
    the max over devices of in/out bytes, per kernel launch (dispatch and dispatch_grad
    push rows, combine and combine_dx pull them back), ÷ the max-rank kernel time."""
    import numpy as np

    B = 2 * CFG2["d_model"]
    r = np.asarray(dec.route, dtype=np.float64)  # [src, e, dst]
    mat = r.sum(axis=1) * B
    np.fill_diagonal(mat, 0.0)
    worst = float(max(mat.sum(axis=1).max(), mat.sum(axis=0).max()))
    out = {"bottleneck_bytes_per_pass": worst, "total_remote_bytes_per_pass": float(mat.sum())}
    for k in ("dispatch", "combine", "dispatch_grad", "combine_dx"):
        if k in keys:
            ms = float(allp[:, keys.index(k)].max())
            out[k + "_gbs"] = worst / (ms * 1e-3) / 1e9 if ms > 0 else None
    return out


# ----------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch

    import paper_2502_02581_b200 as F
    from paper_2502_02581_b200 import _native as NAT
    from paper_2502_02581_b200.layer import create_layer

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    T = args.tokens
    pol = F.Policy(F.PolicyKind.FSSDP, **POLICY)
    layer = create_layer(CFG2["d_model"], CFG2["d_ff"], CFG2["num_experts"], CFG2["top_k"], T,
                         pol, rank=rank, world=world, device=dev, seed=1234,
                         activation=CFG["activation"], grad_dtype=args.grad_dtype)
    E = CFG2["num_experts"]
    p = 1.0 / np.arange(1, E + 1) ** ZIPF_S
    p = p[np.random.default_rng(42).permutation(E)]
    layer.gate_bias.copy_(torch.tensor(np.log(p / p.sum()), dtype=torch.float32))
    # a pool of distinct token batches cycled through the steps: every step routes fresh
    # tokens, so counts, plans and the early-SpAG candidate change from step to step
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    xs = [torch.randn(T, CFG2["d_model"], device=dev, generator=gen).bfloat16()
          for _ in range(INPUT_POOL)]
    dys = [(torch.randn(T, CFG2["d_model"], device=dev, generator=gen) * 0.05).bfloat16()
           for _ in range(INPUT_POOL)]
    it = [0]

    def step():
        i = it[0] % INPUT_POOL
        it[0] += 1
        layer.forward(xs[i])
        dx = layer.backward(dys[i])
        layer.reduce_gate_grad()
        layer.planner.finish()
        return dx

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    layer.timers = None  # the timed region runs uninstrumented
    layer.reset_plan_stats()
    NAT.launch_count = 0
    start, end = torch.cuda.Event(True), torch.cuda.Event(True)
    with ClockSampler(local) as clocks:
        barrier()
        start.record()
        for _ in range(args.steps):
            step()
        end.record()
        barrier()
    launches = NAT.launch_count
    plan_stats = dict(layer.plan_stats)
    ms = start.elapsed_time(end) / args.steps
    # the GPU-side planning gap (count all-gather done -> tables uploaded, dispatch next),
    # probed with just two events per step
    layer.gap_events = []
    barrier()
    for _ in range(args.steps):
        step()
    barrier()
    plan_gap_ms = sum(a.elapsed_time(b) for a, b in layer.gap_events) / max(1, len(layer.gap_events))
    layer.gap_events = None
    # a second, instrumented pass of the same K steps: CUDA events around every kernel
    # (phase breakdown, the GEMM roofline) and host timestamps on the planning path
    # It starts like the timed region — a short rest (the power/clock governor reacts to the
    # recent average: back-to-back passes run increasingly power-capped) and the same number
    # of warm-up steps — so its kernel times describe the kernels of the timed region.
    time.sleep(0.3)
    for _ in range(max(3, args.warmup)):
        step()
    layer.timers = {}
    barrier()
    ref = NAT.NativeEvent()  # timeline origin for the per-kernel launch-timing windows
    ref.record(torch.cuda.current_stream(dev))
    with ClockSampler(local) as inst_clocks:
        for _ in range(args.steps):
            step()
        barrier()
    timers = layer.timers
    marks = timers.pop("marks", [])
    if os.environ.get("FSSDP_TIMELINE"):
        # last timed step's kernels as (start, end) ms from the step's first kernel, one
        # file per rank: $FSSDP_TIMELINE_n{world}_r{rank}.json
        last = []
        for key, ev in timers.items():
            if key == "host_plan_s":
                continue
            per = len(ev) // args.steps
            last += [(key, s_, e_) for s_, e_ in ev[len(ev) - per:]]
        s0 = min(last, key=lambda t: ref.elapsed_time(t[1]))[1]
        rows = sorted((round(s0.elapsed_time(s_), 4), round(s0.elapsed_time(e_), 4), key)
                      for key, s_, e_ in last)
        Path(f"{os.environ['FSSDP_TIMELINE']}_n{world}_r{rank}.json").write_text(json.dumps(rows))
    layer.timers = None
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_max = float(t.item())
    value = world * T / (ms_max * 1e-3)

    def gather(vals):
        """Per-rank float vector -> [world, len] numpy (rank order)."""
        t = torch.tensor(vals, device=dev, dtype=torch.float64)
        if world == 1:
            return t.cpu().numpy()[None, :]
        out = [torch.empty_like(t) for _ in range(world)]
        torch.distributed.all_gather(out, t)
        return torch.stack(out).cpu().numpy()

    # GEMM roofline (dominant kernel family), from the events of the timed region.
    # Algorithmic FLOPs = this rank's real routed token-slots (no padding) x 3 GEMM passes.
    d, f, k = CFG2["d_model"], CFG2["d_ff"], CFG2["top_k"]
    dec = layer.decision
    gemm_ms = sum(s.elapsed_time(e) for key, ev in timers.items() if key.startswith("gemm.")
                  for s, e in ev) / args.steps
    gemm_launches = sum(len(ev) for key, ev in timers.items() if key.startswith("gemm."))
    rows_rank = float(dec.route[:, :, rank].sum())
    nmats = 3 if CFG["activation"] == "swiglu" else 2
    flops_rank = 3 * 2 * rows_rank * nmats * d * f   # fwd + dgrad + wgrad
    spag_ms = sum(s.elapsed_time(e) for key in ("spag", "spag_pre")
                  for s, e in timers.get(key, [])) / args.steps
    sprs_ms = sum(s.elapsed_time(e) for s, e in timers.get("sprs", [])) / args.steps
    t = layer.tables
    n_pre = layer.pre_tables.n_spag if layer.pre_tables is not None else 0
    spag_in = float((t.n_spag + n_pre) * layer.g.slot_param_bytes)
    # SpRS: partials pushed into this rank's staging slots by the holders' wgrad epilogues
    # (NVLink, inside the GEMMs); the "sprs" kernel is the owner-side local reduction, which
    # reads every holder's partial (own slot + staging) and writes the sum
    gb = layer.g.grad_elem_bytes  # bf16 (default) or fp32 weight gradients
    sprs_in = float(t.n_stage * layer.g.slot_grad_elems * gb)
    sprs_reduce_bytes = float(sum(int(c) + 1 for _, _, c in t.sprs_jobs) *
                              layer.g.slot_grad_elems * gb)
    host_ms = 1e3 * sum(timers.get("host_plan_s", [])) / args.steps
    allr = gather([gemm_ms, flops_rank, spag_ms, sprs_ms, spag_in, sprs_in, host_ms, ms,
                   sprs_reduce_bytes, rows_rank, float(t.recv_rows), float(t.n_slots)])
    peaks, peak_src = load_peaks()
    achieved = allr[:, 1].sum() / (allr[:, 0].sum() * 1e-3) / 1e12
    # the GEMMs run inside a ~1.5 ms step at max SM clock: the burst GEMM peak is the
    # denominator (the sustained figure is the seconds-long, power-capped loop's)
    peak = float(peaks.get("bf16_tflops", PEAKS_FALLBACK["bf16_tflops"]))
    peak_sustained = float(peaks.get("bf16_tflops_sustained",
                                     PEAKS_FALLBACK["bf16_tflops_sustained"]))
    traffic, traffic_src = None, None
    tfiles = sorted((ROOT / "profiles").glob("*gemm_traffic.json"))
    if tfiles:  # DRAM bytes of the step's GEMM launches from the committed ncu --set full capture
        traffic = json.loads(tfiles[-1].read_text())["gemm_dram_bytes_per_step"]
        traffic_src = f"{tfiles[-1].name}: dram__bytes_read.sum + dram__bytes_write.sum"
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_unit": "bytes per step "
                "(the N=1 step's GEMM launches)", "traffic_source": traffic_src,
                "kernel": "fssdp grouped_gemm_kernel (tcgen05), all 6 GEMMs of the step",
                "algorithmic_flops": "3 x 2 x routed_rows x n_mats x d_model x d_ff per rank "
                                     "(n_mats 2 GeLU, 3 SwiGLU)",
                "peak_source": f"{peak_src}, burst bf16 (cuBLAS 8192^3 best of 10; the "
                               f"GEMMs run at max SM clock inside a short step)",
                "frac_of_sustained": achieved / peak_sustained,
                "gemm_ms_per_step_per_rank": [round(v, 4) for v in allr[:, 0]],
                "gemm_tflops_per_rank": [round(f / (g * 1e-3) / 1e12, 1)
                                         for g, f in zip(allr[:, 0], allr[:, 1])],
                "routed_rows_per_rank": [int(v) for v in allr[:, 9]],
                "padded_rows_per_rank": [int(v) for v in allr[:, 10]],
                "expert_slots_per_rank": [int(v) for v in allr[:, 11]],
                "gemm_share_of_step": float(allr[:, 0].max() / ms_max),
                "gemm_launches_per_step": gemm_launches / args.steps,
                "host_plan_ms_per_step": float(allr[:, 6].max()),
                "instrumented_pass_clocks": inst_clocks.summary()}
    # per-phase device time (CUDA events around every kernel of the timed steps), max over ranks
    # host planning path: mean microseconds between consecutive marks of a step
    host_us = {}
    for (n0, t0), (n1, t1) in zip(marks, marks[1:]):
        if n1 == "readback":
            continue  # next step
        key = f"{n0}->{n1}"
        host_us[key] = host_us.get(key, 0.0) + (t1 - t0) * 1e6 / args.steps
    keys = sorted(k for k in timers if k != "host_plan_s")
    if world > 1:  # ranks may launch different phases (e.g. no SpAG copies): use the union
        allk = [None] * world
        torch.distributed.all_gather_object(allk, keys)
        keys = sorted(set().union(*allk))
    phase_ms = [sum(s.elapsed_time(e) for s, e in timers.get(k, [])) / args.steps for k in keys]
    allp = gather(phase_ms) if keys else None
    breakdown = {k: round(float(allp[:, i].max()), 4) for i, k in enumerate(keys)} if keys else {}
    breakdown["host_plan"] = round(float(allr[:, 6].max()), 4)
    breakdown["planning_gap_gpu"] = round(float(gather([plan_gap_ms])[:, 0].max()), 4)
    breakdown["sum_of_kernels_max_rank"] = round(float(allp.sum(axis=1).max()), 4) if keys else 0.0
    sparse = None
    if world > 1:
        tr, rep = F.spag_traffic(dec.base, dec.target, layer.g.expert_bytes)
        spag_max, sprs_max = float(allr[:, 2].max()), float(allr[:, 3].max())
        gbs = lambda b, m: (b / (m * 1e-3) / 1e9) if m > 0 else None  # noqa: E731
        sparse = {
            "replicas": len(dec.target.entries) - E,
            "spag_total_bytes": rep.total_interdevice_bytes,
            "spag_bottleneck_bytes": rep.bottleneck_bytes,
            "spag_early_copies_rank0": n_pre, "spag_late_copies_rank0": t.n_spag,
            "spag_ms_max_rank": spag_max, "sprs_ms_max_rank": sprs_max,
            "spag_bottleneck_gbs": gbs(rep.bottleneck_bytes, spag_max),
            "spag_inbound_gbs_per_rank": [gbs(b, m) for b, m in zip(allr[:, 4], allr[:, 2])],
            "sprs_pushed_in_bytes_per_rank": [float(b) for b in allr[:, 5]],
            "sprs_local_reduce_gbs_per_rank": [gbs(b, m) for b, m in zip(allr[:, 8], allr[:, 3])],
            "nvlink_peak_gbs": NVLINK_PEER_GBS, "nvlink_peak_source": NVLINK_PEAK_SRC,
            "spag_bottleneck_frac_of_nvlink": (gbs(rep.bottleneck_bytes, spag_max) or 0.0)
                                              / NVLINK_PEER_GBS,
            "a2a": a2a_stats(dec, allp, keys, world),
            "note": f"SpRS wire is {layer.g.grad_dtype} partials pushed by the wgrad "
                    "epilogue's TMA stores (bf16 = the reference's expert_bytes pricing); "
                    "sprs_ms is the local reduce. "
                    "The early SpAG runs on the copy engines in two windows (W1 parts with the "
                    "gate, W2 parts beside fwd1 — sharing NVLink with the dispatch / GEMM "
                    "traffic); spag_ms sums both windows. Standalone SpAG / SpRS kernel "
                    "bandwidth: profiles/r1_sparse_sweep.txt"}

    # end to end through the public API with host buffers: each step's (x, dy) is copied
    # H2D from pinned host memory on a copy stream one step ahead (double buffered); its y
    # and dx are copied D2H behind the compute (y once the forward is done).
    e2e = None
    if not args.no_e2e:
        HP = 2  # distinct pinned host batches (the device pool's first two)
        xh = [xs[i].cpu().pin_memory() for i in range(HP)]
        dyh = [dys[i].cpu().pin_memory() for i in range(HP)]
        dxh = [torch.empty_like(xh[0]).pin_memory() for _ in range(2)]
        yh = [torch.empty_like(xh[0]).pin_memory() for _ in range(2)]
        xb = [torch.empty_like(xs[0]) for _ in range(2)]
        dyb = [torch.empty_like(dys[0]) for _ in range(2)]
        copy_s = torch.cuda.Stream(device=dev)   # H2D
        d2h_s = torch.cuda.Stream(device=dev)    # D2H: PCIe is full duplex
        main_s = torch.cuda.current_stream(dev)
        in_ev = [torch.cuda.Event() for _ in range(2)]     # x of the step landed
        in_dy_ev = [torch.cuda.Event() for _ in range(2)]  # dy landed (the backward waits)
        done_ev = [torch.cuda.Event() for _ in range(2)]
        fwd_ev = [torch.cuda.Event() for _ in range(2)]

        def prefetch(i):
            b = i % 2
            with torch.cuda.stream(copy_s):
                copy_s.wait_event(done_ev[b])  # step i-2 finished with buffer b
                xb[b].copy_(xh[i % HP], non_blocking=True)
                in_ev[b].record(copy_s)
                dyb[b].copy_(dyh[i % HP], non_blocking=True)
                in_dy_ev[b].record(copy_s)

        def d2h(t, host, ev):
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(ev)
                host.copy_(t, non_blocking=True)
                t.record_stream(d2h_s)

        def run(n):
            # The bulk copies are issued once the step's forward has been planned (the
            # host is past the plan when forward() returns): issued earlier, they share
            # PCIe with the planning path's small SM-driven transfers (counts out, tables
            # in) and stretch the GPU's planning gap (0.054 -> 0.141 ms measured at N=1).
            for ev in done_ev:
                ev.record(main_s)
            prefetch(0)
            for i in range(n):
                b = i % 2
                main_s.wait_event(in_ev[b])
                y = layer.forward(xb[b])
                fwd_ev[b].record(main_s)
                if i + 1 < n:  # next inputs stream in while this step computes
                    prefetch(i + 1)
                d2h(y, yh[b], fwd_ev[b])  # this step's y, behind its forward
                main_s.wait_event(in_dy_ev[b])  # the forward only needed x
                dx = layer.backward(dyb[b])
                # dx is final once the dX combine ran (layer.dx_event), while the last
                # wgrads still compute: it streams out from there
                d2h(dx, dxh[b], layer.dx_event)
                layer.reduce_gate_grad()
                layer.planner.finish()
                done_ev[b].record(main_s)
            main_s.wait_stream(copy_s)
            main_s.wait_stream(d2h_s)

        run(2)
        barrier()
        s2, e2 = torch.cuda.Event(True), torch.cuda.Event(True)
        s2.record()
        run(args.steps)
        e2.record()
        barrier()
        e2e_ms = s2.elapsed_time(e2) / args.steps
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_ms = float(t.item())
        nb = T * CFG2["d_model"] * 2
        e2e = {"value": world * T / (e2e_ms * 1e-3), "unit": "tokens/s",
               "h2d_bytes_per_step": 2 * nb, "d2h_bytes_per_step": 2 * nb, "ms_per_step": e2e_ms,
               "pipeline": "x, dy of step i+1 H2D and y, dx of step i D2H on two copy "
                           "streams (PCIe full duplex), overlapped with the compute "
                           "(FssdpMoE.forward/backward; the forward waits for x only, the "
                           "backward for dy; y streams out after the forward, dx after the "
                           "dX combine, layer.dx_event); two distinct host batches alternate"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = cpu_sample_tokens(1024)
        rate, det = cpu_oracle_rate(sample, 8.0)
        cpu = {"value": rate, "unit": "tokens/s", "cores": det["threads"], "kind": "port",
               "sample": f"{sample}-token batches of {args.config} through oracle/ (numpy fwd+bwd + planner "
                         f"port), {det['steps']} batches in {det['seconds']:.1f} s",
               "planner_ms_per_layer_iteration": planner_compare()}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_max,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                "data": f"synthetic (seeded N(0,1) tokens, {INPUT_POOL} distinct batches cycled "
                        f"per rank, random-init experts, Zipf gate bias)",
                "config": _config(args, world), "roofline": roofline, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": launches, "clocks": clocks.summary(),
                "phase_ms_per_step": breakdown,
                "early_spag": {**plan_stats, "hit_rate": plan_stats["early_hit"] /
                               max(1, plan_stats["early"]),
                               "note": "timed steps: early = an estimate-based candidate was "
                                       "fetched before the gate; hit = the final plan equals "
                                       "it; extended = calibration added replicas (late "
                                       "SpAG); fallback = dropped to the bare partition"},
                "host_plan_path_us": {k: round(v, 1) for k, v in host_us.items()}}
        if sparse:
            line["sparse_collectives"] = sparse
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def select_config(name: str) -> None:
    global CFG, CFG2, POLICY, ZIPF_S
    CFG = CFG2 = CONFIGS[name]
    POLICY = CFG["policy"]
    ZIPF_S = CFG["zipf_s"]


def main():
    args = parse()
    select_config(args.config)
    if os.environ.get("FSSDP_POLICY"):  # experiments: "t,m" overrides the config's knobs
        t, m = (int(v) for v in os.environ["FSSDP_POLICY"].split(","))
        POLICY.update(overlap_override=t, capacity_override=m)
    if args.tokens is None:
        args.tokens = CFG["tokens_per_gpu"]
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
