"""Summarise gpurun_out/n{1,2,4}.json (+ N=4 timelines) after scripts/run_scale.sh."""
import json
import sys

for n in sys.argv[1:] or ["1", "2", "4"]:
    try:
        d = json.loads(open(f"gpurun_out/n{n}.json").read().strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001
        print(n, "no result", exc)
        continue
    e2e = d["e2e"]["value"] / 1e6 if d.get("e2e") else None
    print(f"N={n} {d['value'] / 1e6:.3f}M tok/s {d['ms_per_step']:.3f} ms  e2e {e2e}  "
          f"gemm {d['roofline']['achieved']:.0f} TF/s  clocks {d['clocks']}")
    print("   gemm/rank", d["roofline"]["gemm_ms_per_step_per_rank"],
          "host_plan", round(d["roofline"]["host_plan_ms_per_step"], 4))
    print("  ", d["phase_ms_per_step"])
    for r in range(int(n)):
        try:
            rows = json.loads(open(f"gpurun_out/tl_n{n}_r{r}.json").read())
        except OSError:
            continue
        print(f"   rank {r}:", "  ".join(f"{k}[{a:.3f}-{b:.3f}]" for a, b, k in rows))
