# One-GPU pass: GPU tests, then N=1 bench lines of cfg2 (default) and the other configs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in ${CONFIGS:-cfg2 cfg4}; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c_$c.json 2> gpurun_out/c_$c.err
  python - $c <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/c_{c}.json").read().strip().splitlines()[-1])
    ph = d["phase_ms_per_step"]; r = d["roofline"]
    print(c, round(d["value"] / 1e6, 4), "M", round(d["ms_per_step"], 4), "ms gemm", round(r["achieved"]), round(r["frac"], 3),
          {k: ph[k] for k in sorted(ph) if k.startswith("gemm.")})
except Exception as exc:
    print(c, "FAILED", exc)
PY
done
