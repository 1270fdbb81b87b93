"""Pretty-print SWEEP lines from scripts/sparse_sweep.py output."""
import json
import sys

print(f"{'N':>2} {'variant':7} {'r':>2} {'MiB':>4} {'spag_ms':>8} {'spag_GB/s':>9} "
      f"{'push_ms':>8} {'push_GB/s':>9} {'pull_ms':>8} {'pull_GB/s':>9}  grads")
for line in open(sys.argv[1]):
    if not line.startswith("SWEEP "):
        continue
    d = json.loads(line[6:])
    g = d.get("grad_dtype", "fp32")  # older lines: fp32 keys
    sfx = "_fp32" if "grad_dtype" not in d else ""
    print(f"{d['n_gpus']:>2} {d['variant']:7} {d['replicas']:>2} {d['expert_mib']:>4} "
          f"{d['spag_ms']:8.3f} {d['spag_gbs_bottleneck']:9.0f} {d['sprs_ms']:8.3f} "
          f"{d['sprs_gbs_bottleneck' + sfx]:9.0f} {d.get('sprs_pull_ms', float('nan')):8.3f} "
          f"{d.get('sprs_pull_gbs_bottleneck' + sfx, float('nan')):9.0f}  {g}")
