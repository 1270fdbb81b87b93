# SpRS CTA budget sweep at N=4 (FSSDP_SPRS_CTAS; 0 = one CTA per unit)
for c in 0 16 32 64 148; do
  FSSDP_SPRS_CTAS=$c python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2960$((c % 10)) bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e > gpurun_out/sw_$c.json 2> gpurun_out/sw_$c.err
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
d = json.loads(open(f"gpurun_out/sw_{c}.json").read().strip().splitlines()[-1])
p = d["phase_ms_per_step"]
print("CTAS", c, round(d["value"] / 1e6, 3), "M", round(d["ms_per_step"], 3), "ms",
      {k: p.get(k) for k in ("gemm.dgrad1", "gemm.wgrad1", "gemm.wgrad2", "sprs", "barrier")},
      d["roofline"]["gemm_ms_per_step_per_rank"])
PY
done
