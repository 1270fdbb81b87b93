# A/B of an environment knob at N=${NGPU:-2} on one box: GPU tests first, then interleaved bench runs.
# usage: bash scripts/ab_env2.sh VAR   (compares VAR=0 vs VAR=1)
V=${1:-FSSDP_KEEP_Y}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for rep in 1 2; do
  for val in 0 1; do
    if [ "${NGPU:-2}" = 1 ]; then
      env $V=$val timeout 600 python bench.py --config ${CONFIG:-cfg2} --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${val}_$rep.json 2> gpurun_out/ab_${val}_$rep.err
    else
    env $V=$val timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NGPU:-2} --master-addr 127.0.0.1 --master-port 2960$val bench.py --gpus ${NGPU:-2} --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${val}_$rep.json 2> gpurun_out/ab_${val}_$rep.err
    fi
    python - "$V=$val" gpurun_out/ab_${val}_$rep.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    ph = d["phase_ms_per_step"]
    print(sys.argv[1], round(d["value"] / 1e6, 3), "M", round(d["ms_per_step"], 4), "ms e2e",
          round(d["e2e"]["value"] / 1e6, 3), {k: ph[k] for k in ("dispatch", "combine", "dispatch_grad", "combine_dx", "gate_wgrad", "sprs", "barrier", "gemm.fwd1", "gemm.wgrad2") if k in ph})
except Exception as exc:
    print(sys.argv[1], "FAILED", exc)
PY
  done
done
