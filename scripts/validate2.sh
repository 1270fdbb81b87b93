mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/v_n1.json 2> gpurun_out/v_n1.err; tail -2 gpurun_out/v_n1.err
FSSDP_TIMELINE=gpurun_out/vtl timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29502 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/v_n2.json 2> gpurun_out/v_n2.err; tail -2 gpurun_out/v_n2.err
python - <<'PY'
import json
for name in ("v_n1", "v_n2"):
    try:
        d = json.loads(open(f"gpurun_out/{name}.json").read().strip().splitlines()[-1])
        r = d.get("roofline") or {}
        print(name, round(d["value"] / 1e6, 4), "M", round(d["ms_per_step"], 4), "ms",
              "e2e", round(d["e2e"]["value"] / 1e6, 3), "gemm", round(r.get("achieved", 0)),
              round(r.get("frac", 0), 3), d.get("clocks"))
    except Exception as exc:
        print(name, "FAILED", exc)
PY
