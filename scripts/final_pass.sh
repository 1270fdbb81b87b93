# Round-end validation on a 4-GPU box: all GPU tests (incl. the 2- and 4-process parity
# checks), smoke(), the default N=1 bench line (as the driver runs it), N=2 / N=4 lines
# with timelines, the reference arm, and N=1 lines of cfg1 / cfg3 / cfg4.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/f_n1.json 2> gpurun_out/f_n1.err; tail -1 gpurun_out/f_n1.err
for n in 2 4; do
  FSSDP_TIMELINE=gpurun_out/tl timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/f_n$n.json 2> gpurun_out/f_n$n.err
done
timeout 600 python bench.py --impl reference > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err
for c in cfg1 cfg3 cfg4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/f_$c.json 2> gpurun_out/f_$c.err
done
python - <<'PY'
import json
for name in ("f_n1", "f_n2", "f_n4", "f_ref", "f_cfg1", "f_cfg3", "f_cfg4"):
    try:
        d = json.loads(open(f"gpurun_out/{name}.json").read().strip().splitlines()[-1])
        r = d.get("roofline") or {}
        print(name, round(d["value"] / 1e6, 4), "M", round(d["ms_per_step"], 4), "ms",
              "e2e", round(d["e2e"]["value"] / 1e6, 3), "gemm", round(r.get("achieved", 0)),
              round(r.get("frac", 0), 3), d.get("clocks"))
    except Exception as exc:
        print(name, "FAILED", exc)
PY
echo FINAL_DONE
