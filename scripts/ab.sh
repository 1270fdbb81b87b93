# A/B: the bench in _ab_old (a worktree of an older commit, built in place) and in this
# tree, interleaved, on one GPU
for i in 1 2; do
  (cd _ab_old && python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('OLD', round(d['value']/1e6,3), round(d['ms_per_step'],4))")
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NEW', round(d['value']/1e6,3), round(d['ms_per_step'],4))"
done
