# A/B: _ab_old (a worktree of an older commit, built in place) vs this tree, interleaved,
# on one GPU: the GEMM microbenchmark and the cfg2 bench line
for i in 1 2; do
  (cd _ab_old && python scripts/gemm_pair_bench.py 2>/dev/null | grep "pair=True" | sed 's/^/OLD /')
  python scripts/gemm_pair_bench.py 2>/dev/null | grep "pair=True" | sed 's/^/NEW /'
  (cd _ab_old && python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('OLD step', round(d['value']/1e6,3), round(d['ms_per_step'],4))")
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NEW step', round(d['value']/1e6,3), round(d['ms_per_step'],4))"
done
