# A/B at N GPUs (arg 1): _ab_old (worktree of an older commit, built in place) vs this
# tree, interleaved, cfg2 bench lines (device value + e2e)
N=${1:-1}
run() {
  if [ "$N" = 1 ]; then python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1
  else python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1; fi
}
show() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']/1e6,3), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']/1e6,3))"; }
for i in 1 2 3; do
  (cd _ab_old && run | show OLD)
  run | show NEW
done
