# Early-SpAG footprint at N=4 (step time), interleaved
run() {
  n=$1; shift
  env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29504 bench.py --gpus $n --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$n $*', round(d['value']/1e6,3), round(d['ms_per_step'],4))"
}
for rep in 1 2; do
  run 4 X=1
  run 4 FSSDP_SPAG_PRE_CTAS=74
  run 4 FSSDP_SPAG_PRE_CTAS=37
done
