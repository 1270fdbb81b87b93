# Early-SpAG footprint (FSSDP_SPAG_PRE_CTAS) at N=4 and N=2: step time, interleaved
run() {
  n=$1; shift
  env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29504 bench.py --gpus $n --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$n $*', round(d['value']/1e6,3), round(d['ms_per_step'],4))"
}
for rep in 1 2; do
  for c in 0 74 111 148; do run 4 FSSDP_SPAG_PRE_CTAS=$c; done
done
for c in 0 74 148; do run 2 FSSDP_SPAG_PRE_CTAS=$c; done
