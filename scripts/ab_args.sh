#!/bin/bash
# Interleaved A/B of bench.py argument sets at N GPUs on one box:
#   ab_args.sh N rounds "<args A>" "<args B>"
N=$1; R=$2; A="$3"; B="$4"
run() {
  if [ "$N" = 1 ]; then python bench.py --steps 20 --warmup 5 --no-cpu-baseline $1 2>/dev/null | tail -1
  else python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus $N --steps 20 --warmup 5 --no-cpu-baseline $1 2>/dev/null | tail -1; fi
}
for i in $(seq 1 $R); do
  for v in "$A" "$B"; do
    run "$v" | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$v'.ljust(30), round(d['ms_per_step'],4), round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
