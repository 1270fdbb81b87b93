#!/bin/bash
# Interleaved A/B of env settings on one box: [NGPU=n] ab_env.sh "<envA>" "<envB>" [rounds] [bench args]
A="$1"; B="$2"; R="${3:-3}"; shift 3
N=${NGPU:-1}
for i in $(seq 1 $R); do
  for v in "$A" "$B"; do
    if [ "$N" = 1 ]; then
      out=$(env $v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1)
    else
      out=$(env $v python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port 29571 bench.py --gpus $N --steps 20 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1)
    fi
    echo "$out" | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v'.ljust(40), round(d['ms_per_step'],4), round(d['value']/1e6,3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
