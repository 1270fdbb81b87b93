# interleaved A/B of two bench.py files (e2e): e2e_ab.sh N rounds [bench args]
N=${1:-1}; R=${2:-3}; shift 2
for i in $(seq 1 $R); do
 for b in _bench_old.py bench.py; do
  if [ "$N" = 1 ]; then cmd="python $b --steps 20 --warmup 5 --no-cpu-baseline $@"
  else cmd="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29544 $b --gpus $N --steps 20 --warmup 5 --no-cpu-baseline $@"; fi
  $cmd 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$b'.ljust(16), round(d['ms_per_step'],4), round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3), round(d['e2e']['ms_per_step'],4), d['clocks']['sm_mhz'])"
 done
done
