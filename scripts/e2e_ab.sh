for i in 1 2 3; do
 for b in _bench_old.py bench.py; do
  python $b --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$b'.ljust(16), round(d['ms_per_step'],4), round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3), round(d['e2e']['ms_per_step'],4), d['clocks']['sm_mhz'])"
 done
done
