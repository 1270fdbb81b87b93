for i in 1 2 3; do for v in 0 1; do
FSSDP_GEMM_WIDE_STORE=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']
print('wide=$v', round(d['ms_per_step'],4), 'fwd1', p['gemm.fwd1'], 'fwd2', p['gemm.fwd2'], 'dgrad2', p['gemm.dgrad2'])"
done; done
for v in 0 1; do FSSDP_GEMM_WIDE_STORE=$v TAG=wide$v python scripts/epi_probe.py | head -1; done
