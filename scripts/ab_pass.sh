timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py -q -x 2>&1 | tail -1
for cfg in cfg4 cfg2; do for i in 1 2; do for v in "FSSDP_EPI16=0" "FSSDP_EPI16=wgrad1"; do
env $v python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']
print('$cfg $v'.ljust(30), round(d['ms_per_step'],4), *[(k[5:], p[k]) for k in sorted(p) if k.startswith('gemm.w')])"
done; done; done
