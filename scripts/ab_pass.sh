FSSDP_GEMM_WIDE_DGELU=1 timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py tests/test_parity_full_gpu.py -q -x 2>&1 | tail -1
for i in 1 2 3; do for v in 0 1; do
FSSDP_GEMM_WIDE_DGELU=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']
print('wdg=$v', round(d['ms_per_step'],4), *[(k[5:], p[k]) for k in sorted(p) if k.startswith('gemm.d')])"
done; done
