FSSDP_LIB=build/v_mn96.so timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_gate_gpu.py tests/test_layer_gpu.py -q -x 2>&1 | tail -1
for i in 1 2; do for v in paper_2502_02581_b200/libfssdp.so build/v_mn96.so build/v_mn128.so; do
FSSDP_LIB=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']
print('$v'.ljust(34), round(d['ms_per_step'],4), *[(k[5:], p[k]) for k in sorted(p) if k.startswith('gemm')])"
done; done
bash scripts/ab_env.sh "FSSDP_LIB=paper_2502_02581_b200/libfssdp.so" "FSSDP_LIB=build/v_mn96.so" 2 --config cfg4
