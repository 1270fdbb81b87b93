for i in 1 2; do for v in build/v_bk64.so paper_2502_02581_b200/libfssdp.so build/v_bk128.so; do
FSSDP_LIB=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']
print('$v'.ljust(34), round(d['ms_per_step'],4), *[(k[5:], p[k]) for k in sorted(p) if k.startswith('gemm')])"
done; done
nvidia-smi --query-gpu=name,serial,clocks.max.sm,power.limit --format=csv
