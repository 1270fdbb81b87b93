timeout 900 python -m pytest tests/test_dist_gpu.py -q -x 2>&1 | tail -1
NGPU=4 bash scripts/ab_env.sh "FSSDP_EARLY_GATE_REDUCE=0" "FSSDP_EARLY_GATE_REDUCE=1" 3
