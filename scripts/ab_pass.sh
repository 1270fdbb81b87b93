timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
bash scripts/ab_env.sh "FSSDP_PUSH_SIDE=0" "FSSDP_PUSH_SIDE=1" 4
