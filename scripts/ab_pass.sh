timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
bash scripts/ab_env.sh "FSSDP_LATE_DOTS=0" "FSSDP_LATE_DOTS=1" 4
