timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
NGPU=4 bash scripts/ab_env.sh "FSSDP_P2P_GATE_REDUCE=0" "FSSDP_P2P_GATE_REDUCE=1" 3
