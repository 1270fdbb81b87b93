timeout 900 python -m pytest tests/test_gemm_gpu.py -q -x -k swap 2>&1 | tail -3
timeout 300 python scripts/swap_probe.py
bash scripts/ab_env.sh "FSSDP_SWAP_TAIL=dgrad2,fwd2,dgrad1" "FSSDP_X=1" 4 --config cfg4
