timeout 900 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q -x -k "swiglu or cfg4 or Swiglu" 2>&1 | tail -2
bash scripts/ab_env.sh "FSSDP_SWAP_TAIL=fwd1,fwd2,dgrad1" "FSSDP_X=1" 3 --config cfg4
