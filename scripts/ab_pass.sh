FSSDP_DISPATCH_PDL=1 timeout 900 python -m pytest tests/test_layer_gpu.py tests/test_dist_gpu.py -q -x 2>&1 | tail -1
bash scripts/ab_env.sh "FSSDP_DISPATCH_PDL=0" "FSSDP_DISPATCH_PDL=1" 3
NGPU=4 bash scripts/ab_env.sh "FSSDP_DISPATCH_PDL=0" "FSSDP_DISPATCH_PDL=1" 3
