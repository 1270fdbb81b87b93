cd /root/repo
for cfg in cfg2 cfg4; do
./scripts/ab_env.sh "FSSDP_X=0" "FSSDP_COMBINE_DX_CTAS=148" 2 --config $cfg
./scripts/ab_env.sh "FSSDP_COMBINE_DX_CTAS=296" "FSSDP_COMBINE_DX_CTAS=74" 1 --config $cfg
./scripts/ab_env.sh "FSSDP_X=0" "FSSDP_GEMM_DYN=wgrad1" 2 --config $cfg
done
