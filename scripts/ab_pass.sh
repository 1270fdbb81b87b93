for v in build/v_nohoist.so paper_2502_02581_b200/libfssdp.so build/v_nohoist.so paper_2502_02581_b200/libfssdp.so; do FSSDP_LIB=$v python scripts/kernel_bench.py 2>&1 | grep KBENCH | cut -c1-150; done
bash scripts/ab_env.sh "FSSDP_LIB=build/v_nohoist.so" "FSSDP_X=1" 3
