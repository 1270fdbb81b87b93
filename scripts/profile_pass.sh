# Round-2 measurement pass on one GPU: the default bench line, the ncu launch list of the
# same workload (cold, serialised: shares only), and one ncu --set full capture of a whole
# N=1 step's kernels (GEMM DRAM traffic for bench.py's roofline.traffic).
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
K='regex:gate_topk|dispatch|grouped_gemm|combine|gate_wgrad|push_host|pull_host|spag|sprs'
timeout 600 python bench.py > gpurun_out/p_n1.json 2> gpurun_out/p_n1.err
timeout 600 $B > gpurun_out/p_plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv \
    --log-file gpurun_out/p_launches.csv $B > gpurun_out/p_ncu1.log 2>&1
echo launches=$?
# one step = 14 launches at N = 1; skip the 3 warm-up steps
timeout 1500 ncu --set full --clock-control none --import-source on -k "$K" -s 42 -c 14 \
    -o gpurun_out/p_step_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/p_ncu2.log 2>&1
echo full=$?
