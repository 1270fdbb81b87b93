# quick iteration pass on one GPU: tests, kernel microbenchmarks, GEMM pair bench, N=1 step
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python scripts/kernel_bench.py 2>&1 | grep KBENCH
python scripts/gemm_pair_bench.py 2>&1 | tail -3
FSSDP_TIMELINE=gpurun_out/tl python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/n1.json 2> gpurun_out/n1.err
