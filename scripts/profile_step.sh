# One-GPU profile pass: tests, a clean bench line, then the ncu launch list and a full
# capture of one step's 14 kernels (each only after the same command exited 0 without ncu).
set -e
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
FSSDP_TIMELINE=gpurun_out/tl python bench.py --steps 20 --warmup 5 > gpurun_out/n1.json 2> gpurun_out/n1.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
# warm-up 3 + timed 1 + gap-probe 1 steps: 4 x 13 matching launches skipped (gate, dispatch,
# 6 GEMMs, combine, dispatch_grad, combine_dx, gate_wgrad x2), then one step captured
ncu --set full --clock-control none --import-source on \
    -k regex:"dispatch|combine|gate|route_scan|grouped_gemm" --launch-skip 52 -c 13 \
    -f -o gpurun_out/step_full \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
echo PROFILE_DONE
