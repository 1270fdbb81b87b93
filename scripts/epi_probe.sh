# epilogue probe: the default build with wide stores on / off (FSSDP_GEMM_WIDE_STORE)
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -2
for r in 1 2; do
  for w in 1 0; do FSSDP_GEMM_WIDE_STORE=$w TAG=wide$w timeout 120 python scripts/epi_probe.py; done
done
