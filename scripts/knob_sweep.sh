for tm in 8,4 8,6 10,6 12,8; do
  for n in 4; do
    FSSDP_POLICY=$tm python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e > gpurun_out/k_${tm/,/_}_$n.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/k_${tm/,/_}_$n.json').read().strip().splitlines()[-1]); print('KNOB $tm N=$n', round(d['value']/1e6,3), round(d['ms_per_step'],3), d['roofline']['gemm_ms_per_step_per_rank'], d['sparse_collectives']['replicas'])"
  done
done
