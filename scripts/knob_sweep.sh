# FSSDP knob sweep at N GPUs (default 4): t (overlap degree) x m (replica slots), cfg2
N=${1:-4}
for tm in ${KNOBS:-8,4 8,6 10,6 12,8 16,8}; do
  for rep in 1 2; do
    FSSDP_POLICY=$tm python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/k_${tm/,/_}_$N.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/k_${tm/,/_}_$N.json').read().strip().splitlines()[-1]); print('KNOB $tm N=$N', round(d['value']/1e6,3), round(d['ms_per_step'],3), d['roofline']['gemm_ms_per_step_per_rank'], d['roofline']['routed_rows_per_rank'], d['sparse_collectives']['replicas'])"
  done
done
