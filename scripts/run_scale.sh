# GPU tests, then N=1/2/4 benches (N=4 with the per-rank step timeline on stderr)
python -m pytest tests -m gpu -x -q 2>&1 | tail -4
FSSDP_TIMELINE=gpurun_out/tl python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/n1.json 2> gpurun_out/n1.err
for n in 2 4; do
FSSDP_TIMELINE=gpurun_out/tl python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/n$n.json 2> gpurun_out/n$n.err
done
