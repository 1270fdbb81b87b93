# N=2 / N=4 bench lines (with timelines) and the cfg5 sparse collective sweep at N=4
for n in 2 4; do
FSSDP_TIMELINE=gpurun_out/tl python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/n$n.json 2> gpurun_out/n$n.err
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 scripts/sparse_sweep.py --quick > gpurun_out/sweep4.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 scripts/sparse_sweep.py --quick > gpurun_out/sweep2.log 2>&1
echo SCALE_DONE
