# SpRS pull transport: kernel tests, then the cfg5 sweep (push vs pull columns) at N=4
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sparse_gpu.py -q -x > gpurun_out/pull_tests.log 2>&1; echo "tests rc $?"
tail -3 gpurun_out/pull_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 scripts/sparse_sweep.py > gpurun_out/sweep_n4.log 2>&1; echo "sweep4 rc $?"
python scripts/sweep_table.py gpurun_out/sweep_n4.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 scripts/sparse_sweep.py > gpurun_out/sweep_n2.log 2>&1; echo "sweep2 rc $?"
python scripts/sweep_table.py gpurun_out/sweep_n2.log
