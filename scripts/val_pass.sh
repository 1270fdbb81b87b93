mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/v_n1.json 2> gpurun_out/v_n1.err; tail -2 gpurun_out/v_n1.err; cat gpurun_out/v_n1.json | cut -c1-400
