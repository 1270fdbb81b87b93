# N=1 bench lines of the other BASELINE configs (reference measurements; cfg2 is the metric)
for c in cfg1 cfg3 cfg4; do
  python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
  tail -1 gpurun_out/cfg_$c.err
done
echo CONFIGS_DONE
