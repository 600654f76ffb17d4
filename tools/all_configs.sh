#!/bin/bash
# Bench every BASELINE config on one GPU (cfg2 is the headline; the others are recorded
# in profiles/ as evidence).  usage (under gpurun): bash tools/all_configs.sh TAG
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
for c in cfg1 cfg3 cfg4 cfg5; do
  steps=3
  [ $c = cfg1 ] && steps=20  # 4.5 ms steps: a longer timed region
  timeout 900 python bench.py --config $c --steps $steps --warmup 3 --no-cpu-baseline > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err
  tail -c 300 $O/${TAG}_bench_$c.json; echo
done
