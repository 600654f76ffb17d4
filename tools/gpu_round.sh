#!/bin/bash
# One GPU session: gpu tests, smoke, bench (+reference arm), ncu launch list, ncu full captures.
# usage (under gpurun): bash tools/gpu_round.sh TAG
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke exit $?" >> $O/${TAG}_smoke.log
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
timeout 300 python bench.py --impl reference > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err
for d in bf16 f32; do
  V=151936; [ $d = f32 ] && V=32000
  timeout 300 python tools/kbench.py --rows 32768 --vocab $V --dtype $d >> $O/${TAG}_kbench.jsonl 2>>$O/${TAG}_kbench.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-fused-head > $O/${TAG}_ncu_bench.log 2>&1
[ -n "$FULL" ] && timeout 600 ncu --set full --clock-control none --import-source on -k regex:logprob_ring -c 1 \
  -o $O/${TAG}_k1 -f python tools/kbench.py --rows 8192 --which k1 --iters 1 > $O/${TAG}_ncu_k1.log 2>&1
[ -n "$FULL" ] && timeout 600 ncu --set full --clock-control none --import-source on -k regex:ppo_ -c 1 \
  -o $O/${TAG}_k2 -f python tools/kbench.py --rows 8192 --which k2 --iters 1 > $O/${TAG}_ncu_k2.log 2>&1
ls -la $O
