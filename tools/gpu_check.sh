#!/bin/bash
# Quick GPU session: full gpu tests, smoke, cfg2 bench, reference arm, 2-rank strong-scaling check.
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke exit $?" >> $O/${TAG}_smoke.log
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
timeout 600 python bench.py --impl reference > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --share-gpu --dist-backend gloo --scaling strong --steps 2 --warmup 3 --no-cpu-baseline \
  > $O/${TAG}_bench_strong2_gloo.json 2> $O/${TAG}_bench_strong2_gloo.err
ls -la $O | tail -20
