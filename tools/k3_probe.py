"""K3 at a BASELINE shape for ncu captures: python tools/k3_probe.py [--config cfg2] [--iters 3]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_24298_b200 import kernels as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
W = bench.workload_arrays(bench.CONFIGS[a.config])
dev = torch.device("cuda", 0)
bd = torch.as_tensor(W["bounds"], device=dev)
rw = torch.as_tensor(W["rewards"], device=dev)
out = torch.empty(W["T"], dtype=torch.float64, device=dev)
for _ in range(a.iters):
    K.advantages(rw, bd, W["T"], out=out)
torch.cuda.synchronize()
