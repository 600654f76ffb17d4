"""Latency of the small kernels (K3 advantages, K4 allocation + packing plan, K5
gather) at BASELINE shapes, next to the oracle (same algorithm as the reference,
numpy / pure Python) on the host CPU.

    python tools/plan_bench.py [--iters 50]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import oracle as O  # noqa: E402
from paper_2505_24298_b200 import kernels as K  # noqa: E402
from paper_2505_24298_b200.trainer import minibatch_items  # noqa: E402


def cuda_time(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    out = {}
    for name in ("cfg1", "cfg2", "cfg3", "cfg5"):
        cfg = bench.CONFIGS[name]
        W = bench.workload_arrays(cfg)
        bounds = W["bounds"]
        T = W["T"]
        bd = torch.as_tensor(bounds, device=dev)
        rw = torch.as_tensor(W["rewards"], device=dev)
        r = {"tokens": T, "rollouts": W["n"]}
        # K3 (reference mode, bit-identical normalisation)
        r["k3_us"] = cuda_time(lambda: K.advantages(rw, bd, T), a.iters)
        t0 = time.perf_counter()
        O.compute_advantages_ref(W["rewards"], bounds)
        r["k3_cpu_oracle_us"] = (time.perf_counter() - t0) * 1e6
        # K4 + K5 for all minibatches of one step
        items = minibatch_items(bounds, cfg["minibatches"])
        mb_off = np.concatenate([[0], np.cumsum([len(x) for x in items])]).astype(np.int32)
        lens = np.diff(bounds)
        mb_tok = [int(lens[x].sum()) for x in items]
        mb_start = np.concatenate([[0], np.cumsum(mb_tok)[:-1]]).astype(np.int64)
        flat = torch.as_tensor(np.concatenate(items).astype(np.int32), device=dev)

        def plan():
            p = K.plan_microbatches(bd, flat, mb_off, mb_start, cfg["budget"], 1)
            K.fill_gather(bd, p, int(sum(mb_tok)))
        r["k4k5_us"] = cuda_time(plan, a.iters)
        t0 = time.perf_counter()
        for x in items:
            O.allocate_microbatches([int(lens[k]) for k in x], cfg["budget"], 1)
        r["k4_cpu_oracle_us"] = (time.perf_counter() - t0) * 1e6
        out[name] = r
    print(json.dumps(out))


if __name__ == "__main__":
    main()
