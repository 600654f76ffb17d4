"""Sustained (power-capped) bandwidth: torch copy vs K1 / K2 over ~4 s each, CUDA events.
MEASURED_PEAKS.json's hbm_gbs is a best-of-10 burst; inside bench.py's ~2 s timed region
the GPU runs at its power cap, so this is the like-for-like denominator.
    python tools/sustained.py [--lib build/variants/libareal_b200_X.so] [--which copy,k1,k2]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2505_24298_b200 import _lib
ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None, help="a tuning build from tools/variants.py")
ap.add_argument("--which", default="copy,k1,k2")
ap.add_argument("--seconds", type=float, default=4.0)
ap.add_argument("--rows", type=int, default=32768)
ap.add_argument("--k2-variant", default="plain",
                help="plain | gather (row_index permutation) | step (gather + versions + eta mask)")
args = ap.parse_args()
if args.lib:
    _lib.use_library(args.lib)
from paper_2505_24298_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda", 0)
T, V = args.rows, 151936
x = torch.empty(T, V, dtype=torch.bfloat16, device=dev).normal_(0, 2)
y = torch.empty_like(x)
tok = torch.randint(0, V, (T,), device=dev)
lp, _ = K.logprob_fwd(x, tok, with_entropy=False)
behav = lp + 0.1
adv = torch.randn(T, dtype=torch.float64, device=dev)
stats = torch.zeros(8, dtype=torch.float64, device=dev)
nbytes = x.numel() * 2


from bench import ClockSampler  # noqa: E402


def run(fn, seconds=None):
    seconds = seconds or args.seconds
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); fn(); e.record(); torch.cuda.synchronize()
    n = max(3, int(seconds * 1e3 / s.elapsed_time(e)))
    with ClockSampler(0) as clk:
        s.record()
        for _ in range(n):
            fn()
        e.record(); torch.cuda.synchronize()
    c = clk.summary()
    run.last_clock = dict(sm_mhz=c["sm_mhz"], reasons=c["reasons"],
                          power_w=float(np.median([float(r[2]) for r in clk.rows])) if clk.rows else None)
    return s.elapsed_time(e) / n, n


out = {"lib": args.lib, "rows": T, "k2_variant": args.k2_variant}
which = args.which.split(",")
if "copy" in which:
    ms, n = run(lambda: y.copy_(x))
    out["copy"] = dict(ms=ms, iters=n, gbs=2 * nbytes / ms / 1e6, **run.last_clock)
if "k1" in which:
    ms, n = run(lambda: K.logprob_fwd(x, tok, lp_out=lp, with_entropy=False))
    out["k1"] = dict(ms=ms, iters=n, gbs=T * (V * 2 + 16) / ms / 1e6, **run.last_clock)
if "k2" in which:
    kw = {}
    if args.k2_variant in ("gather", "step"):
        kw["row_index"] = torch.randperm(T, device=dev).to(torch.int32)
    if args.k2_variant == "step":
        kw.update(versions=torch.randint(90, 101, (T,), dtype=torch.int32, device=dev),
                  current_version=100, eta_mask=8)
    ms, n = run(lambda: K.ppo_fwd_bwd(x, tok, behav, lp, adv, dlogits=y, stats=stats, **kw))
    out["k2"] = dict(ms=ms, iters=n, gbs=T * (2 * V * 2 + 52) / ms / 1e6, **run.last_clock)
if "copy" in which:
    ms, n = run(lambda: y.copy_(x))
    out["copy_again"] = dict(ms=ms, iters=n, gbs=2 * nbytes / ms / 1e6, **run.last_clock)
    if "k2" in which:
        out["k2_frac_of_sustained_copy"] = out["k2"]["gbs"] / max(out["copy"]["gbs"],
                                                                  out["copy_again"]["gbs"])
print(json.dumps(out))
