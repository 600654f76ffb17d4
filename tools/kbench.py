"""Kernel micro-benchmark: K1 / K2 on one synthetic micro-batch (used for ncu captures
and tuning).  python tools/kbench.py [--rows R] [--vocab V] [--dtype bf16] [--iters N]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_24298_b200 import kernels as K

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=32768)
ap.add_argument("--vocab", type=int, default=151936)
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--algo", default="auto")
ap.add_argument("--which", default="k1,k2")
ap.add_argument("--lib", default=None, help="a tuning build from tools/variants.py")
ap.add_argument("--tune", action="append", default=[], help="knob=value (areal_set_tuning)")
a = ap.parse_args()
if a.lib:
    from paper_2505_24298_b200 import _lib
    _lib.use_library(a.lib)
for kv in a.tune:
    k_, v_ = kv.split("=")
    K.set_tuning(k_, int(v_))
dt = {"bf16": torch.bfloat16, "f32": torch.float32, "f16": torch.float16, "f64": torch.float64}[a.dtype]
dev = torch.device("cuda", 0)
T, V = a.rows, a.vocab
x = torch.empty(T, V, dtype=dt, device=dev).normal_(0, 2)
dl = torch.empty_like(x)
tok = torch.randint(0, V, (T,), device=dev)
lp, _ = K.logprob_fwd(x, tok, with_entropy=False, algo=a.algo)
behav = lp + 0.1 * torch.randn(T, dtype=torch.float64, device=dev)
adv = torch.randn(T, dtype=torch.float64, device=dev)
stats = torch.zeros(8, dtype=torch.float64, device=dev)
es = x.element_size()
out = {}
for which in a.which.split(","):
    fn = (lambda: K.logprob_fwd(x, tok, lp_out=lp, with_entropy=False, algo=a.algo)) if which == "k1" \
        else (lambda: K.ppo_fwd_bwd(x, tok, behav, lp, adv, dlogits=dl, stats=stats, algo=a.algo))
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.iters
    nbytes = T * (V * es + 16) if which == "k1" else T * (2 * V * es + 52)
    out[which] = dict(ms=ms, gbs=nbytes / ms / 1e6, tok_s=T / ms * 1e3)
print(json.dumps(dict(rows=T, vocab=V, dtype=a.dtype, algo=a.algo, **out)))
