"""K2 timing on different logits distributions / in-place (lm-head backward investigation).
python tools/k2_probe.py [--rows 32768]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_24298_b200 import kernels as K
ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=32768)
ap.add_argument("--vocab", type=int, default=151936)
a = ap.parse_args()
dev = torch.device("cuda", 0)
T, V = a.rows, a.vocab
tok = torch.randint(0, V, (T,), device=dev)
adv = torch.randn(T, dtype=torch.float64, device=dev)
st = torch.zeros(8, dtype=torch.float64, device=dev)


def timeit(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


out = {}
for name, std in (("randn_std2", 2.0), ("randn_std4", 4.0), ("randn_std8", 8.0)):
    x = (torch.randn(T, V, device=dev) * std).to(torch.bfloat16)
    dl = torch.empty_like(x)
    lp, _ = K.logprob_fwd(x, tok, with_entropy=False)
    for bname, behav in (("behav_near", lp + 0.1), ("behav_-12", torch.full_like(lp, -12.0))):
        prox = behav + 0.01 if bname == "behav_-12" else lp
        ms = timeit(lambda: K.ppo_fwd_bwd(x, tok, behav, prox, adv, dlogits=dl, stats=st))
        out[f"{name}/{bname}/oop"] = ms
    xs = x.clone()
    ms = timeit(lambda: (x.copy_(xs), K.ppo_fwd_bwd(x, tok, lp + 0.1, lp, adv, dlogits=x, stats=st)))
    cp = timeit(lambda: x.copy_(xs))
    out[f"{name}/inplace_fresh(minus copy)"] = ms - cp
    del x, dl, xs
print(json.dumps(out, indent=0))
