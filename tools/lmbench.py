"""Fused LM-head + logprob (K7, tcgen05) vs the materialised path (cuBLAS bf16 GEMM ->
logits [T, V] bf16 -> K1).  python tools/lmbench.py [--rows T] [--vocab V] [--dim d]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_24298_b200 import kernels as K

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=16384)
ap.add_argument("--vocab", type=int, default=151936)
ap.add_argument("--dim", type=int, default=1536)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--which", default="fused,unfused")
ap.add_argument("--cg", type=int, default=0)
a = ap.parse_args()
dev = torch.device("cuda", 0)
T, V, d = a.rows, a.vocab, a.dim
h = torch.randn(T, d, device=dev).to(torch.bfloat16)
w = (torch.randn(V, d, device=dev) / d ** 0.5 * 4).to(torch.bfloat16)
b = torch.randn(V, device=dev)
tok = torch.randint(0, V, (T,), device=dev)
lp = torch.empty(T, dtype=torch.float64, device=dev)
out = dict(rows=T, vocab=V, dim=d, tflop=2 * T * V * d / 1e12)


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / a.iters


behav = torch.full((T,), -12.0, dtype=torch.float64, device=dev)
prox = behav + 0.01
adv = torch.randn(T, dtype=torch.float64, device=dev)

for which in a.which.split(","):
    if which == "fused":
        ms = timeit(lambda: K.linear_logprob_fwd(h, w, tok, bias=b, lp_out=lp, cta_group=a.cg))
    elif which.startswith("ppo"):  # loss + backward through the head, chunked (ppo<chunk>)
        from paper_2505_24298_b200.hotpath import linear_ppo_fwd_bwd
        chunk = int(which[3:] or 8192)
        gw = torch.zeros(V, d, dtype=torch.float32, device=dev)
        gb = torch.zeros(V, dtype=torch.float32, device=dev)
        ms = timeit(lambda: linear_ppo_fwd_bwd(h, w, tok, behav, prox, adv, bias=b,
                                               chunk_tokens=chunk, grad_weight=gw, grad_bias=gb))
        out[which] = dict(ms=ms, tflops_3gemm=6 * T * V * d / ms / 1e9, tok_s=T / ms * 1e3,
                          peak_logits_gb=min(chunk, T) * V * 2 / 1e9)
        continue
    elif which == "gemm":
        ms = timeit(lambda: torch.addmm(b.to(torch.bfloat16), h, w.t()))
    else:
        def unfused():
            logits = torch.addmm(b.to(torch.bfloat16), h, w.t())
            K.logprob_fwd(logits, tok, lp_out=lp, with_entropy=False)
        ms = timeit(unfused)
    out[which] = dict(ms=ms, tflops=2 * T * V * d / ms / 1e9, tok_s=T / ms * 1e3)
print(json.dumps(out))
