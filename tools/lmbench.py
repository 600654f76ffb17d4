"""LM-head benchmarks.  python tools/lmbench.py [--rows T] [--vocab V] [--dim d] [--which ...]

  fused       K7 fused head + log-prob (tcgen05) ...
  unfused     ... vs cuBLAS bf16 GEMM -> logits [T, V] -> K1
  ppo<chunk>  loss + backward through the head (hotpath.linear_ppo_fwd_bwd: the library's
              tcgen05 LOGITS / DHIDDEN / DWEIGHT GEMMs + K2 + colsum), <chunk> tokens per chunk
  cublas<chunk>  the same chunked backward with cuBLAS GEMMs around K2 (round-1 product
              path, kept here only as the comparison arm)
  g_logits / g_dhidden / g_dweight / c_logits / c_dhidden / c_dweight
              one GEMM of the chunk, ours (g_) vs cuBLAS (c_), at T x V x d"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_24298_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None, help="a tuning build from tools/variants.py")
ap.add_argument("--rows", type=int, default=16384)
ap.add_argument("--vocab", type=int, default=151936)
ap.add_argument("--dim", type=int, default=1536)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--which", default="fused,unfused")
ap.add_argument("--cg", type=int, default=0)
ap.add_argument("--tune", action="append", default=[], help="knob=value (areal_set_tuning)")
ap.add_argument("--repeat", type=int, default=1, help="run the --which list this many times, "
                "report the median of each item (power-capped clocks drift)")
ap.add_argument("--cool", type=float, default=0.0, help="idle seconds before each timed item "
                "(sustained GEMM load heats the part and the clocks fall)")
a = ap.parse_args()
if a.lib:
    _lib.use_library(a.lib)
from paper_2505_24298_b200 import kernels as K  # noqa: E402
for kv in a.tune:
    k_, v_ = kv.split("=")
    K.set_tuning(k_, int(v_))
dev = torch.device("cuda", 0)
T, V, d = a.rows, a.vocab, a.dim
h = torch.randn(T, d, device=dev).to(torch.bfloat16)
w = (torch.randn(V, d, device=dev) / d ** 0.5 * 4).to(torch.bfloat16)
b = torch.randn(V, device=dev)
tok = torch.randint(0, V, (T,), device=dev)
lp = torch.empty(T, dtype=torch.float64, device=dev)


def timeit(fn):
    if a.cool > 0:
        import time
        torch.cuda.synchronize()
        time.sleep(a.cool)
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

def run_all():
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
        elif which.startswith("cublas"):  # the round-1 chunked path: cuBLAS GEMMs around K2
            chunk = int(which[6:] or 8192)
            gw = torch.zeros(V, d, dtype=torch.float32, device=dev)
            gb = torch.zeros(V, dtype=torch.float32, device=dev)
            dh = torch.empty_like(h)
            buf = torch.empty((min(chunk, T), V), dtype=h.dtype, device=dev)
            st = torch.zeros(8, dtype=torch.float64, device=dev)
            b16 = b.to(torch.bfloat16)

            def cublas_path():
                for lo in range(0, T, chunk):
                    hi = min(T, lo + chunk)
                    lg = buf[: hi - lo]
                    torch.addmm(b16, h[lo:hi], w.t(), out=lg)
                    K.ppo_fwd_bwd(lg, tok, behav, prox, adv, row_index=torch.arange(
                        lo, hi, dtype=torch.int32, device=dev), dlogits=lg, stats=st)
                    torch.mm(lg, w, out=dh[lo:hi])
                    gw.add_(torch.mm(lg.t(), h[lo:hi], out_dtype=torch.float32))
                    gb.add_(lg.sum(dim=0, dtype=torch.float32))
            ms = timeit(cublas_path)
            out[which] = dict(ms=ms, tflops_3gemm=6 * T * V * d / ms / 1e9, tok_s=T / ms * 1e3)
            continue
        elif which[:2] in ("g_", "c_"):  # one GEMM of the backward at T x V x d
            op = which[2:]
            if not hasattr(a, "_lg"):
                a._lg = torch.randn(T, V, device=dev).to(torch.bfloat16)
            lg = a._lg
            if which[0] == "g":
                fn = {"logits": lambda: K.lm_head_gemm("logits", h, w, lg, bias=b),
                      "dhidden": lambda: K.lm_head_gemm("dhidden", lg, w),
                      "dweight": lambda: K.lm_head_gemm("dweight", lg, h)}[op]
            else:
                b16 = b.to(torch.bfloat16)
                fn = {"logits": lambda: torch.addmm(b16, h, w.t(), out=lg),
                      "dhidden": lambda: torch.mm(lg, w),
                      "dweight": lambda: torch.mm(lg.t(), h, out_dtype=torch.float32)}[op]
            ms = timeit(fn)
            out[which] = dict(ms=ms, tflops=2 * T * V * d / ms / 1e9)
            continue
        elif which == "bwd":  # the grouped backward launch alone (DHIDDEN + DWEIGHT + grad_b)
            if not hasattr(a, "_lg"):
                a._lg = (torch.randn(T, V, device=dev) * 1e-3).to(torch.bfloat16)
            gw = torch.zeros(V, d, dtype=torch.float32, device=dev)
            gb = torch.zeros(V, dtype=torch.float32, device=dev)
            ms = timeit(lambda: K.lm_head_backward(a._lg, h, w, grad_weight=gw, grad_bias=gb))
            ms_nb = timeit(lambda: K.lm_head_backward(a._lg, h, w, grad_weight=gw, with_bias=False))
            out[which] = dict(ms=ms, tflops=4 * T * V * d / ms / 1e9, ms_without_grad_b=ms_nb)
            continue
        elif which in ("k2", "colsum"):  # the non-GEMM launches of the backward at T x V
            if not hasattr(a, "_lg"):
                a._lg = torch.randn(T, V, device=dev).to(torch.bfloat16)
            lg = a._lg
            st = torch.zeros(8, dtype=torch.float64, device=dev)
            fn = (lambda: K.ppo_fwd_bwd(lg, tok, behav, prox, adv, dlogits=lg, stats=st)) if which == "k2" \
                else (lambda: K.colsum(lg))
            ms = timeit(fn)
            out[which] = dict(ms=ms, gbs=(2 if which == "k2" else 1) * T * V * 2 / ms / 1e6)
            continue
        elif which == "gemm":
            ms = timeit(lambda: torch.addmm(b.to(torch.bfloat16), h, w.t()))
        else:
            def unfused():
                logits = torch.addmm(b.to(torch.bfloat16), h, w.t())
                K.logprob_fwd(logits, tok, lp_out=lp, with_entropy=False)
            ms = timeit(unfused)
        out[which] = dict(ms=ms, tflops=2 * T * V * d / ms / 1e9, tok_s=T / ms * 1e3)


runs = []
for _ in range(max(1, a.repeat)):
    out = dict(rows=T, vocab=V, dim=d, tflop=2 * T * V * d / 1e12)
    run_all()
    runs.append(out)
if len(runs) > 1:  # median per item (by ms); the per-run ms lists beside it
    import statistics
    out = dict(runs[0])
    for k_ in runs[0]:
        if isinstance(runs[0][k_], dict) and "ms" in runs[0][k_]:
            ms_all = [r[k_]["ms"] for r in runs]
            med = sorted(runs, key=lambda r: r[k_]["ms"])[len(runs) // 2][k_]
            out[k_] = dict(med, ms_runs=ms_all, ms_min=min(ms_all))
print(json.dumps(out))
