"""Decode-shape benchmark of rollout-side behaviour log-prob recording (SURVEY §8f rank 4,
rollout.py:154-159): one decode step of B live sequences at V = 151,936 bf16.

    python tools/emission_bench.py [--batches 64,256,1024] [--vocab 151936] [--dim 1536]

Per B it reports, each as CUDA-event time per step over --iters steps:
  k1_hbm    K1 alone on logits rotated through > L2 of buffers (HBM-resident logits),
            launched from a CUDA graph (device time, no host overhead): roofline line,
            algorithmic bytes B * (V * 2 + 16); eager_us = the same from Python
  k1_l2hot  K1 on the logits the LM head just wrote (one buffer, L2-resident) — the
            in-engine case, reported without a roofline (L2 is not the HBM bound)
  step      EmissionRecorder.step (append kernel + K1), eager and CUDA-graph replayed
  k7        EmissionRecorder.step from hidden states through the fused head (K7; no
            logits): bound by reading W [V, d] once per step — bytes V * d * 2
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_24298_b200 import _lib  # noqa: E402
if "--lib" in sys.argv:  # a tuning build from tools/variants.py (before the first load)
    _lib.use_library(sys.argv[sys.argv.index("--lib") + 1])
from paper_2505_24298_b200 import kernels as K  # noqa: E402
from paper_2505_24298_b200.hotpath import EmissionRecorder  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="64,256,1024")
ap.add_argument("--vocab", type=int, default=151936)
ap.add_argument("--dim", type=int, default=1536)
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--out", default=None)
ap.add_argument("--lib", default=None, help="a tuning build from tools/variants.py")
a = ap.parse_args()

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
V, d = a.vocab, a.dim
peaks = {}
try:
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "MEASURED_PEAKS.json")) as f:
        peaks = json.load(f)
except OSError:
    pass
hbm_peak = float(peaks.get("hbm_gbs") or 6543.7)
L2 = 126 * 2 ** 20


def timed(fn, iters):
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


lines = []
W = (torch.randn(V, d, device=dev) * 0.02).to(torch.bfloat16)
for B in [int(x) for x in a.batches.split(",")]:
    nbuf = max(2, -(-3 * L2 // (B * V * 2)))
    bufs = [torch.randn(B, V, device=dev).to(torch.bfloat16) for _ in range(nbuf)]
    tok = torch.randint(0, V, (B,), device=dev)
    lp = torch.empty(B, dtype=torch.float64, device=dev)
    it = [0]

    def k1_rot():
        it[0] = (it[0] + 1) % nbuf
        K.logprob_fwd(bufs[it[0]], tok, lp_out=lp, with_entropy=False)

    us_hbm_eager = timed(k1_rot, a.iters)
    # device time without the host: G launches over the rotating buffers in one CUDA graph
    G = 4 * nbuf

    def graph_of(fn):
        st_ = torch.cuda.Stream()
        st_.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st_):
            fn()
        torch.cuda.current_stream().wait_stream(st_)
        torch.cuda.synchronize()
        g_ = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_):
            fn()
        return g_

    def k1_all():
        for i in range(G):
            K.logprob_fwd(bufs[i % nbuf], tok, lp_out=lp, with_entropy=False)
    gk1 = graph_of(k1_all)
    us_hbm = timed(gk1.replay, max(3, a.iters // G)) / G

    def k1_hot_all():
        for i in range(G):
            K.logprob_fwd(bufs[0], tok, lp_out=lp, with_entropy=False)
    us_hot = timed(graph_of(k1_hot_all).replay, max(3, a.iters // G)) / G
    by = B * (V * 2 + 16)
    rec = EmissionRecorder(n_slots=B, max_len=a.iters * 4 + 64, device=dev)
    slots = torch.arange(B, dtype=torch.int32, device=dev)
    rec.set_version(7)
    us_step = timed(lambda: rec.step(slots, tok, logits=bufs[0]), a.iters)
    rec.lengths.zero_()
    # graph: capture one step (version read from the device), replay
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        rec.step(slots, tok, logits=bufs[0])
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        rec.step(slots, tok, logits=bufs[0])
    us_graph = timed(g.replay, a.iters)
    rec.check()
    h = (torch.randn(B, d, device=dev) * 0.5).to(torch.bfloat16)
    rec7 = EmissionRecorder(n_slots=B, max_len=a.iters * 2 + 16, device=dev)
    us_k7 = timed(lambda: rec7.step(slots, tok, 1, hidden=h, weight=W), a.iters)
    rec7.check()
    w_bytes = V * d * 2
    line = {
        "metric": "emission log-prob recording, one decode step", "B": B, "vocab": V,
        "dtype": "bf16",
        "k1_hbm": {"us": us_hbm, "gbs": by / us_hbm / 1e3, "frac": by / us_hbm / 1e3 / hbm_peak,
                   "bytes": by, "rotating_buffers": nbuf, "timing": "CUDA graph of %d launches" % G,
                   "eager_us": us_hbm_eager},
        "k1_l2hot": {"us": us_hot, "gbs_effective": by / us_hot / 1e3},
        "step_eager_us": us_step, "step_graph_us": us_graph, "launches_per_step": 2,
        "k7": {"us": us_k7, "dim": d, "weight_gbs": w_bytes / us_k7 / 1e3,
               "frac": w_bytes / us_k7 / 1e3 / hbm_peak,
               "tflops": 2 * B * V * d / us_k7 / 1e6},
        "hbm_peak_gbs": hbm_peak,
    }
    lines.append(line)
    print(json.dumps(line), flush=True)
    del bufs
if a.out:
    with open(a.out, "w") as f:
        for ln in lines:
            f.write(json.dumps(ln) + "\n")
