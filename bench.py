"""Benchmark of the decoupled-PPO training hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg1|cfg2|cfg3|cfg4|cfg5] [--scaling weak|strong]

One step = one pass of the hot path over one synthetic global batch of the
named shape: K3 advantages, K4/K5 allocation + packing of every minibatch, K1
prox log-probs over every token, then per minibatch K2 (fused decoupled-PPO
loss + backward -> dlogits) over every micro-batch and one NCCL all-reduce of
the statistics (N > 1).  The model is out of scope: its logits are synthetic
bf16 tensors resident in HBM (rotating 10 GB buffers, larger than L2, so no L2
flush is needed) handed to the hot path through the same callback a real model
would use.  Prints ONE JSON line on rank 0.

``--impl reference`` times the reference algorithm on the host CPU (the float64
numpy oracle restating trainer.py, all cores) on a bounded sample of the same
workload; only rank 0 works under torchrun.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "packed tokens/sec for logprob+decoupled-PPO fwd/bwd; % HBM roofline"

CONFIGS = {
    # BASELINE.json configs[1]: the headline single-GPU workload
    "cfg2": dict(workload="Qwen2-1.5B shape (BASELINE configs[1])", vocab=151936, rollouts=512,
                 prompts=128, len_lo=128, len_hi=8192, dtype="bf16", budget=32768,
                 minibatches=4, hidden=1536),
    # configs[0]: CPU-reference synthetic case
    "cfg1": dict(workload="CPU-ref synthetic (BASELINE configs[0])", vocab=32000, rollouts=64,
                 prompts=16, len_lo=128, len_hi=2048, dtype="fp32", budget=32768, minibatches=4),
    # configs[2]: Qwen2-7B shape, eta=4 staleness mask
    "cfg3": dict(workload="Qwen2-7B shape (BASELINE configs[2])", vocab=152064, rollouts=1024,
                 prompts=256, len_lo=128, len_hi=27648, dtype="bf16", budget=32768,
                 minibatches=4, eta=4, hidden=3584),
    # configs[3]: GRPO group-normalised advantages, 16 samples/prompt, versions lag 0..8
    "cfg4": dict(workload="GRPO 16 samples/prompt, mixed versions (BASELINE configs[3])",
                 vocab=151936, rollouts=1024, prompts=64, len_lo=128, len_hi=8192, dtype="bf16",
                 budget=32768, minibatches=4, eta=8, adv_norm="group_sequence"),
    # configs[4]: heavy-tailed stress, reference Pareto sampler (timeline.py:84-90)
    "cfg5": dict(workload="stress: 4096 rollouts, Pareto lengths 64-32768 (BASELINE configs[4])",
                 vocab=151936, rollouts=4096, prompts=1024, pareto=(1.2, 64.0, 32768, 64),
                 len_lo=64, len_hi=32768, dtype="bf16", budget=32768, minibatches=4),
}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def _tensor_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", 0.0)) or None, \
            "MEASURED_PEAKS.json bf16_tflops (cuBLAS 8192^3 burst)"
    except Exception:
        return 2250.0, None, "nominal 2.25 PFLOP/s dense bf16"


def fused_head_bench(cfg, dev, iters=5):
    """Auxiliary measurement of K7: the prox pass with the model's
    LM head fused in (hidden [C, d] x W [V, d] -> log-probs, no [C, V] logits), on one
    full micro-batch of the config's shape, against the materialised path (cuBLAS
    bf16 GEMM -> bf16 logits -> K1).  Random hidden states / head weights."""
    import torch
    from paper_2505_24298_b200 import kernels as K
    C, V, d = cfg["budget"], cfg["vocab"], cfg["hidden"]
    g = torch.Generator(device=dev).manual_seed(11)
    h = torch.randn(C, d, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(V, d, device=dev, generator=g) / d ** 0.5 * 4).to(torch.bfloat16)
    b = torch.randn(V, device=dev, generator=g)
    tok = torch.randint(0, V, (C,), device=dev, generator=g)
    lp = torch.empty(C, dtype=torch.float64, device=dev)
    bb = b.to(torch.bfloat16)

    def t(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / iters

    def unfused():
        K.logprob_fwd(torch.addmm(bb, h, w.t()), tok, lp_out=lp, with_entropy=False)

    # interleaved, best of 3 each: both arms see the same (power-capped) thermal state
    fused = base = float("inf")
    for _ in range(3):
        fused = min(fused, t(lambda: K.linear_logprob_fwd(h, w, tok, bias=b, lp_out=lp)))
        base = min(base, t(unfused))
    flop = 2.0 * C * V * d
    peak, sustained, src = _tensor_peak()
    tf = flop / (fused * 1e-3) / 1e12
    return dict(kernel="areal_linear_logprob_fwd (K7, tcgen05 cta_group::2)", tokens=C, vocab=V,
                hidden=d, ms=fused, tokens_per_s=C / (fused * 1e-3), tflops=tf,
                frac_of_peak=tf / peak, peak_tflops=peak, peak_source=src,
                frac_of_sustained=(tf / sustained) if sustained else None,
                unfused_ms=base, unfused="cuBLAS bf16 GEMM -> bf16 logits -> K1",
                timing="interleaved fused/unfused, best of 3 x %d iterations each" % iters,
                speedup_vs_unfused=base / fused)


def head_backward_bench(cfg, dev, iters=2):
    """Auxiliary measurement of K8 (backward half): the loss + backward
    through the LM head on one full micro-batch of the config's shape in 8,192-token
    chunks (hotpath.linear_ppo_fwd_bwd: LOGITS GEMM -> K2 in place -> grouped dH / dW ->
    grad_b, this library's tcgen05 kernels only), against the same chunking with cuBLAS
    GEMMs around K2.  Random hidden states / head weights."""
    import torch
    from paper_2505_24298_b200 import kernels as K
    from paper_2505_24298_b200.hotpath import linear_ppo_fwd_bwd
    C, V, d, chunk = cfg["budget"], cfg["vocab"], cfg["hidden"], 8192
    g = torch.Generator(device=dev).manual_seed(12)
    h = torch.randn(C, d, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(V, d, device=dev, generator=g) / d ** 0.5 * 4).to(torch.bfloat16)
    b = torch.randn(V, device=dev, generator=g)
    tok = torch.randint(0, V, (C,), device=dev, generator=g)
    behav = torch.full((C,), -12.0, dtype=torch.float64, device=dev)
    prox = behav + 0.01
    adv = torch.randn(C, dtype=torch.float64, device=dev, generator=g)
    gw = torch.zeros(V, d, dtype=torch.float32, device=dev)
    gb = torch.zeros(V, dtype=torch.float32, device=dev)
    dh = torch.empty_like(h)
    buf = torch.empty((chunk, V), dtype=h.dtype, device=dev)
    st = torch.zeros(8, dtype=torch.float64, device=dev)
    bb = b.to(torch.bfloat16)

    def ours():
        linear_ppo_fwd_bwd(h, w, tok, behav, prox, adv, bias=b, chunk_tokens=chunk,
                           grad_weight=gw, grad_bias=gb)

    def cublas():
        for lo in range(0, C, chunk):
            hi = min(C, lo + chunk)
            lg = buf[: hi - lo]
            torch.addmm(bb, h[lo:hi], w.t(), out=lg)
            K.ppo_fwd_bwd(lg, tok, behav, prox, adv, row_index=torch.arange(
                lo, hi, dtype=torch.int32, device=dev), dlogits=lg, stats=st)
            torch.mm(lg, w, out=dh[lo:hi])
            gw.add_(torch.mm(lg.t(), h[lo:hi], out_dtype=torch.float32))
            gb.add_(lg.sum(dim=0, dtype=torch.float32))

    def t(fn):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / iters

    mine = base = float("inf")
    for _ in range(2):  # interleaved, best of 2 each: the same (power-capped) thermal state
        mine = min(mine, t(ours))
        base = min(base, t(cublas))
    flop = 6.0 * C * V * d
    return dict(path="hotpath.linear_ppo_fwd_bwd (K8 LOGITS + K2 + grouped dH/dW + colsum)",
                tokens=C, vocab=V, hidden=d, chunk_tokens=chunk, ms=mine,
                tflops_3gemm=flop / (mine * 1e-3) / 1e12, cublas_ms=base,
                cublas="cuBLAS GEMMs (addmm, mm, mm) around the same K2 and column sums",
                speedup_vs_cublas=base / mine,
                timing="interleaved, best of 2 x %d iterations each" % iters)


def lengths_label(cfg) -> str:
    if "pareto" in cfg:
        a, sc, cap, fl = cfg["pareto"]
        return (f"{sc:g} * (1 + Pareto({a:g})) clipped to [1, {cap}], floored at {fl} "
                f"(timeline.py:84-90), seed 0")
    return f"U[{cfg['len_lo']},{cfg['len_hi']}] seed 0"


def workload_arrays(cfg, n_copies=1, seed=0):
    """Synthetic rollouts: lengths U[lo, hi], tokens uniform, rewards +-5, prompt groups."""
    rng = np.random.default_rng(seed)
    n = cfg["rollouts"] * n_copies
    if "pareto" in cfg:  # scale * (1 + pareto(alpha)) clipped to [1, cap], floored (timeline.py:84-90)
        alpha, scale, cap, floor = cfg["pareto"]
        draw = scale * (1.0 + rng.pareto(alpha, size=n))
        lengths = np.maximum(np.minimum(np.maximum(draw, 1.0), cap).astype(np.int64), floor)
    else:
        lengths = rng.integers(cfg["len_lo"], cfg["len_hi"] + 1, size=n)
    bounds = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    T = int(bounds[-1])
    tokens = rng.integers(0, cfg["vocab"], size=T, dtype=np.int64)
    rewards = rng.choice([5.0, -5.0], size=n)
    per = cfg["rollouts"] // cfg["prompts"]
    group_ids = (np.arange(n) // per).astype(np.int32)
    eta = cfg.get("eta", 0)
    start_ver = 100 - rng.integers(0, eta + 1, size=n)
    versions = np.repeat(start_ver, lengths).astype(np.int32)
    return dict(bounds=bounds, tokens=tokens, rewards=rewards, group_ids=group_ids,
                versions=versions, T=T, n=n)


# ------------------------------------------------------------------ CPU reference path
def _ref_log_softmax():
    """policy.log_softmax (policy.py:145-147) from the UNMODIFIED reference install in
    baseline/_ref when present (the reference's own code), else the oracle's restatement
    of it (identical numpy calls).  Returns (fn, source)."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(path, "asyncrl")):
        if path not in sys.path:
            sys.path.insert(0, path)
        try:
            import asyncrl.policy as P
            return P.log_softmax, "asyncrl.policy.log_softmax (baseline/_ref)"
        except Exception:  # pragma: no cover - broken install
            pass
    import oracle as O
    return O.log_softmax, "oracle.log_softmax (restatement of policy.py:145-147)"


def _ref_tokens(log_softmax, x, tok, behav, adv, clip_eps=0.2):
    """The reference's per-token work on given logits, one micro-batch (no entropy):
    trainer.py:128-137 (prox = log_softmax(x)[tok], policy.py:159-163) and then
    trainer.py:163-195 (log_softmax again under the current params, ratios, clip,
    objective, coef, the score residual coef * (onehot - softmax) and the counters).
    The linear model's GEMMs (163's feats @ W.T, 183-184) are the model, out of scope."""
    ar = np.arange(len(tok))
    prox = log_softmax(x)[ar, tok]                                       # 134
    all_lp = log_softmax(x)                                              # 163
    lp = all_lp[ar, tok]
    scale = np.exp(prox - behav)
    ratio = np.exp(lp - prox)
    valid = np.isfinite(scale) & np.isfinite(ratio)
    term_plain = ratio * adv
    term_clip = np.clip(ratio, 1 - clip_eps, 1 + clip_eps) * adv
    objective = np.where(valid, scale * np.minimum(term_plain, term_clip), 0.0)
    take_plain = (term_plain <= term_clip) & valid
    coef = np.where(take_plain, scale * adv * ratio, 0.0)
    resid = -np.exp(all_lp)                                              # 180-182
    resid[ar, tok] += 1.0
    resid *= coef[:, None]
    return (float(objective.sum()), int(np.count_nonzero(valid)),
            int(np.count_nonzero(valid & (term_clip < term_plain))),
            float(np.where(valid, ratio, 0.0).sum()))


def _cpu_worker(job):
    """One process: `rows` tokens of bf16-valued N(0, 2^2) logits, processed in
    micro-batch chunks of `chunk` rows (memory), timed around the reference work only."""
    seed, rows, V, chunk = job
    log_softmax, _ = _ref_log_softmax()
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((rows, V), dtype=np.float32) * 2.0
    x = (x.view(np.uint32) & 0xFFFF0000).view(np.float32).astype(np.float64)  # bf16 values
    tok = rng.integers(0, V, size=rows)
    behav = rng.normal(-12.0, 0.3, size=rows)
    adv = rng.normal(size=rows)
    t0 = time.perf_counter()
    for lo in range(0, rows, chunk):
        hi = min(rows, lo + chunk)
        _ref_tokens(log_softmax, x[lo:hi], tok[lo:hi], behav[lo:hi], adv[lo:hi])
    return rows, time.perf_counter() - t0


def _cpu_model() -> str:
    cpu = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            cpu = next((l.split(":", 1)[1].strip() for l in f if l.startswith("model name")), cpu)
    except OSError:
        pass
    return cpu


def _chunk_rows(V):
    # micro-batch-sized blocks (~256 MB float64 per array; the reference runs a whole
    # micro-batch per call, trainer.py:321) within host memory for one process per core
    return max(1, min(1024, int(256e6 / (V * 8))))


def cpu_rate(V, rows_per_proc, procs):
    """Reference per-token work on `procs` host processes (one per core), each over
    `rows_per_proc` tokens; returns (tokens/s by wall clock, tokens, wall seconds)."""
    chunk = _chunk_rows(V)
    jobs = [(1000 + i, rows_per_proc, V, chunk) for i in range(procs)]
    if procs == 1:
        done, wall = _cpu_worker(jobs[0])
        return done / wall, done, wall
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        pool.map(_cpu_worker, [(7, 1, V, 1)] * procs)  # fork + import warm-up, untimed
        t0 = time.perf_counter()
        res = pool.map(_cpu_worker, jobs)
        wall = time.perf_counter() - t0
    done = sum(r[0] for r in res)
    return done / wall, done, wall


def cpu_baseline(V, target_s=10.0, workers=None):
    """The reference's per-token path (``_ref_tokens``) on the host: 1 core and all cores,
    each on a bounded sample of about target_s seconds."""
    workers = workers or os.cpu_count() or 1
    probe_rows = max(2, _chunk_rows(V))
    r1, _, dt1 = cpu_rate(V, probe_rows, 1)                 # per-core rate probe
    rows1 = int(max(2, min(4096, r1 * target_s)))
    v1, n1, _ = cpu_rate(V, rows1, 1)
    mem_rows = max(1, int(24e9 / (V * 8 * 8) / workers))
    rowsN = int(max(2, min(4096, mem_rows, v1 * target_s)))
    vN, nN, wN = cpu_rate(V, rowsN, workers)
    _, src = _ref_log_softmax()
    return dict(value=vN, unit="tokens/s", cores=workers, kind="port",
                cores_1=v1, cores_all=vN, cpu_model=_cpu_model(), os_cpu_count=os.cpu_count(),
                sample=(f"V={V} bf16-valued logits; 1 core: {n1} tokens; {workers} cores: "
                        f"{nN} tokens ({workers} procs x {rowsN}); per token the reference's "
                        f"2 log-softmax passes (prox trainer.py:134, loss 163), ratios, clip, "
                        f"objective, coef and the score residual (163-195), no entropy; "
                        f"log_softmax = {src}"),
                wall_s=wN)


def cfg1_full_cpu(workers=None):
    """BASELINE configs[0] IN FULL on the host: all 70,843 tokens of cfg1 (V = 32,000,
    seed-0 lengths) through the reference's per-token path, every core."""
    workers = workers or os.cpu_count() or 1
    cfg = CONFIGS["cfg1"]
    T = int(workload_arrays(cfg)["T"])
    per = [T // workers + (1 if i < T % workers else 0) for i in range(workers)]
    chunk = _chunk_rows(cfg["vocab"])
    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as pool:
        pool.map(_cpu_worker, [(7, 1, cfg["vocab"], 1)] * workers)
        t0 = time.perf_counter()
        res = pool.map(_cpu_worker, [(2000 + i, n, cfg["vocab"], chunk)
                                     for i, n in enumerate(per) if n])
        wall = time.perf_counter() - t0
    done = sum(r[0] for r in res)
    return dict(tokens=done, wall_s=wall, tokens_per_s=done / wall, cores=workers,
                note="cfg1 in full (no sampling, no extrapolation)")


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    V = cfg["vocab"]
    workers = os.cpu_count() or 1
    # 1-core figure (bounded sample) once; each step is an all-core bounded sample
    r1, _, _ = cpu_rate(V, max(2, _chunk_rows(V)), 1)
    rows1 = int(max(2, min(4096, r1 * args.ref_seconds)))
    v1, n1, _ = cpu_rate(V, rows1, 1)
    mem_rows = max(1, int(24e9 / (V * 8 * 8) / workers))
    rowsN = int(max(2, min(4096, mem_rows, v1 * args.ref_seconds)))
    times, vals, toks = [], [], 0
    for i in range(args.warmup + args.steps):
        vN, nN, wN = cpu_rate(V, rowsN, workers)
        if i >= args.warmup:
            times.append(wN)
            vals.append(vN)
            toks = nN
    value = float(np.mean(vals))
    _, src = _ref_log_softmax()
    full = cfg1_full_cpu(workers) if not args.no_cfg1_full else None
    line = dict(metric=METRIC, value=value, unit="tokens/s", n_gpus=args.gpus, steps=args.steps,
                warmup=args.warmup, ms_per_step=1e3 * float(np.mean(times)),
                higher_is_better=True, scaling="weak", vs_baseline=None, dtype="f64",
                data="synthetic", impl="reference",
                config=dict(workload=cfg["workload"], vocab=V,
                            note=f"each step: {toks} tokens ({workers} procs x {rowsN}) of the "
                                 f"config's logits shape, a bounded sample"),
                cpu_baseline=dict(value=value, unit="tokens/s", cores=workers, kind="port",
                                  cores_1=v1, cores_all=value, cpu_model=_cpu_model(),
                                  sample=(f"{toks} tokens per step on {workers} cores, {n1} on "
                                          f"1 core; per token the reference's 2 log-softmax "
                                          f"passes (trainer.py:134, 163), ratios, clip, "
                                          f"objective, coef, score residual (163-195), no "
                                          f"entropy; log_softmax = {src}")),
                cfg1_full=full,
                e2e=dict(value=value, unit="tokens/s", h2d_bytes_per_step=0,
                         d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}",
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["nvidia-smi unavailable"], samples=0)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        return dict(sm_mhz=float(np.median(sm)) if sm else None,
                    sm_max_mhz=max(mx) if mx else None, reasons=reasons, samples=len(self.rows))


# ------------------------------------------------------------------ our arm
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_base = cpu_baseline(cfg["vocab"], target_s=args.cpu_seconds)  # before CUDA init
        cpu_base.pop("wall_s", None)

    # --dist-backend gloo --share-gpu: several ranks on one GPU (a functional check of
    # the multi-rank path on a 1-GPU box; NCCL refuses duplicate GPUs)
    local_dev = 0 if args.share_gpu else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if args.dist_backend == "nccl":
            # the communicator's own report (ranks, NVLS/NVLink transport) on stderr
            if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
                os.environ["NCCL_DEBUG"] = "INFO"
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,ENV")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    from paper_2505_24298_b200 import kernels as K
    from paper_2505_24298_b200.hotpath import (DecoupledPPOStep, HostRollouts, HotPathConfig,
                                               PackedRollouts, load_summary)

    # weak scaling: the global batch is N copies of the config's batch shape; strong:
    # the config's batch itself, split over the N ranks
    strong = args.scaling == "strong"
    W = workload_arrays(cfg, n_copies=1 if strong else world)
    V = cfg["vocab"]
    ldt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    C = cfg["budget"]
    hp = HotPathConfig(minibatches=cfg["minibatches"], micro_token_budget=C,
                       micro_min_groups=max(1, world), eta_mask=cfg.get("eta", -1),
                       adv_norm=cfg.get("adv_norm", "global"))
    runner = DecoupledPPOStep(hp, dev)

    # synthetic model outputs: rotating logits buffers (> L2) + one dlogits buffer
    n_buf = args.logit_buffers
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    bufs = []
    for _ in range(n_buf):
        b = torch.empty((C, V), dtype=ldt, device=dev)
        b.normal_(0.0, 2.0, generator=gen)
        bufs.append(b)
    dl_buf = torch.empty((C, V), dtype=ldt, device=dev)
    counter = [0]
    micro_id = {}

    def logits_fn(phase, m, g, rows):
        # the same micro-batch sees the same synthetic logits in the prox and train
        # phases (a model whose weights did not move); micro-batches rotate buffers
        key = (m, g)
        if key not in micro_id:
            micro_id[key] = len(micro_id)
        counter[0] += 1
        return bufs[micro_id[key] % n_buf][: rows.numel()]

    def dlogits_fn(m, g, logits):
        return dl_buf[: logits.shape[0]]

    # pinned host copies (e2e path) and device-resident copies (value path)
    pin = lambda a: torch.from_numpy(a).pin_memory()
    host = dict(traj_bounds=pin(W["bounds"]), tokens=pin(W["tokens"]),
                behav=pin(np.zeros(W["T"])), rewards=pin(W["rewards"]),
                versions=pin(W["versions"]) if "eta" in cfg else None,
                group_ids=pin(W["group_ids"]) if cfg.get("adv_norm", "").startswith("group")
                else None)
    ro = PackedRollouts.from_host(**host, device=dev)
    torch.cuda.synchronize()

    def step(r):
        counter[0] = 0
        return runner.run(r, logits_fn, dlogits_fn=dlogits_fn, current_version=100)

    # one pass to get prox under the synthetic logits, then behaviour = prox + noise
    runner.record_events = False
    sp = runner.plan(ro)
    counter[0] = 0
    prox = runner.prox_logprobs(ro, sp, logits_fn)
    if world > 1:
        dist.all_reduce(prox)  # each token's prox lives on one rank (others hold garbage)
    noise = torch.randn(W["T"], dtype=torch.float64, device=dev,
                        generator=torch.Generator(device=dev).manual_seed(7)) * 0.1
    behav = prox + noise
    ro.behav.copy_(behav)
    host["behav"].copy_(behav.cpu())
    torch.cuda.synchronize()

    for i in range(args.warmup):
        runner.record_events = i == args.warmup - 1  # fills the runner's timing-event pool
        step(ro)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---------------- timed region: device-resident inputs
    runner.launches = 0
    runner.reset_events()
    runner.k1_bytes = runner.k2_bytes = 0
    runner.record_events = True
    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_dev) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s_ev.record()
        for _ in range(args.steps):
            res = step(ro)
        e_ev.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    runner.record_events = False
    ms = s_ev.elapsed_time(e_ev) / args.steps
    launches = runner.launches  # all K steps of the timed region
    k2_ms = sum(s.elapsed_time(e) for s, e in runner.k2_events)
    k1_ms = sum(s.elapsed_time(e) for s, e in runner.k1_events)
    k3_ms = sum(s.elapsed_time(e) for s, e in runner.k3_events)
    k45_ms = sum(s.elapsed_time(e) for s, e in runner.k45_events)
    k2_bytes, k1_bytes = runner.k2_bytes, runner.k1_bytes
    n_k2 = len(runner.k2_events)
    # K3 device time alone (the in-step events also hold the host's launch overhead of a
    # sub-100 us kernel): 20 back-to-back launches on the step's rollouts
    k3_s, k3_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    runner.advantages(ro)
    torch.cuda.synchronize()
    k3_s.record()
    for _ in range(20):
        runner.advantages(ro)
    k3_e.record()
    torch.cuda.synchronize()
    k3_kernel_us = 1e3 * k3_s.elapsed_time(k3_e) / 20

    # ---------------- e2e: public API with pinned host inputs and a D2H of the result
    e2e_steps = max(1, args.e2e_steps)
    res_host = torch.empty((cfg["minibatches"], 8), dtype=torch.float64).pin_memory()
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # pinned host rollouts: run() uploads the trajectory-level arrays and, per rank, only
    # the per-token arrays of the trajectories in that rank's micro-batches
    host_ro = HostRollouts(**host)
    step(host_ro)  # untimed e2e warm-up
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s2.record()
    h2d = d2h = 0
    for _ in range(e2e_steps):
        out = step(host_ro)  # returns host stats (one D2H of the minibatch sums)
        h2d = runner.h2d_bytes
        d2h = out.minibatch_stats.nbytes
    e2.record()
    torch.cuda.synchronize()
    e2e_ms = s2.elapsed_time(e2) / e2e_steps
    del res_host

    t_max = torch.tensor([ms, e2e_ms, k2_ms, k1_ms, h2d], dtype=torch.float64, device=dev)
    job_bytes = torch.tensor([float(k1_bytes + k2_bytes)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        dist.all_reduce(job_bytes)
    ms, e2e_ms = float(t_max[0]), float(t_max[1])
    h2d_max = int(t_max[4])
    job_bytes = float(job_bytes[0]) / args.steps  # algorithmic K1 + K2 bytes, all ranks
    comm = None
    if world > 1:
        comm = dict(backend=dist.get_backend(), world_size=dist.get_world_size(),
                    nccl_debug=os.environ.get("NCCL_DEBUG"))
    T = W["T"]
    if rank == 0:
        peak, peak_src = _peaks()
        k2_gbs = (k2_bytes / (k2_ms * 1e-3)) / 1e9 if k2_ms > 0 else 0.0
        k1_gbs = (k1_bytes / (k1_ms * 1e-3)) / 1e9 if k1_ms > 0 else 0.0
        # DRAM bytes per token of K2 from the committed ncu --set full capture, scaled
        # to this run's average launch
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            try:
                with open(tp) as f:
                    tj = json.load(f)
                key = f"k2_{cfg['dtype']}_V{V}_dram_bytes_per_token"
                if key in tj and n_k2:
                    traffic = tj[key] * (k2_bytes / (2 * V * (2 if ldt == torch.bfloat16 else 4) + 52)) / n_k2
            except Exception:
                traffic = None
        es = 2 if ldt == torch.bfloat16 else 4
        line = dict(
            metric=METRIC, value=T / (ms * 1e-3), unit="tokens/s", n_gpus=world,
            steps=args.steps, warmup=args.warmup, ms_per_step=ms, higher_is_better=True,
            scaling=args.scaling, vs_baseline=None, dtype=cfg["dtype"],
            data="synthetic (random bf16 logits in rotating HBM buffers; rollouts seeded)",
            config=dict(workload=cfg["workload"], vocab=V, rollouts=W["n"], tokens=T,
                        lengths=lengths_label(cfg),
                        micro_token_budget=C, minibatches=cfg["minibatches"],
                        micro_min_groups=hp.micro_min_groups, logits_dtype=cfg["dtype"],
                        l2="inputs > L2: %d rotating %.1f GB logits buffers" % (
                            n_buf, C * V * es / 1e9),
                        parallelism=f"dp{world}", micro_batches=res.microbatches),
            roofline=dict(bound="hbm", kernel="areal_ppo_fwd_bwd (K2, %s)" % (
                              "ppo_tmem_kernel" if V * es > 220 * 1024 else "ppo_ring_kernel"),
                          achieved=k2_gbs, peak=peak, unit="GB/s", frac=k2_gbs / peak,
                          traffic=traffic, peak_source=peak_src,
                          algorithmic_bytes_per_token=2 * V * es + 52,
                          launches=n_k2, avg_launch_ms=k2_ms / max(n_k2, 1),
                          nominal_peak_gbs=8000.0, frac_of_nominal=k2_gbs / 8000.0),
            k1=dict(kernel="areal_logprob_fwd (K1)", achieved_gbs=k1_gbs, frac=k1_gbs / peak,
                    bytes_per_token=V * es + 16, ms_per_step=k1_ms / args.steps),
            k2=dict(ms_per_step=k2_ms / args.steps, tokens_per_s=T / (k2_ms / args.steps * 1e-3)),
            k3=dict(kernel="areal_advantages (K3)", us_per_step=1e3 * k3_ms / args.steps,
                    kernel_us=k3_kernel_us, mode=hp.adv_mode, norm=hp.adv_norm,
                    note="us_per_step: in-step events incl. the host launch; kernel_us: "
                         "back-to-back launches (one cooperative kernel in reference mode)"),
            k4_k5=dict(kernel="areal_plan_microbatches + areal_fill_gather (K4/K5)",
                       us_per_step=1e3 * k45_ms / args.steps,
                       note="all minibatches' allocation + packing plan, including the one "
                            "small device->host read of the plan that sizes the model calls"),
            e2e=dict(value=T / (e2e_ms * 1e-3), unit="tokens/s", h2d_bytes_per_step=h2d,
                     d2h_bytes_per_step=d2h,
                     note="public API DecoupledPPOStep.run(HostRollouts) from pinned host "
                          "rollouts (per-token arrays uploaded only for this rank's "
                          "micro-batches; bytes of rank 0); logits are device-resident "
                          "model outputs"),
            step_roofline=dict(
                bound="hbm", bytes_per_step=job_bytes, unit="GB/s",
                achieved=job_bytes / (ms * 1e-3) / 1e9 / world, peak=peak,
                frac=job_bytes / (ms * 1e-3) / 1e9 / world / peak,
                note="whole step (K1 + K2 algorithmic bytes; K3/K4/K5 and the host work "
                     "between launches count as time) per GPU against the copy peak"),
            data_parallel=dict(world_size=world, scaling=args.scaling, comm=comm,
                               **load_summary(runner.last_plan.load if runner.last_plan
                                              else None),
                               h2d_bytes_per_step_max_rank=h2d_max,
                               note="micro-batches dealt longest-first by tokens; "
                                    "efficiency_bound = sum_m mean / sum_m max rank load"),
            gpu_launches=launches,
            gpu_launches_per_step=launches // args.steps,
            clocks=clk.summary(),
            cpu_baseline=cpu_base,
            loss=res.loss, clip_fraction=res.clip_fraction,
        )
        if world == 1 and "hidden" in cfg and not args.no_fused_head:
            line["fused_head"] = fused_head_bench(cfg, dev)
        if world == 1 and "hidden" in cfg and not args.no_head_backward:
            line["head_backward"] = head_backward_bench(cfg, dev)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: cfg2 (BASELINE configs[1]) for weak scaling, cfg3 "
                         "(configs[2], the 1/2/4/8-GPU batch) for strong scaling")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: the global batch is N copies of the config's batch; strong: "
                         "the config's batch split over the N ranks")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--logit-buffers", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-seconds", type=float, default=6.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cfg1-full", action="store_true",
                    help="reference arm: skip the full cfg1 run on all host cores")
    ap.add_argument("--no-fused-head", action="store_true",
                    help="skip the auxiliary K7 fused LM-head measurement")
    ap.add_argument("--no-head-backward", action="store_true",
                    help="skip the auxiliary K8 loss + backward through the LM head measurement")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--share-gpu", action="store_true",
                    help="all ranks on cuda:0 (functional multi-rank check on one GPU)")
    ap.add_argument("--lib", default=None,
                    help="tuning only: a compile-time variant from tools/variants.py")
    args = ap.parse_args()
    if args.lib:
        from paper_2505_24298_b200 import _lib
        _lib.use_library(args.lib)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.config is None:
        args.config = "cfg3" if args.scaling == "strong" else "cfg2"
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
