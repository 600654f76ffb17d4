"""Data-parallel hot path on the GPU: DecoupledPPOStep.run with world_size 2 (two
processes sharing cuda:0, gloo for the one collective — NCCL refuses two ranks on
one device; the box has one GPU) against the single-process run of the SAME global
batch.  SURVEY 8e: replicated K4 plan, LPT micro-batch dealing, one all-reduce of
the 8 statistics per minibatch; prox is written by exactly one rank per token."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as tmp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _batch(seed=0, n=48, V=4096):
    rng = np.random.default_rng(seed)
    lengths = rng.integers(10, 500, size=n)
    bounds = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    T = int(bounds[-1])
    tokens = rng.integers(0, V, size=T)
    behav = rng.normal(-8.3, 0.3, size=T)
    rewards = rng.choice([5.0, -5.0], size=n)
    versions = rng.integers(95, 101, size=T).astype(np.int32)
    return bounds, tokens, behav, rewards, versions, T, V


def _run(world, rank, port=None, q=None):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2505_24298_b200.hotpath import DecoupledPPOStep, HotPathConfig, PackedRollouts
        bounds, tokens, behav, rewards, versions, T, V = _batch()
        g = torch.Generator(device="cuda").manual_seed(123)
        table = (torch.randn(T, V, device="cuda", generator=g) * 2).to(torch.bfloat16)
        cfg = HotPathConfig(minibatches=3, micro_token_budget=1500, micro_min_groups=2,
                            eta_mask=3)
        ro = PackedRollouts.from_host(bounds, tokens, behav, rewards, versions=versions)
        runner = DecoupledPPOStep(cfg)
        sp = runner.plan(ro)
        prox = runner.prox_logprobs(ro, sp, lambda ph, m, g_, rows: table.index_select(0, rows.long()))
        if world > 1:
            pc = prox.cpu()
            dist.all_reduce(pc)
            prox = pc.cuda()
        lf = lambda ph, m, g_, rows: table.index_select(0, rows.long())
        res = runner.run(ro, lf, current_version=100)
        # the e2e form: pinned host rollouts, per-token arrays uploaded only for the
        # trajectories of this rank's micro-batches (strong scaling: the batch is split)
        from paper_2505_24298_b200.hotpath import HostRollouts
        host = HostRollouts.from_arrays(bounds, tokens, behav, rewards, versions=versions)
        res_h = runner.run(host, lf, current_version=100)
        meta = 8 * (len(bounds) + len(rewards))
        out = (res.minibatch_stats, prox.cpu().numpy(), [len(x) for x in sp.mine], res.microbatches,
               res_h.minibatch_stats, runner.h2d_bytes - meta, T)
        if q is not None:
            q.put((rank, out))
        return out
    finally:
        if world > 1:
            dist.destroy_process_group()


def test_two_ranks_match_single_rank():
    single = _run(1, 0)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_run, args=(2, r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    st0, prox0, mine0, micro0, sth0, tok_bytes0, T = res[0]
    st1, prox1, mine1, _, sth1, tok_bytes1, _ = res[1]
    st, prox, _, micro, sth, tok_bytes, _ = single
    # host-rollout runs reproduce the device-resident runs bitwise; per-token uploads
    # partition the batch between the ranks (8 + 8 + 4 bytes per token)
    assert np.array_equal(sth0, st0) and np.array_equal(sth1, st1) and np.array_equal(sth, st)
    assert tok_bytes == 20 * T and tok_bytes0 + tok_bytes1 == 20 * T
    assert 0 < tok_bytes0 < 20 * T and 0 < tok_bytes1 < 20 * T
    assert np.array_equal(st0, st1)                 # every rank holds the same all-reduced sums
    assert np.array_equal(prox0, prox)              # each token's prox comes from one rank, bitwise
    assert micro0 == micro                          # same replicated plan
    assert all(a >= 1 and b >= 1 for a, b in zip(mine0, mine1))  # k_min = 2: both ranks busy
    counts = [1, 2, 4, 5, 7]                        # n_valid, n_clipped, n_excluded, n_masked, n_tokens
    assert np.array_equal(st0[:, counts], st[:, counts])
    np.testing.assert_allclose(st0, st, rtol=1e-12, atol=1e-12)  # fp64 sums, different order
