"""LM-scale hot path (hotpath.DecoupledPPOStep.run, the call bench.py measures)
vs the oracle's train_step structure (trainer.py:285-346) on given logits."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2505_24298_b200.hotpath import DecoupledPPOStep, HotPathConfig, PackedRollouts


def _setup(n=40, V=2048, lo=5, hi=300, seed=0, dtype=torch.bfloat16):
    rng = np.random.default_rng(seed)
    lengths = rng.integers(lo, hi, size=n)
    lengths[3] = 0  # empty trajectory is skipped (trainer.py:310)
    bounds = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    T = int(bounds[-1])
    g = torch.Generator().manual_seed(seed)
    # one logits row per global token, fixed across phases ("model" output)
    table = (torch.randn(T, V, generator=g, dtype=torch.float64) * 2).to(dtype)
    x64 = table.double().numpy()
    tokens = rng.integers(0, V, size=T)
    lp = O.token_logprobs(x64, tokens)
    behav = lp + rng.normal(0, 0.3, size=T)
    rewards = rng.choice([5.0, -5.0], size=n)
    versions = rng.integers(5, 10, size=T).astype(np.int32)
    return bounds, T, V, table, x64, tokens, behav, rewards, versions


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_run_matches_oracle_minibatch_sums(dtype):
    bounds, T, V, table, x64, tokens, behav, rewards, versions = _setup(dtype=dtype)
    cfg = HotPathConfig(minibatches=3, micro_token_budget=700, micro_min_groups=2,
                        eta_mask=3)
    ro = PackedRollouts.from_host(bounds, tokens, behav, rewards, versions=versions)
    dev_table = table.cuda()
    seen = []

    def logits_fn(phase, m, g, rows):
        seen.append((phase, m, g, rows.numel()))
        return dev_table.index_select(0, rows.long())

    grads = {}

    def backward_fn(m, g, dl):
        grads[(m, g)] = dl.double().cpu().numpy()

    runner = DecoupledPPOStep(cfg)
    res = runner.run(ro, logits_fn, backward_fn=backward_fn, current_version=10)
    plan = O.train_step_plan(bounds, 3, 700, 2)
    adv = O.compute_advantages_ref(rewards, bounds)
    prox = O.token_logprobs(x64, tokens)
    tol = 1e-5 if dtype == torch.float32 else 2e-2
    assert res.minibatch_updates == len(plan)
    assert res.microbatches == sum(len(mb["groups"]) for mb in plan)
    for m, mb in enumerate(plan):
        idx = np.concatenate(mb["gather"])
        ref = O.surrogate_terms(x64[idx], tokens[idx], behav[idx], prox[idx], adv[idx],
                                versions=versions[idx], current_version=10, eta_mask=3)
        got = res.minibatch_stats[m]
        assert got[1] == ref["stats"][1] and got[5] == ref["stats"][5] and got[7] == len(idx)
        assert abs(got[0] - ref["stats"][0]) <= tol * max(1.0, abs(ref["stats"][0]))
        for g, gi in enumerate(mb["gather"]):
            r = O.surrogate_terms(x64[gi], tokens[gi], behav[gi], prox[gi], adv[gi],
                                  versions=versions[gi], current_version=10, eta_mask=3)
            d = grads[(m, g)]
            assert np.allclose(d, r["dlogits"], rtol=tol, atol=tol * 1e-2)
    # prox pass covers every micro-batch before any train-phase forward
    phases = [p for p, *_ in seen]
    assert phases.index("train") == phases.count("prox")


def test_run_rejects_oversized_sequences():
    from paper_2505_24298_b200.trainer import BatchError
    bounds, T, V, table, x64, tokens, behav, rewards, versions = _setup(n=6, V=64, lo=50, hi=90)
    ro = PackedRollouts.from_host(bounds, tokens, behav, rewards)
    with pytest.raises(BatchError, match="exceeds capacity"):
        DecoupledPPOStep(HotPathConfig(micro_token_budget=40)).run(
            ro, lambda *a: None)


def test_run_with_fused_head_prox_matches_logits_path():
    # prox through K7 (hidden states + LM head, no logits) == prox through K1 on the
    # materialised fp32 logits of the same head
    rng = np.random.default_rng(4)
    lengths = rng.integers(20, 400, size=24)
    bounds = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    T, V, d = int(bounds[-1]), 3000, 128
    g = torch.Generator(device="cuda").manual_seed(4)
    H = torch.randn(T, d, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(V, d, device="cuda", generator=g) / d ** 0.5 * 3).to(torch.bfloat16)
    b = torch.randn(V, device="cuda", generator=g)
    table = torch.addmm(b, H.float(), W.float().t())  # fp32 logits of the same head
    tokens = rng.integers(0, V, size=T)
    behav = rng.normal(-8, 0.3, size=T)
    rewards = rng.choice([5.0, -5.0], size=24)
    ro = PackedRollouts.from_host(bounds, tokens, behav, rewards)
    cfg = HotPathConfig(minibatches=2, micro_token_budget=1500)
    outs = []
    for fused in (False, True):
        runner = DecoupledPPOStep(cfg)
        sp = runner.plan(ro)
        if fused:
            prox = runner.prox_logprobs(ro, sp, head_fn=lambda m, g_, rows: (
                H.index_select(0, rows.long()), W, b))
        else:
            prox = runner.prox_logprobs(ro, sp, lambda ph, m, g_, rows: table.index_select(0, rows.long()))
        outs.append(prox)
    torch.testing.assert_close(outs[1], outs[0], rtol=0, atol=2e-4)


def test_emission_logprobs_k1_and_k7():
    from paper_2505_24298_b200.hotpath import emission_logprobs
    g = torch.Generator(device="cuda").manual_seed(9)
    B, V, d = 64, 5000, 256
    H = torch.randn(B, d, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(V, d, device="cuda", generator=g) / 8).to(torch.bfloat16)
    tok = torch.randint(0, V, (B,), device="cuda", generator=g)
    x = H.double() @ W.double().t()
    ref = O.token_logprobs(x.cpu().numpy(), tok.cpu().numpy())
    lp7 = emission_logprobs(tok, hidden=H, weight=W)
    lp1 = emission_logprobs(tok, logits=x.float())
    np.testing.assert_allclose(lp7.cpu().numpy(), ref, atol=2e-4)
    np.testing.assert_allclose(lp1.cpu().numpy(), ref, atol=1e-4)
    with pytest.raises(ValueError):
        emission_logprobs(tok)


def test_pack_trajectories_to_device():
    from types import SimpleNamespace
    from paper_2505_24298_b200.hotpath import pack_trajectories
    rng = np.random.default_rng(3)
    trajs = []
    for k in range(30):
        m = int(rng.integers(0, 50))
        trajs.append(SimpleNamespace(
            trajectory_id=k, prompt=SimpleNamespace(id=100 + k // 3),
            tokens=[int(x) for x in rng.integers(0, 1000, size=m)],
            behavior_logprobs=[float(x) for x in rng.normal(size=m)],
            versions=[7] * m, reward=SimpleNamespace(reward=float(k % 2))))
    ro, host = pack_trajectories(trajs)
    torch.cuda.synchronize()
    assert np.array_equal(ro.tokens.cpu().numpy(), np.concatenate([t.tokens for t in trajs]))
    assert np.array_equal(ro.behav.cpu().numpy(),
                          np.concatenate([t.behavior_logprobs for t in trajs]))
    assert ro.versions is not None and int(ro.versions.sum()) == 7 * ro.n_tokens
    assert ro.group_ids.cpu().tolist() == [k // 3 for k in range(30)]
    assert ro.traj_bounds_host[-1] == ro.n_tokens


def test_failed_plan_keeps_packing_in_bounds():
    """A minibatch whose plan fails (sequence > budget) must still leave K5 a valid
    packing: poison the allocator's recycled memory, fail the plan, and check the
    device is healthy afterwards (regression: K5 read uninitialised plan entries)."""
    from paper_2505_24298_b200.trainer import BatchError
    junk = torch.full((1 << 24,), -7, dtype=torch.int64, device="cuda")
    del junk
    bounds = np.array([0, 50, 5000, 5100, 5200], dtype=np.int64)
    tokens = np.zeros(5200, dtype=np.int64)
    ro = PackedRollouts.from_host(bounds, tokens, np.zeros(5200), np.array([1.0, -1, 1, -1]))
    runner = DecoupledPPOStep(HotPathConfig(minibatches=2, micro_token_budget=1000))
    with pytest.raises(BatchError, match="exceeds capacity"):
        runner.plan(ro)
    torch.cuda.synchronize()
    assert float(torch.ones(4, device="cuda").sum()) == 4.0


def test_fused_first_prox_matches_unfused():
    # fuse_first_prox (K2 computes minibatch 0's prox in its own read of the logits)
    # == the unfused path (K1 prox pass over every micro-batch), same logits
    bounds, T, V, table, x64, tokens, behav, rewards, versions = _setup(seed=5)
    ro = PackedRollouts.from_host(bounds, tokens, behav, rewards, versions=versions)
    dev_table = table.cuda()
    outs = []
    for fuse in (False, True):
        calls = []

        def logits_fn(phase, m, g, rows):
            calls.append((phase, m))
            return dev_table.index_select(0, rows.long())
        cfg = HotPathConfig(minibatches=3, micro_token_budget=700, micro_min_groups=2,
                            fuse_first_prox=fuse)
        runner = DecoupledPPOStep(cfg)
        res = runner.run(ro, logits_fn, current_version=10)
        outs.append((res.minibatch_stats, runner.last_prox.cpu().numpy(), calls))
    (s0, p0, c0), (s1, p1, c1) = outs
    assert not any(ph == "prox" and m == 0 for ph, m in c1)   # no prox forward for minibatch 0
    assert any(ph == "prox" and m == 0 for ph, m in c0)
    counts = [1, 2, 4, 5, 7]
    assert np.array_equal(s0[:, counts], s1[:, counts])
    np.testing.assert_allclose(s1, s0, rtol=2e-2, atol=1e-6)
    np.testing.assert_allclose(p1, p0, rtol=0, atol=2e-5)


def test_run_degenerate_batches():
    """Empty trajectories only, fewer trajectories than minibatches, a single token:
    the step completes with the reference's counts (trainer.py:300-315: empty chunks
    and zero-length trajectories are dropped)."""
    V = 512
    table = torch.randn(4, V, device="cuda").to(torch.bfloat16)
    lf = lambda ph, m, g, rows: table.index_select(0, rows.long())
    # all trajectories empty
    ro = PackedRollouts.from_host(np.array([0, 0, 0], dtype=np.int64), np.zeros(0, np.int64),
                                  np.zeros(0), np.array([1.0, -1.0]))
    res = DecoupledPPOStep(HotPathConfig(minibatches=4)).run(ro, lf)
    assert res.minibatch_updates == 0 and res.tokens == 0
    # 3 trajectories, 4 minibatches (array_split leaves one chunk empty), 4 tokens total
    bounds = np.array([0, 1, 3, 4], dtype=np.int64)
    ro = PackedRollouts.from_host(bounds, np.array([1, 2, 3, 4]), np.full(4, -6.0),
                                  np.array([5.0, -5.0, 5.0]))
    res = DecoupledPPOStep(HotPathConfig(minibatches=4)).run(ro, lf)
    assert res.minibatch_updates == 3 and res.tokens == 4
    assert res.minibatch_stats[:, 7].sum() == 4
