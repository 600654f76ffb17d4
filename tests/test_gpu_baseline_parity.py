"""BASELINE configs end to end against the float64 oracle, at full size.

* cfg1 (BASELINE configs[0], the CPU-reference synthetic case) IN FULL: 64 rollouts,
  lengths ``default_rng(0).integers(128, 2049)`` (T = 70,843), V = 32,000 fp32 logits,
  4 minibatches, budgets C = 8,192 and 32,768, through the public
  ``DecoupledPPOStep.run`` — the call bench.py measures — with the oracle run on the
  host for every micro-batch (trainer.py:285-346 structure, 150-195 per token):
  plan / packing order / advantages bit-exact, counters exact, lp and sums 1e-5
  relative, dlogits element-wise 1e-5 |d| (+ 1e-7 |g| on the token element) on 100%
  of the elements of every micro-batch.  Minibatches 1-3 train under perturbed logits
  (a model that moved after each update), so ratios spread across the clip range.
* cfg3 (V = 152,064, eta = 4 with real version lags up to eta + 1) and cfg4 (GRPO
  group-normalised advantages, versions lagging 0-9 behind, eta_mask = 8): the full
  global batch's plan and advantages against the oracle, then two FULL micro-batches
  (every row, every element) of bf16 logits through K2 at the bf16 bounds.
"""
import numpy as np
import pytest
import torch

import oracle as O
import parity as PY

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2505_24298_b200 import kernels as K
    from paper_2505_24298_b200.hotpath import DecoupledPPOStep, HotPathConfig, PackedRollouts


def _to_host(t, lo, hi):
    return t[lo:hi].double().cpu().numpy()


@pytest.fixture(scope="module")
def cfg1():
    rng = np.random.default_rng(0)
    lengths = rng.integers(128, 2049, size=64)
    bounds = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    T, V = int(bounds[-1]), 32000
    assert T == 70843
    g = torch.Generator(device="cuda").manual_seed(0)
    table = torch.empty(T, V, dtype=torch.float32, device="cuda").normal_(0.0, 2.0, generator=g)
    tokens = rng.integers(0, V, size=T)
    rewards = rng.choice([5.0, -5.0], size=64)
    # prox under the batch-arrival "params" (the table), oracle-side (trainer.py:295)
    prox_ref = PY.oracle_logprobs(lambda lo, hi: _to_host(table, lo, hi), tokens, T)
    behav = prox_ref + rng.normal(0.0, 0.1, size=T)
    yield dict(bounds=bounds, T=T, V=V, table=table, tokens=tokens, rewards=rewards,
               prox=prox_ref, behav=behav)
    del table
    torch.cuda.empty_cache()


@pytest.mark.parametrize("C", [32768, 8192])
def test_cfg1_in_full_through_run(cfg1, C):
    c = cfg1
    bounds, T, tokens, behav, prox_ref = c["bounds"], c["T"], c["tokens"], c["behav"], c["prox"]
    table = c["table"]
    hp = HotPathConfig(minibatches=4, micro_token_budget=C, micro_min_groups=1)
    ro = PackedRollouts.from_host(bounds, tokens, behav, c["rewards"])
    plan = O.train_step_plan(bounds, 4, C, 1)
    adv_ref = O.compute_advantages_ref(c["rewards"], bounds)
    runner = DecoupledPPOStep(hp)
    assert np.array_equal(runner.advantages(ro).cpu().numpy(), adv_ref)  # bit-exact (K3)

    seen, results = {}, {}

    def logits_fn(phase, m, g, rows):
        x = table.index_select(0, rows.long())
        if phase == "train":
            if m > 0:  # the model moved after each minibatch update
                gen = torch.Generator(device="cuda").manual_seed(1000 * m + g)
                x.add_(torch.empty_like(x).normal_(0.0, 0.05 * m, generator=gen))
            seen[(m, g)] = (rows.cpu().numpy(), x)
        return x

    def backward_fn(m, g, dl):
        rows, x = seen.pop((m, g))
        # packed order: group placement order of trainer.py:320, bit-exact
        assert np.array_equal(rows, plan[m]["gather"][g]), (m, g)
        pt = dict(tokens=tokens[rows], behav=behav[rows], prox=prox_ref[rows], adv=adv_ref[rows])
        results[(m, g)] = PY.oracle_rows(lambda lo, hi: _to_host(x, lo, hi), len(rows), pt,
                                         dt="f32", got_rows=lambda lo, hi: _to_host(dl, lo, hi))

    res = runner.run(ro, logits_fn, backward_fn=backward_fn, current_version=0)
    assert res.minibatch_updates == len(plan)
    assert res.microbatches == sum(len(mb["groups"]) for mb in plan) == len(results)
    PY.check_lp(runner.last_prox.cpu().numpy(), prox_ref, what="prox")
    tot = np.zeros(8)
    worst = 0.0
    n_bnd = 0
    for m, mb in enumerate(plan):
        parts = [results[(m, g)] for g in range(len(mb["groups"]))]
        rs = np.sum([p["stats"] for p in parts], axis=0)
        nb = int(sum(p["boundary"].sum() for p in parts))
        got = res.minibatch_stats[m]
        PY.check_counters(got, rs, nb, what=f"minibatch {m}")
        PY.check_sums(got, rs, sum(p["abs_obj"] for p in parts),
                      sum(p["abs_ratio"] for p in parts), what=f"minibatch {m}")
        worst = max(worst, max(p["worst"] for p in parts))
        tot += rs
        n_bnd += nb
    # the step statistics (trainer.py:336-345)
    d = max(tot[1], 1)
    assert res.tokens == T and res.excluded_tokens == int(tot[4])
    assert abs(res.loss - (-tot[0] / d)) <= 1e-5 * max(1.0, abs(tot[0] / d))
    assert abs(res.mean_ratio - tot[3] / d) <= 1e-5
    assert abs(res.clip_fraction - tot[2] / d) <= (n_bnd + 0.5) / d
    # the perturbed minibatches exercise both clip branches
    assert tot[2] > 0 and tot[2] < tot[1]
    print(f"cfg1 C={C}: {res.microbatches} micro-batches, worst dlogits err/bound {worst:.3f}, "
          f"{n_bnd} clip-boundary tokens")


def _versions_with_lags(bounds, rng, current, max_lag):
    """Per-token versions: each trajectory starts ``U{0..max_lag}`` versions behind and its
    tokens' versions rise (non-decreasing) to at most ``current`` (interruptible rollouts
    re-weight mid-trajectory, rollout.py:154-159)."""
    n = len(bounds) - 1
    lens = np.diff(bounds)
    start = current - rng.integers(0, max_lag + 1, size=n)
    out = np.empty(int(bounds[-1]), dtype=np.int32)
    for k in range(n):
        L = int(lens[k])
        if L == 0:
            continue
        steps = rng.integers(0, current - start[k] + 1)
        out[bounds[k]:bounds[k + 1]] = start[k] + (np.arange(L) * (steps + 1)) // L
    return out


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_full_microbatches_vs_oracle(name):
    import bench
    cfg = bench.CONFIGS[name]
    W = bench.workload_arrays(cfg)
    rng = np.random.default_rng(17)
    bounds, T, V = W["bounds"], W["T"], cfg["vocab"]
    current = 100
    if name == "cfg3":   # eta = 4: lags reach eta + 1, those tokens are masked
        eta, max_lag, norm = 4, 5, "global"
    else:                # GRPO, versions 0..9 behind
        eta, max_lag, norm = 8, 9, "group"
    versions = _versions_with_lags(bounds, rng, current, max_lag)
    rewards = W["rewards"] if name == "cfg3" else rng.normal(0.0, 1.0, size=W["n"])
    hp = HotPathConfig(minibatches=cfg["minibatches"], micro_token_budget=cfg["budget"],
                       eta_mask=eta, adv_norm=norm)
    behav0 = np.zeros(T)
    ro = PackedRollouts.from_host(bounds, W["tokens"], behav0, rewards, versions=versions,
                                  group_ids=W["group_ids"] if norm == "group" else None)
    runner = DecoupledPPOStep(hp)
    sp = runner.plan(ro)
    adv = runner.advantages(ro)
    # the whole global batch: plan and packing order bit-exact, advantages
    plan = O.train_step_plan(bounds, cfg["minibatches"], cfg["budget"], 1)
    gather = sp.gather.cpu().numpy()
    assert [mb["traj_ids"] for mb in plan] == sp.items
    for m, mb in enumerate(plan):
        assert int(sp.n_groups[m]) == len(mb["groups"])
        for g, idx in enumerate(mb["gather"]):
            gg = [x for x in sp.micro if x[0] == m and x[1] == g][0]
            assert np.array_equal(gather[gg[2]:gg[3]], idx)
    adv_h = adv.cpu().numpy()
    if norm == "global":
        assert np.array_equal(adv_h, O.compute_advantages_ref(rewards, bounds))
    else:
        raw = np.repeat(rewards, np.diff(bounds))  # the reference's raw (trainer.py:116-118)
        ref_adv = O.normalize_group(raw, bounds, W["group_ids"], 0.0, "token")
        np.testing.assert_allclose(adv_h, ref_adv, rtol=1e-12, atol=1e-12)
    # two FULL micro-batches: the largest of the first and of the last minibatch
    M = len(plan)
    picks = []
    for m in (0, M - 1):  # the largest micro-batch holding tokens past the staleness bound
        cands = sorted((x for x in sp.micro if x[0] == m), key=lambda x: -(x[3] - x[2]))
        stale = [x for x in cands if ((current - versions[gather[x[2]:x[3]]]) > eta).any()]
        picks.append(stale[0])
    tokens_d = ro.tokens
    vers = versions
    for (m, g, lo, hi) in picks:
        rows = sp.gather[lo:hi]
        n = hi - lo
        gen = torch.Generator(device="cuda").manual_seed(31 * m + g)
        x = torch.empty(n, V, dtype=torch.bfloat16, device="cuda").normal_(0.0, 2.0, generator=gen)
        lp0, _ = K.logprob_fwd(x, tokens_d, row_index=rows, with_entropy=False)
        idx = rows.long()
        prox_d = lp0.clone()
        prox_d[idx] += torch.randn(n, dtype=torch.float64, device="cuda", generator=gen) * 0.1
        behav_d = prox_d.clone()
        behav_d[idx] += torch.randn(n, dtype=torch.float64, device="cuda", generator=gen) * 0.2
        lp_d = torch.zeros(T, dtype=torch.float64, device="cuda")
        dl, st = K.ppo_fwd_bwd(x, tokens_d, behav_d, prox_d, adv, versions=ro.versions,
                               current_version=current, eta_mask=eta, row_index=rows,
                               lp_out=lp_d)
        r = rows.cpu().numpy()
        pt = dict(tokens=W["tokens"][r], behav=behav_d.cpu().numpy()[r],
                  prox=prox_d.cpu().numpy()[r], adv=adv_h[r], versions=vers[r])
        ref = PY.oracle_rows(lambda a, b: _to_host(x, a, b), n, pt, dt="bf16",
                             got_rows=lambda a, b: _to_host(dl, a, b),
                             current_version=current, eta_mask=eta)
        s = st.cpu().numpy()
        what = f"{name} minibatch {m} micro {g} ({n} rows)"
        PY.check_counters(s, ref["stats"], int(ref["boundary"].sum()), what=what)
        PY.check_sums(s, ref["stats"], ref["abs_obj"], ref["abs_ratio"], what=what)
        PY.check_lp(lp_d.cpu().numpy()[r], ref["lp"], what=what + " lp")
        assert ref["stats"][5] > 0, "the staleness mask must be exercised"
        print(f"{what}: worst dlogits err/bound {ref['worst']:.3f}, masked {int(s[5])}")
        del x, dl
        torch.cuda.empty_cache()
