"""Drop-in parity: paper_2505_24298_b200.trainer vs the reference's own outputs
(golden vectors from asyncrl's train_step / losses, tests/golden/trainstep.npz)
at the reference's float64 tolerances, plus the reference test semantics
(test_trainer.py:222-349) re-run against the B200 module."""
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from conftest import load_cases

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2505_24298_b200 import trainer as T


def _batch(c):
    rewards = c["rewards"]
    trajs = [SimpleNamespace(reward=SimpleNamespace(reward=float(r)), trajectory_id=k,
                             prompt=SimpleNamespace(id=k)) for k, r in enumerate(rewards)]
    return T.TrainBatch(trajectories=trajs, step_index=0, features=c["features"],
                        tokens=c["tokens"], behavior_logprobs=c["behav"],
                        traj_bounds=c["bounds"])


def test_train_step_matches_reference_golden():
    for c in load_cases("trainstep.npz"):
        batch = _batch(c)
        params = T.VersionedParams(3, c["W"], c["b"])
        opt = T.AdamState.zeros_like(params)
        cfg = T.TrainerConfig(clip_eps=float(c["clip_eps"]), minibatches=int(c["minibatches"]),
                              micro_token_budget=int(c["budget"]),
                              micro_min_groups=int(c["kmin"]),
                              objective="decoupled" if bool(c["decoupled"]) else "naive")
        newp, stats = T.train_step(batch, params, opt, cfg)
        assert np.allclose(batch.prox_logprobs, c["prox"], rtol=0, atol=1e-12)
        assert np.array_equal(batch.advantages, c["adv"])  # bit-exact (numpy pairwise replay)
        assert newp.version == int(c["version_new"])
        assert np.allclose(newp.weights, c["W_new"], rtol=1e-10, atol=1e-12)
        assert np.allclose(newp.bias, c["b_new"], rtol=1e-10, atol=1e-12)
        assert opt.step == int(c["opt_step"])
        assert np.allclose(opt.m_weights, c["m_w"], rtol=1e-9, atol=1e-13)
        assert np.allclose(opt.v_bias, c["v_b"], rtol=1e-9, atol=1e-15)
        ref = c["stats"]
        got = [stats.loss, stats.clip_fraction, stats.mean_ratio, stats.tokens,
               stats.minibatch_updates, stats.microbatches, stats.excluded_tokens]
        assert np.allclose(got, ref, rtol=1e-10, atol=1e-12)


def test_losses_match_reference_golden():
    for c in load_cases("trainstep.npz"):
        for name, fn in (("dec", T.decoupled_ppo_loss), ("nai", T.naive_ppo_loss)):
            batch = _batch(c)
            batch.prox_logprobs = c[f"{name}_prox"]
            T.compute_advantages(batch)
            r = fn(batch, T.VersionedParams(1, c["W"], c["b"]), clip_eps=float(c["clip_eps"]))
            assert r.loss == pytest.approx(float(c[f"{name}_loss"]), rel=1e-11, abs=1e-13)
            assert np.allclose(r.grad.weights, c[f"{name}_gw"], rtol=1e-10, atol=1e-13)
            assert np.allclose(r.grad.bias, c[f"{name}_gb"], rtol=1e-10, atol=1e-13)
            misc = c[f"{name}_misc"]
            assert r.n_tokens == int(misc[0]) and r.excluded == int(misc[3])
            assert r.clip_fraction == pytest.approx(float(misc[1]), abs=1e-12)
            assert r.mean_ratio == pytest.approx(float(misc[2]), rel=1e-11)


def test_loss_requires_prox_and_advantages():
    c = load_cases("trainstep.npz")[0]
    with pytest.raises(T.BatchError):
        T.decoupled_ppo_loss(_batch(c), T.VersionedParams(0, c["W"], c["b"]))


def test_allocate_microbatches_reference_semantics():
    # test_trainer.py:222-267
    lengths = [7, 5, 4, 3, 1]
    plan = T.allocate_microbatches(lengths, capacity=10, min_groups=1)
    assert [[lengths[i] for i in g] for g in plan.groups] == [[7, 3], [5, 4, 1]]
    assert sorted(len(g) for g in T.allocate_microbatches([2, 2], 10, 2).groups) == [1, 1]
    assert T.allocate_microbatches([10], 10, 1).groups == ((0,),)
    with pytest.raises(T.BatchError, match="exceeds capacity"):
        T.allocate_microbatches([11], capacity=10)
    with pytest.raises(T.BatchError, match="positive"):
        T.allocate_microbatches([0, 3], capacity=10)
    with pytest.raises(T.BatchError):
        T.allocate_microbatches([3], capacity=10, min_groups=0)
    rng = np.random.default_rng(7)
    for _ in range(100):
        n = int(rng.integers(1, 40))
        cap = int(rng.integers(8, 64))
        ls = [int(rng.integers(1, cap + 1)) for _ in range(n)]
        k = int(rng.integers(1, 5))
        p = T.allocate_microbatches(ls, cap, k)
        assert sorted(i for g in p.groups for i in g) == list(range(n))
        assert all(sum(ls[i] for i in g) <= cap for g in p.groups)
        assert len(p.groups) >= min(k, n)
    assert T.allocate_microbatches([9, 9, 5, 5, 5, 2, 2, 1], 16, 2) == \
        T.allocate_microbatches([9, 9, 5, 5, 5, 2, 2, 1], 16, 2)


def test_train_step_empty_trajectory_and_minibatch_count():
    # test_trainer.py:270-288, 336-349
    rng = np.random.default_rng(0)
    F, V = 12, 16
    lengths = [0, 1]
    feats = rng.normal(size=(1, F))
    trajs = [SimpleNamespace(reward=SimpleNamespace(reward=r), trajectory_id=k,
                             prompt=SimpleNamespace(id=k)) for k, r in enumerate([-5.0, 5.0])]
    batch = T.TrainBatch(trajs, 0, feats, np.array([2]), np.array([-2.0]),
                         np.array([0, 0, 1]))
    params = T.VersionedParams(0, np.zeros((V, F)), np.zeros(V))
    opt = T.AdamState.zeros_like(params)
    newp, stats = T.train_step(batch, params, opt, T.TrainerConfig(minibatches=2))
    assert stats.tokens == 1 and newp.version == 1 and stats.minibatch_updates == 1
    del lengths


def test_train_step_deterministic():
    c = load_cases("trainstep.npz")[1]
    outs = []
    for _ in range(2):
        params = T.VersionedParams(3, c["W"], c["b"])
        newp, _ = T.train_step(_batch(c), params, T.AdamState.zeros_like(params), T.TrainerConfig())
        outs.append(newp)
    assert np.array_equal(outs[0].weights, outs[1].weights)
    assert np.array_equal(outs[0].bias, outs[1].bias)


def test_surrogate_terms_mirror_matches_loss():
    # _surrogate_terms (trainer.py:150-195) over all tokens == _ppo_loss's raw sums
    c = load_cases("trainstep.npz")[0]
    batch = _batch(c)
    batch.prox_logprobs = c["dec_prox"]
    T.compute_advantages(batch)
    params = T.VersionedParams(1, c["W"], c["b"])
    t = T._surrogate_terms(batch, np.arange(batch.n_tokens), params, float(c["clip_eps"]), True)
    r = T.decoupled_ppo_loss(batch, params, clip_eps=float(c["clip_eps"]))
    n = max(t["n_valid"], 1)
    assert t["n_valid"] == r.n_tokens and t["n_excluded"] == r.excluded
    assert -t["objective_sum"] / n == pytest.approx(r.loss, rel=1e-12, abs=1e-14)
    assert np.allclose(-t["grad_w_sum"] / n, r.grad.weights, rtol=1e-12, atol=1e-15)
    assert np.allclose(c["dec_gw"], r.grad.weights, rtol=1e-10, atol=1e-13)
    empty = T._surrogate_terms(batch, np.zeros(0, dtype=np.int64), params, 0.2, True)
    assert empty["n_valid"] == 0 and empty["objective_sum"] == 0.0
