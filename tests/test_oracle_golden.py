"""Pin the CPU oracle to the reference (CPU only, no GPU).

Golden vectors come from running the real reference (tests/golden/make_golden.py);
the hand cases are the reference tests' own KATs (cited per test).
"""
import math

import numpy as np
import pytest

from conftest import load_cases
import oracle as O


# ------------------------------------------------------------------ golden
def test_surrogate_matches_reference_golden():
    for c in load_cases("surrogate.npz"):
        dec = bool(c["decoupled"])
        t = O.surrogate_terms(c["logits"], c["tokens"], c["behav"], c["prox"], c["adv"],
                              float(c["eps"]), dec)
        s = t["stats"]
        assert np.allclose(t["lp"], c["lp"], rtol=0, atol=1e-12)
        assert s[0] == pytest.approx(float(c["objective_sum"]), rel=1e-12, abs=1e-12)
        assert int(s[1]) == int(c["n_valid"])
        assert int(s[2]) == int(c["n_clipped"])
        assert s[3] == pytest.approx(float(c["ratio_sum"]), rel=1e-12)
        assert int(s[4]) == int(c["n_excluded"])
        # dlogits (g = 1) is minus the reference's residual
        assert np.allclose(t["dlogits"], -c["resid"], rtol=1e-12, atol=1e-13)
        n = max(int(s[1]), 1)
        assert -s[0] / n == pytest.approx(float(c["loss"]), rel=1e-12, abs=1e-14)


def test_advantages_bit_exact_vs_reference_golden():
    for c in load_cases("advantages.npz"):
        adv = O.compute_advantages_ref(c["rewards"], c["bounds"])
        assert np.array_equal(adv, c["adv"])  # same numpy calls: bit-exact


def test_allocator_bit_exact_vs_reference_golden():
    for c in load_cases("allocator.npz"):
        groups = O.allocate_microbatches(c["lengths"], int(c["cap"]), int(c["kmin"]))
        gid = np.full(len(c["lengths"]), -1)
        slot = np.full(len(c["lengths"]), -1)
        for g, members in enumerate(groups):
            for s, i in enumerate(members):
                gid[i], slot[i] = g, s
        assert np.array_equal(gid, c["gid"]) and np.array_equal(slot, c["slot"])


def test_linear_train_step_matches_reference_golden():
    for c in load_cases("trainstep.npz"):
        W, b, opt, stats, prox, adv = O.linear_train_step(
            c["features"], c["tokens"], c["behav"], c["bounds"], c["rewards"], c["W"], c["b"],
            clip_eps=float(c["clip_eps"]), minibatches=int(c["minibatches"]),
            capacity=int(c["budget"]), min_groups=int(c["kmin"]),
            decoupled=bool(c["decoupled"]))
        assert np.allclose(prox, c["prox"], rtol=0, atol=1e-12)
        assert np.array_equal(adv, c["adv"])
        assert np.allclose(W, c["W_new"], rtol=1e-10, atol=1e-12)
        assert np.allclose(b, c["b_new"], rtol=1e-10, atol=1e-12)
        assert opt[4] == int(c["opt_step"])
        ref = c["stats"]
        got = [stats["loss"], stats["clip_fraction"], stats["mean_ratio"], stats["tokens"],
               stats["minibatch_updates"], stats["microbatches"], stats["excluded_tokens"]]
        assert np.allclose(got, ref, rtol=1e-10, atol=1e-12)


def test_linear_loss_matches_reference_golden():
    for c in load_cases("trainstep.npz"):
        for name, dec in (("dec", True), ("nai", False)):
            adv = O.compute_advantages_ref(c["rewards"], c["bounds"])
            r = O.linear_loss(c["features"], c["tokens"], c["behav"], c[f"{name}_prox"], adv,
                              c["W"], c["b"], float(c["clip_eps"]), dec)
            assert r["loss"] == pytest.approx(float(c[f"{name}_loss"]), rel=1e-11, abs=1e-13)
            assert np.allclose(r["grad_w"], c[f"{name}_gw"], rtol=1e-10, atol=1e-13)
            assert np.allclose(r["grad_b"], c[f"{name}_gb"], rtol=1e-10, atol=1e-13)
            misc = c[f"{name}_misc"]
            assert r["n_tokens"] == int(misc[0]) and r["excluded"] == int(misc[3])
            assert r["clip_fraction"] == pytest.approx(misc[1], abs=1e-12)


# ------------------------------------------------------------------ numpy pairwise sum
@pytest.mark.parametrize("n", [1, 7, 8, 9, 127, 128, 129, 257, 1000, 8193, 70843])
def test_pairwise_sum_is_numpy_sum(n):
    rng = np.random.default_rng(n)
    x = rng.normal(size=n) * 10 ** rng.uniform(-3, 3, size=n)
    assert O.numpy_pairwise_sum(x) == float(np.sum(x))


# ------------------------------------------------------------------ reference hand cases
def _single(lp_theta_logits, behav, prox, adv, eps=0.2, decoupled=True):
    return O.surrogate_terms(lp_theta_logits, [0], [behav], [prox], [adv], eps, decoupled)


def test_hand_case_positive_advantage():
    # test_trainer.py:115-127: r = 0.8, u = 1.25, A = +1 -> -0.96
    x = np.zeros((1, 16))
    lp = math.log(1 / 16)
    prox = lp - math.log(1.25)
    t = _single(x, prox - math.log(0.8), prox, 1.0)
    s = t["stats"]
    assert -s[0] / max(s[1], 1) == pytest.approx(-0.96, abs=1e-12)
    assert s[2] / s[1] == 1.0


def test_hand_case_negative_advantage():
    # test_trainer.py:130-138: A = -1 -> +1.0, clip_fraction 0
    x = np.zeros((1, 16))
    lp = math.log(1 / 16)
    prox = lp - math.log(1.25)
    s = _single(x, prox - math.log(0.8), prox, -1.0)["stats"]
    assert -s[0] / s[1] == pytest.approx(1.0, abs=1e-12)
    assert s[2] == 0


def test_naive_hand_cases():
    # test_trainer.py:141-153
    x = np.zeros((1, 16))
    lp = math.log(1 / 16)
    s = _single(x, lp - math.log(1.5), lp, 1.0, decoupled=False)["stats"]
    assert -s[0] / s[1] == pytest.approx(-1.2, abs=1e-12)
    for a in (2.5, -0.7):
        s = _single(x, lp, lp, a, decoupled=False)["stats"]
        assert -s[0] / s[1] == pytest.approx(-a, abs=1e-12)


def test_clip_grid():
    # test_trainer.py:170-185
    x = np.zeros((1, 16))
    lp = math.log(1 / 16)
    eps = 0.2
    for r in (0.5, 0.8, 1.0, 1.25, 2.0):
        for u in (0.5, 0.79, 1.0, 1.21, 1.5):
            for a in (-2.0, -1.0, 0.5, 1.0, 2.0):
                prox = lp - math.log(u)
                s = _single(x, prox - math.log(r), prox, a, eps)["stats"]
                direct = r * min(u * a, min(max(u, 1 - eps), 1 + eps) * a)
                assert -s[0] / s[1] == pytest.approx(-direct, rel=1e-12)


def test_non_finite_behaviour_excluded():
    # test_trainer.py:212-219
    t = _single(np.zeros((1, 16)), -np.inf, math.log(1 / 16), 1.0)
    assert t["stats"][4] == 1 and np.all(np.isfinite(t["dlogits"]))


def test_reduction_identity_on_policy():
    # test_trainer.py:156-167 / acceptance criterion 1: prox == behav -> decoupled == naive
    rng = np.random.default_rng(5)
    for _ in range(10):
        x = rng.normal(0, 2, size=(30, 50))
        tok = rng.integers(0, 50, size=30)
        lp = O.token_logprobs(x, tok)
        adv = rng.normal(size=30)
        d = O.surrogate_terms(x, tok, lp, lp, adv, 0.2, True)
        n = O.surrogate_terms(x, tok, lp, lp, adv, 0.2, False)
        assert abs(d["stats"][0] - n["stats"][0]) <= 1e-12
        assert np.max(np.abs(d["dlogits"] - n["dlogits"])) <= 1e-12


def test_log_softmax_hand_cases():
    # test_policy.py:12-18, 48-53, 56-63
    assert np.allclose(O.log_softmax(np.zeros(16)), math.log(1 / 16), atol=1e-15)
    lp = O.log_softmax(np.array([0.0, math.log(3.0)]))
    assert lp[1] == pytest.approx(math.log(0.75), abs=1e-15)
    assert lp[0] == pytest.approx(math.log(0.25), abs=1e-15)
    rng = np.random.default_rng(3)
    for _ in range(100):
        x = rng.normal(0, rng.uniform(0.1, 3.0), size=16)
        assert abs(np.exp(O.log_softmax(x)).sum() - 1) <= 1e-12


def test_dlogits_is_autograd_of_loss():
    # self-consistency of the fused backward: finite differences on the logits
    rng = np.random.default_rng(11)
    x = rng.normal(0, 1.5, size=(6, 9))
    tok = rng.integers(0, 9, size=6)
    prox = O.token_logprobs(x, tok) + rng.normal(0, 0.1, size=6)
    behav = prox + rng.normal(0, 0.2, size=6)
    adv = rng.normal(size=6)

    def loss(z):
        return -O.surrogate_terms(z, tok, behav, prox, adv, 0.2, True, want_dlogits=False)["stats"][0]

    d = O.surrogate_terms(x, tok, behav, prox, adv, 0.2, True)["dlogits"]
    h = 1e-6
    for _ in range(20):
        dx = rng.normal(size=x.shape)
        num = (loss(x + h * dx) - loss(x - h * dx)) / (2 * h)
        assert abs(num - float(np.sum(d * dx))) <= 1e-6 * max(1.0, abs(num))


# ------------------------------------------------------------------ allocator KATs
def test_allocator_hand_traces():
    # test_trainer.py:222-245; SURVEY §8c probe KATs
    lengths = [7, 5, 4, 3, 1]
    assert [[lengths[i] for i in g] for g in O.allocate_microbatches(lengths, 10, 1)] == \
        [[7, 3], [5, 4, 1]]
    assert O.allocate_microbatches([10], 10, 1) == ((0,),)
    assert O.allocate_microbatches([5, 5, 5], 10, 1) == ((0, 1), (2,))
    assert O.allocate_microbatches([3, 5, 3, 5], 8, 2) == ((1, 0), (3, 2))
    assert O.allocate_microbatches([2, 2], 10, 5) == ((0,), (1,))
    assert O.allocate_microbatches([6, 4, 4, 2, 2, 2], 10, 1) == ((0, 1), (2, 3, 4, 5))
    for bad in (([11], 10, 1), ([0, 3], 10, 1), ([3], 10, 0)):
        with pytest.raises(O.OracleBatchError):
            O.allocate_microbatches(*bad)


def test_minibatch_split_semantics():
    assert [len(s) for s in O.minibatch_splits(10, 4)] == [3, 3, 2, 2]
    assert [len(s) for s in O.minibatch_splits(3, 4)] == [1, 1, 1]


# ------------------------------------------------------------------ extensions reduce to reference
def test_gae_reduces_to_reference_raw():
    rng = np.random.default_rng(1)
    lengths = rng.integers(0, 40, size=12)
    bounds = np.concatenate([[0], np.cumsum(lengths)])
    rewards = rng.choice([5.0, -5.0], size=12)
    raw = O.gae_raw(rewards, bounds, 1.0, 1.0)
    ref = np.repeat(rewards, lengths)
    assert np.array_equal(raw, ref)
    assert np.array_equal(O.advantages(rewards, bounds, mode="gae"),
                          O.compute_advantages_ref(rewards, bounds))


def test_gae_recurrence():
    bounds = np.array([0, 3])
    v = np.array([0.5, -0.2, 0.1])
    a = O.gae_raw([2.0], bounds, 0.9, 0.8, values=v)
    d2 = 2.0 + 0 - 0.1
    d1 = 0 + 0.9 * 0.1 + 0.2
    d0 = 0 + 0.9 * -0.2 - 0.5
    assert np.allclose(a, [d0 + 0.72 * (d1 + 0.72 * d2), d1 + 0.72 * d2, d2])


def test_group_norm_one_group_is_global():
    rng = np.random.default_rng(2)
    lengths = rng.integers(1, 30, size=10)
    bounds = np.concatenate([[0], np.cumsum(lengths)])
    raw = np.repeat(rng.normal(size=10), lengths)
    assert np.array_equal(O.normalize_group(raw, bounds, np.zeros(10)), O.normalize_global(raw))


def test_stale_mask_disabled_is_reference():
    rng = np.random.default_rng(4)
    x = rng.normal(size=(20, 30))
    tok = rng.integers(0, 30, size=20)
    lp = O.token_logprobs(x, tok)
    behav = lp + rng.normal(0, 0.3, size=20)
    adv = rng.normal(size=20)
    ver = rng.integers(0, 9, size=20)
    a = O.surrogate_terms(x, tok, behav, lp, adv)
    b = O.surrogate_terms(x, tok, behav, lp, adv, versions=ver, current_version=8, eta_mask=-1)
    assert np.array_equal(a["stats"], b["stats"]) and np.array_equal(a["dlogits"], b["dlogits"])
    c = O.surrogate_terms(x, tok, behav, lp, adv, versions=ver, current_version=8, eta_mask=4)
    stale = (8 - ver) > 4
    assert c["stats"][5] == stale.sum()
    assert np.all(c["dlogits"][stale] == 0)


def test_adam_oracle_bit_exact_vs_reference_golden():
    """oracle._adam (policy.py:225-258 restated) reproduces the reference's
    apply_update after grad.scale_(-1/n) bit for bit over 3 chained steps."""
    for c in load_cases("adam.npz"):
        cfg = O.AdamCfg(lr=float(c["lr"]), clip_norm=float(c["clip"]), weight_decay=float(c["wd"]))
        W, b = c["W0"], c["b0"]
        m_w, v_w = np.zeros_like(W), np.zeros_like(W)
        m_b, v_b = np.zeros_like(b), np.zeros_like(b)
        step = 0
        for k in range(int(c["steps"])):
            s = -1.0 / int(c[f"n{k}"])
            gw, gb = c[f"gw{k}"] * s, c[f"gb{k}"] * s
            assert math.sqrt(float(np.sum(gw ** 2) + np.sum(gb ** 2))) == float(c[f"norm{k}"])
            W, b, m_w, v_w, m_b, v_b, step = O.adam_update(W, b, gw, gb, m_w, v_w, m_b, v_b, step, cfg)
            assert step == int(c[f"step{k}"])
        for got, key in ((W, "W"), (b, "b"), (m_w, "mw"), (v_w, "vw"), (m_b, "mb"), (v_b, "vb")):
            assert np.array_equal(got, c[key]), key


def test_pairwise_cut_depth_nodes_split_at_most_once():
    """K3's fused kernel (advantages.cu) cuts numpy's pairwise tree at the depth where the
    smallest node is <= 128 and relies on every node there being <= 143, i.e. split by numpy
    at most once more into two <= 128 leaves.  Checked over small n exhaustively and over
    large n around every power-of-two boundary."""
    def split(n):
        n2 = n // 2
        return n2 - n2 % 8, n - (n2 - n2 % 8)

    def depth(n, cap=20):
        d = 0
        while d < cap and n > 128:
            n, d = split(n)[0], d + 1
        return d

    def extremes(n, d):  # (smallest, largest) node at depth d: leftmost / rightmost paths
        lo = hi = n
        for _ in range(d):
            lo, hi = split(lo)[0], split(hi)[1]
        return lo, hi

    rng = np.random.default_rng(0)
    cases = list(range(1, 20000)) + [int(x) for x in rng.integers(1, 128 << 20, 3000)] + \
        [(128 << k) + j for k in range(21) for j in range(-40, 41)]
    for n in cases:
        if n < 1 or n > (128 << 20):
            continue
        d = depth(n)
        lo, hi = extremes(n, d)
        assert lo <= 128 and hi <= 143, (n, d, lo, hi)
        if d > 0:
            assert extremes(n, d - 1)[0] > 128  # every node above the cut splits
        if hi > 128:
            assert max(split(hi)) <= 128
