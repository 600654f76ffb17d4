"""Generate golden vectors by running the REAL reference (asyncrl) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes small ``.npz`` fixtures next to this file.  The GPU box has no
/root/reference, so these committed fixtures are how the CUDA path and the CPU
oracle are pinned to the reference there.  Nothing here is imported by the
product package.

Fixtures
--------
surrogate.npz   logits-level `_surrogate_terms` (trainer.py:150-195) via the
                identity-feature trick: features = I_T and W = logits.T, b = 0
                make the reference's logits equal the chosen logits and its
                grad_w_sum equal resid.T, i.e. the per-logit backward.
advantages.npz  `compute_advantages` (trainer.py:114-125) on random rewards /
                lengths, including zero-length trajectories and the constant-0.1
                quirk (np.std of a constant that is not exactly representable).
allocator.npz   `allocate_microbatches` (trainer.py:235-270) on the reference's
                property-test distributions, hand cases and large Pareto cases.
adam.npz        `grad.scale_(-1/n)` + `apply_update` (trainer.py:329-331,
                policy.py:215-258) over 3 consecutive steps: clipped and
                unclipped gradients, shapes from 1x1 to 64x300.
trainstep.npz   `train_step` / `decoupled_ppo_loss` / `naive_ppo_loss` on real
                rollout batches from the reference's RolloutWorker
                (test_trainer.py:14-26 recipe).
"""
from __future__ import annotations

import os
import sys
from types import SimpleNamespace

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from asyncrl import policy as P  # noqa: E402
from asyncrl import trainer as T  # noqa: E402
from asyncrl.rollout import GenerateRequest, RolloutWorker  # noqa: E402
from asyncrl.tasks import SEP_TOKEN, Prompt, RewardResult  # noqa: E402
from asyncrl.timeline import LengthDistribution  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def _fake_traj(reward):
    return SimpleNamespace(reward=SimpleNamespace(reward=float(reward)))


# ---------------------------------------------------------------- surrogate
def make_surrogate(rng):
    cases = []
    specs = [
        # (T, V, decoupled, eps, logit_scale, prox_noise, behav_noise)
        (1, 16, True, 0.2, 0.0, 0.0, 0.0),
        (7, 16, True, 0.2, 1.0, 0.05, 0.1),
        (50, 37, True, 0.2, 2.0, 0.02, 0.1),
        (50, 37, False, 0.2, 2.0, 0.02, 0.1),
        (64, 64, True, 0.1, 3.0, 0.3, 0.5),
        (64, 64, False, 0.3, 3.0, 0.3, 0.5),
        (33, 128, True, 0.2, 8.0, 0.5, 1.0),
        (40, 16, True, 0.2, 2.0, 0.0, 0.0),   # on-policy: prox == behav
    ]
    for (n, v, dec, eps, sc, pn, bn) in specs:
        logits = rng.normal(0.0, sc, size=(n, v)) if sc > 0 else np.zeros((n, v))
        if n >= 33:
            logits[3, :] += 40.0  # large common offset (exercise the max shift)
            logits[5, 7] = -1e4   # very negative logit
        tokens = rng.integers(0, v, size=n)
        lp_true = T.P.log_softmax(logits)[np.arange(n), tokens]
        prox = lp_true + rng.normal(0.0, pn, size=n)
        behav = prox + rng.normal(0.0, bn, size=n)
        adv = rng.normal(0.0, 1.0, size=n)
        if n >= 33:
            behav[1] = -np.inf            # invalid scale -> excluded (test_trainer.py:212-219)
            prox[2] = behav[2] + 800.0    # exp overflows -> inf scale -> excluded
            adv[4] = 0.0
        params = P.VersionedParams(0, np.ascontiguousarray(logits.T), np.zeros(v))
        batch = T.TrainBatch(trajectories=[], step_index=0, features=np.eye(n),
                             tokens=tokens.astype(np.int64), behavior_logprobs=behav,
                             traj_bounds=np.array([0, n]), prox_logprobs=prox,
                             advantages=adv)
        lp_ref = P.batch_token_log_probs(params, np.eye(n), tokens)
        with np.errstate(over="ignore", invalid="ignore"):
            t = T._surrogate_terms(batch, np.arange(n), params, eps, dec)
        resid = t["grad_w_sum"].T  # (n, v): coef * (onehot - softmax)
        assert np.allclose(t["grad_b_sum"], resid.sum(axis=0), atol=1e-12)
        loss = (T.decoupled_ppo_loss if dec else T.naive_ppo_loss)
        with np.errstate(over="ignore", invalid="ignore"):
            lr = loss(batch, params, clip_eps=eps)
        cases.append(dict(logits=logits, tokens=tokens, behav=behav, prox=prox, adv=adv,
                          decoupled=np.array(dec), eps=np.array(eps), lp=lp_ref,
                          objective_sum=np.array(t["objective_sum"]),
                          n_valid=np.array(t["n_valid"]), n_clipped=np.array(t["n_clipped"]),
                          ratio_sum=np.array(t["ratio_sum"]),
                          n_excluded=np.array(t["n_excluded"]), resid=resid,
                          loss=np.array(lr.loss), clip_fraction=np.array(lr.clip_fraction),
                          mean_ratio=np.array(lr.mean_ratio)))
    flat = {f"c{i}_{k}": v for i, c in enumerate(cases) for k, v in c.items()}
    flat["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(OUT, "surrogate.npz"), **flat)


# ---------------------------------------------------------------- advantages
def make_advantages(rng):
    cases = []

    def add(rewards, lengths):
        bounds = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
        batch = SimpleNamespace(trajectories=[_fake_traj(r) for r in rewards],
                                traj_bounds=bounds, n_tokens=int(bounds[-1]),
                                advantages=None)
        batch.token_range = lambda k, b=bounds: np.arange(b[k], b[k + 1])
        adv = T.compute_advantages(batch)
        cases.append((np.asarray(rewards, dtype=np.float64), bounds, adv))

    add([5.0, -5.0], [6, 6])                       # test_trainer.py:49-61
    add([5.0, 5.0, -5.0, -5.0], [2, 2, 2, 2])      # test_trainer.py:64-78
    add([5.0, 5.0, 5.0], [3, 5, 2])                # test_trainer.py:81-85 (zeros)
    add([0.1] * 7, [3, 1, 4, 1, 5, 9, 2])          # constant 0.1 quirk
    add([5.0, -5.0, 5.0], [0, 4, 3])               # zero-length trajectory
    for _ in range(12):
        n = int(rng.integers(1, 80))
        lengths = rng.integers(0, 300, size=n)
        lengths[0] = max(lengths[0], 1)
        kind = rng.integers(0, 3)
        if kind == 0:
            rewards = rng.choice([5.0, -5.0], size=n)
        elif kind == 1:
            rewards = rng.normal(0, 3, size=n)
        else:
            rewards = rng.choice([0.1, 0.7, -0.3], size=n)
        add(rewards, lengths)
    # larger (> 8192 tokens: crosses several pairwise levels)
    add(rng.choice([5.0, -5.0], size=64), rng.integers(128, 2049, size=64))
    add(rng.normal(size=200), rng.integers(1, 400, size=200))
    flat = {}
    for i, (r, b, a) in enumerate(cases):
        flat[f"c{i}_rewards"] = r
        flat[f"c{i}_bounds"] = b
        flat[f"c{i}_adv"] = a
    flat["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(OUT, "advantages.npz"), **flat)


# ---------------------------------------------------------------- allocator
def make_allocator(rng):
    cases = []

    def add(lengths, cap, kmin):
        plan = T.allocate_microbatches(list(map(int, lengths)), int(cap), int(kmin))
        n = len(lengths)
        gid = np.full(n, -1, dtype=np.int32)
        slot = np.full(n, -1, dtype=np.int32)
        for g, members in enumerate(plan.groups):
            for s, i in enumerate(members):
                gid[i], slot[i] = g, s
        cases.append((np.asarray(lengths, dtype=np.int64), cap, kmin, gid, slot))

    add([7, 5, 4, 3, 1], 10, 1)          # test_trainer.py:222-226
    add([2, 2], 10, 2)                   # 229-231
    add([10], 10, 1)                     # 234-236
    add([5, 5, 5], 10, 1)
    add([3, 5, 3, 5], 8, 2)
    add([2, 2], 10, 5)
    add([6, 4, 4, 2, 2, 2], 10, 1)
    add([9, 9, 5, 5, 5, 2, 2, 1], 16, 2)  # 263-267
    for _ in range(300):                 # test_trainer.py:248-260 distribution
        n = int(rng.integers(1, 40))
        cap = int(rng.integers(8, 64))
        add([int(rng.integers(1, cap + 1)) for _ in range(n)], cap, int(rng.integers(1, 5)))
    for _ in range(200):                 # test_acceptance.py:224-234 distribution
        n = int(rng.integers(1, 50))
        cap = int(rng.integers(4, 80))
        add([int(rng.integers(1, cap + 1)) for _ in range(n)], cap,
            int(rng.integers(1, min(n, 4) + 1)))
    dist = LengthDistribution(kind="pareto", alpha=1.2, scale=64.0, cap=32768)
    for n, kmin in ((1024, 1), (4096, 1), (1024, 8)):
        lengths = [max(64, dist.sample(rng)) for _ in range(n)]
        add(lengths, 32768, kmin)
    lengths = rng.integers(128, 8193, size=128)   # cfg2 minibatch
    add(lengths, 32768, 1)
    flat = {}
    for i, (l, c, k, g, s) in enumerate(cases):
        flat[f"c{i}_lengths"] = l
        flat[f"c{i}_cap"] = np.array(c)
        flat[f"c{i}_kmin"] = np.array(k)
        flat[f"c{i}_gid"] = g
        flat[f"c{i}_slot"] = s
    flat["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(OUT, "allocator.npz"), **flat)


# ---------------------------------------------------------------- train step
def _copy_prompt(payload, prompt_id=0):
    return Prompt(id=prompt_id, tokens=tuple(payload) + (SEP_TOKEN,), task_kind="copy",
                  target=tuple(payload))


def _random_params(featurizer, rng, scale=0.5, version=0):
    v = featurizer.config.vocab_size
    return P.VersionedParams(version=version,
                             weights=rng.normal(0, scale, size=(v, featurizer.feature_dim)),
                             bias=rng.normal(0, scale, size=v))


def _rollout_batch(featurizer, params, n_traj, seed, rewards=None, max_new=6):
    worker = RolloutWorker(params, featurizer, seed=seed)
    trajs = []
    for k in range(n_traj):
        traj = worker.generate(GenerateRequest(
            prompt=_copy_prompt([k % 10, (k + 3) % 10], prompt_id=k),
            max_new_tokens=max_new, trajectory_id=k))
        r = rewards[k] if rewards is not None else (5.0 if k % 2 == 0 else -5.0)
        traj.reward = RewardResult(k, r, r > 0)
        trajs.append(traj)
    return T.build_train_batch(trajs, featurizer, 0)


def make_trainstep(rng):
    featurizer = P.ContextFeaturizer(P.PolicyConfig())
    flat = {}
    cfgs = [
        dict(),
        dict(minibatches=1),
        dict(objective="naive"),
        dict(micro_token_budget=8, micro_min_groups=2),
        dict(minibatches=3, micro_token_budget=12, clip_eps=0.1),
    ]
    i = 0
    for seed in (8, 10, 21):
        for cfg_kw in cfgs:
            behavior = _random_params(featurizer, rng, scale=0.5)
            batch = _rollout_batch(featurizer, behavior, n_traj=8, seed=seed,
                                   rewards=[float(rng.choice([5.0, -5.0])) for _ in range(8)])
            # stale arrival: the trainer's params differ from the behaviour params
            current = P.VersionedParams(
                3, behavior.weights + 0.2 * rng.normal(size=behavior.weights.shape),
                behavior.bias + 0.1 * rng.normal(size=behavior.bias.shape))
            cfg = T.TrainerConfig(**cfg_kw)
            opt = P.AdamState.zeros_like(current)
            snap = dict(features=batch.features.copy(), tokens=batch.tokens.copy(),
                        behav=batch.behavior_logprobs.copy(),
                        bounds=batch.traj_bounds.copy(),
                        rewards=np.array([t.reward.reward for t in batch.trajectories]),
                        W=current.weights.copy(), b=current.bias.copy())
            new_params, stats = T.train_step(batch, current, opt, cfg)
            out = dict(snap)
            out.update(prox=batch.prox_logprobs, adv=batch.advantages,
                       W_new=new_params.weights, b_new=new_params.bias,
                       version_new=np.array(new_params.version),
                       m_w=opt.m_weights, v_w=opt.v_weights, m_b=opt.m_bias, v_b=opt.v_bias,
                       opt_step=np.array(opt.step),
                       stats=np.array([stats.loss, stats.clip_fraction, stats.mean_ratio,
                                       stats.tokens, stats.minibatch_updates,
                                       stats.microbatches, stats.excluded_tokens]),
                       clip_eps=np.array(cfg.clip_eps), minibatches=np.array(cfg.minibatches),
                       budget=np.array(cfg.micro_token_budget),
                       kmin=np.array(cfg.micro_min_groups),
                       decoupled=np.array(cfg.objective == "decoupled"))
            # whole-batch losses under the (pre-step) current params
            b2 = T.build_train_batch(batch.trajectories, featurizer, 0)
            T.recompute_prox_logprobs(b2, behavior)   # prox from behaviour params (stale)
            T.compute_advantages(b2)
            for name, fn in (("dec", T.decoupled_ppo_loss), ("nai", T.naive_ppo_loss)):
                lr = fn(b2, current, clip_eps=cfg.clip_eps)
                out[f"{name}_prox"] = b2.prox_logprobs
                out[f"{name}_loss"] = np.array(lr.loss)
                out[f"{name}_gw"] = lr.grad.weights
                out[f"{name}_gb"] = lr.grad.bias
                out[f"{name}_misc"] = np.array([lr.n_tokens, lr.clip_fraction, lr.mean_ratio,
                                                lr.excluded])
            for k, v in out.items():
                flat[f"c{i}_{k}"] = np.asarray(v)
            i += 1
    flat["n_cases"] = np.array(i)
    np.savez_compressed(os.path.join(OUT, "trainstep.npz"), **flat)


# ---------------------------------------------------------------- adam
def make_adam():
    rng = np.random.default_rng(7)
    cases = []
    specs = [  # (V, F, grad magnitude per step, lr, clip_norm, weight_decay)
        (1, 1, (0.3, 50.0, 1e-3), 2e-2, 1.0, 0.05),
        (16, 12, (1e-2, 1e-2, 3.0), 2e-2, 1.0, 0.05),
        (37, 185, (5.0, 1e-4, 0.2), 2e-2, 1.0, 0.05),
        (64, 300, (1e-3, 40.0, 1.0), 1e-3, 1.0, 0.05),
        (64, 33, (2.0, 2.0, 2.0), 2e-2, 0.0, 0.0),  # clipping disabled
    ]
    for V, F, mags, lr, clip, wd in specs:
        cfg = P.AdamConfig(lr=lr, clip_norm=clip, weight_decay=wd)
        params = P.VersionedParams(0, rng.normal(0, 0.5, size=(V, F)), rng.normal(0, 0.5, size=V))
        opt = P.AdamState.zeros_like(params)
        case = dict(W0=np.array(params.weights), b0=np.array(params.bias), lr=np.array(lr),
                    clip=np.array(clip), wd=np.array(wd), steps=np.array(len(mags)))
        for k, mag in enumerate(mags):
            gw = rng.normal(0, mag, size=(V, F))
            gb = rng.normal(0, mag, size=V)
            n = int(rng.integers(1, 5000))
            grad = P.ParamGrad(gw.copy(), gb.copy())
            grad.scale_(-1.0 / n)                                    # trainer.py:330
            norm = grad.global_norm()
            params = P.apply_update(params, grad, opt, cfg)          # trainer.py:331
            case.update({f"gw{k}": gw, f"gb{k}": gb, f"n{k}": np.array(n),
                         f"norm{k}": np.array(norm), f"step{k}": np.array(opt.step)})
        case.update(W=np.array(params.weights), b=np.array(params.bias), mw=opt.m_weights.copy(),
                    vw=opt.v_weights.copy(), mb=opt.m_bias.copy(), vb=opt.v_bias.copy())
        cases.append(case)
    flat = {f"c{i}_{k}": v for i, c in enumerate(cases) for k, v in c.items()}
    flat["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(OUT, "adam.npz"), **flat)


if __name__ == "__main__":
    only = set(sys.argv[1:])
    rng = np.random.default_rng(20250530)
    if not only:
        make_surrogate(rng)
        make_advantages(rng)
        make_allocator(rng)
        make_trainstep(rng)
    if not only or "adam" in only:
        make_adam()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
