"""float64 numpy restatement of the AReaL (asyncrl) training hot path.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Never shipped, never
on the product path.  All references are to ``/root/reference/pkg/src/asyncrl``.

The reference computes logits from a linear policy inside the loss
(trainer.py:163).  The B200 path receives the logits from the model, so the
oracle here is restated *given logits* ``x[T, V]``; the linear-policy wrapper
at the bottom (``linear_*``) re-adds ``feats @ W.T + b`` for drop-in parity with
the reference's own train_step.

Extensions named by the north star but absent from the reference (entropy,
GAE with gamma*lambda < 1 / values, GRPO group normalisation, the version
staleness mask and the behaviour-weight cap) are defined here; each reduces to
reference behaviour at its default (checked in tests/test_oracle_golden.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "OracleBatchError", "log_softmax", "token_logprobs", "token_entropy",
    "surrogate_terms", "STAT_NAMES", "compute_advantages_ref", "numpy_pairwise_sum",
    "gae_raw", "normalize_global", "normalize_group", "advantages",
    "allocate_microbatches", "minibatch_splits", "train_step_plan",
    "AdamCfg", "adam_update", "linear_logits", "linear_train_step", "linear_loss",
]


class OracleBatchError(ValueError):
    """Mirrors ``trainer.BatchError`` (trainer.py:34-35)."""


# ---------------------------------------------------------------------------
# log-softmax / gather / entropy  (policy.py:145-147, 159-163)
# ---------------------------------------------------------------------------

def log_softmax(x: np.ndarray) -> np.ndarray:
    """Max-shifted log-softmax over the last axis (policy.py:145-147)."""
    x = np.asarray(x, dtype=np.float64)
    m = np.max(x, axis=-1, keepdims=True)
    z = x - m
    return z - np.log(np.sum(np.exp(z), axis=-1, keepdims=True))


def token_logprobs(logits: np.ndarray, tokens: np.ndarray) -> np.ndarray:
    """lp[t] = log_softmax(x_t)[a_t]  (policy.py:159-163 with logits given)."""
    all_lp = log_softmax(logits)
    return all_lp[np.arange(len(tokens)), np.asarray(tokens, dtype=np.int64)]


def token_entropy(logits: np.ndarray) -> np.ndarray:
    """Extension: H_t = -sum_v p log p (0 log 0 := 0).  Not in the reference."""
    all_lp = log_softmax(logits)
    p = np.exp(all_lp)
    terms = np.where(p > 0, p * all_lp, 0.0)
    return -terms.sum(axis=-1)


# ---------------------------------------------------------------------------
# decoupled / naive PPO surrogate, fused backward  (trainer.py:150-195)
# ---------------------------------------------------------------------------

STAT_NAMES = ("objective_sum", "n_valid", "n_clipped", "ratio_sum",
              "n_excluded", "n_masked", "entropy_sum", "n_tokens")


def surrogate_terms(logits, tokens, behav, prox, adv, clip_eps=0.2, decoupled=True,
                    versions=None, current_version=0, eta_mask=-1,
                    behav_weight_cap=0.0, grad_scale=1.0, want_dlogits=True):
    """Per-token surrogate over given logits; returns stats + per-token outputs.

    Follows trainer.py:163-195 term by term:
      all_lp = log_softmax(x) (163); lp = gather (164);
      decoupled: scale = exp(prox - behav), ratio = exp(lp - prox) (165-167);
      naive: scale = 1, ratio = exp(lp - behav) (168-170);
      valid = isfinite(scale) & isfinite(ratio) (172);
      P = ratio*A, Cl = clip(ratio, 1-eps, 1+eps)*A (173-174);
      obj = where(valid, scale*min(P, Cl), 0) (175-176);
      take = (P <= Cl) & valid (177); coef = where(take, scale*A*ratio, 0) (179);
      resid = coef * (onehot - softmax) (180-182)  ==  d obj / d logits;
      counters (186-195).
    The returned ``dlogits`` is the gradient of the *loss* (the negated
    objective) scaled by ``grad_scale``: ``grad_scale*coef*(p - onehot)``, i.e.
    ``-grad_scale*resid``.  With grad_scale = 1/n this is d(loss)/d(logits) of
    _ppo_loss (trainer.py:204-207).

    Extensions (defaults reproduce the reference exactly):
      * eta_mask >= 0: tokens with current_version - versions[t] > eta_mask are
        masked (excluded, counted in n_masked and n_excluded);
      * behav_weight_cap > 0: valid tokens with scale > cap are masked likewise;
      * entropy_sum accumulates H_t over valid (unmasked) tokens.
    """
    x = np.asarray(logits, dtype=np.float64)
    toks = np.asarray(tokens, dtype=np.int64)
    behav = np.asarray(behav, dtype=np.float64)
    if prox is None:
        # first minibatch of a step: prox was computed under the same params as the
        # current forward (trainer.py:295 vs 315-321), i.e. prox == lp exactly
        prox = log_softmax(x)[np.arange(len(toks)), toks]
    prox = np.asarray(prox, dtype=np.float64)
    adv = np.asarray(adv, dtype=np.float64)
    n = len(toks)
    all_lp = log_softmax(x)
    rows = np.arange(n)
    lp = all_lp[rows, toks]
    p = np.exp(all_lp)
    ent = -np.where(p > 0, p * all_lp, 0.0).sum(axis=-1)
    with np.errstate(over="ignore", invalid="ignore"):
        if decoupled:
            scale = np.exp(prox - behav)
            ratio = np.exp(lp - prox)
        else:
            scale = np.ones_like(lp)
            ratio = np.exp(lp - behav)
        valid = np.isfinite(scale) & np.isfinite(ratio)
        masked = np.zeros(n, dtype=bool)
        if eta_mask is not None and eta_mask >= 0 and versions is not None:
            masked |= (current_version - np.asarray(versions, dtype=np.int64)) > eta_mask
        if behav_weight_cap and behav_weight_cap > 0:
            masked |= valid & (scale > behav_weight_cap)
        valid_eff = valid & ~masked
        term_plain = ratio * adv
        term_clip = np.clip(ratio, 1 - clip_eps, 1 + clip_eps) * adv
        obj = np.where(valid_eff, scale * np.minimum(term_plain, term_clip), 0.0)
        take = (term_plain <= term_clip) & valid_eff
        coef = np.where(take, scale * adv * ratio, 0.0)
        clipped = valid_eff & (term_clip < term_plain)
    stats = np.array([
        obj.sum(),
        np.count_nonzero(valid_eff),
        np.count_nonzero(clipped),
        np.where(valid_eff, ratio, 0.0).sum(),
        n - np.count_nonzero(valid_eff),
        np.count_nonzero(masked),
        np.where(valid_eff, ent, 0.0).sum(),
        n,
    ], dtype=np.float64)
    out = {"stats": stats, "lp": lp, "entropy": ent, "coef": coef, "valid": valid_eff,
           "clipped": clipped, "masked": masked, "take": take, "obj": obj,
           "ratio": ratio, "scale": scale}
    if want_dlogits:
        d = p.copy()
        d[rows, toks] -= 1.0
        out["dlogits"] = (grad_scale * coef)[:, None] * d
    return out


# ---------------------------------------------------------------------------
# advantages  (trainer.py:114-125) + GAE / GRPO extensions
# ---------------------------------------------------------------------------

def compute_advantages_ref(rewards, traj_bounds) -> np.ndarray:
    """Reference advantages, same numpy calls as trainer.py:116-124.

    raw_t = reward of the trajectory owning t; np.std population std; zero
    std -> zeros; else (raw - mean) / std.
    """
    bounds = np.asarray(traj_bounds, dtype=np.int64)
    raw = np.empty(int(bounds[-1]))
    for k, r in enumerate(rewards):
        raw[bounds[k]:bounds[k + 1]] = r
    return normalize_global(raw)


def numpy_pairwise_sum(a) -> float:
    """numpy's float64 add.reduce order (blocks of 8 accumulators, split at n/2
    rounded down to a multiple of 8, leaves <= 128).  Verified bit-exact
    against np.sum in tests/test_oracle_golden.py; the CUDA advantage kernel
    replays this tree so the reference's np.mean/np.std are reproduced bit for
    bit."""
    a = np.asarray(a, dtype=np.float64)

    def rec(lo, n):
        if n < 8:
            res = 0.0
            for i in range(n):
                res += float(a[lo + i])
            return res
        if n <= 128:
            r = [float(a[lo + j]) for j in range(8)]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] += float(a[lo + i + j])
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += float(a[lo + i])
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return rec(lo, n2) + rec(lo + n2, n - n2)

    return rec(0, len(a))


def normalize_global(raw) -> np.ndarray:
    """Token-weighted global normalisation exactly as trainer.py:119-123."""
    raw = np.asarray(raw, dtype=np.float64)
    if raw.size == 0:
        return raw.copy()
    std = float(np.std(raw))
    if std == 0.0:
        return np.zeros_like(raw)
    return (raw - np.mean(raw)) / std


def gae_raw(rewards, traj_bounds, gamma=1.0, lam=1.0, values=None,
            token_rewards=None) -> np.ndarray:
    """Extension: per-sequence GAE reverse scan (not in the reference).

    r_t = reward on the final token of each trajectory (the reference's
    terminal reward, trainer.py:19-22) unless ``token_rewards`` is given;
    V_t = values (0 if None), V past the end = 0;
    delta_t = r_t + gamma*V_{t+1} - V_t;  A_t = delta_t + gamma*lam*A_{t+1}.
    gamma = lam = 1 with no values gives A_t = R_k: the reference's raw.
    """
    bounds = np.asarray(traj_bounds, dtype=np.int64)
    T = int(bounds[-1])
    out = np.zeros(T)
    vals = np.zeros(T) if values is None else np.asarray(values, dtype=np.float64)
    for k in range(len(bounds) - 1):
        s, e = int(bounds[k]), int(bounds[k + 1])
        acc = 0.0
        for t in range(e - 1, s - 1, -1):
            if token_rewards is not None:
                r = float(token_rewards[t])
            else:
                r = float(rewards[k]) if t == e - 1 else 0.0
            v_next = float(vals[t + 1]) if t + 1 < e else 0.0
            delta = r + gamma * v_next - float(vals[t])
            acc = delta + gamma * lam * acc
            out[t] = acc
    return out


def normalize_group(raw, traj_bounds, group_ids, eps=0.0, weighting="token") -> np.ndarray:
    """Extension: GRPO-style per-group normalisation (not in the reference).

    Group = trajectories sharing ``group_ids[k]`` (the reference's prompt id,
    tasks.py:80).  ``weighting='token'``: mean / population std over the
    group's tokens (one group == reference global normalisation).
    ``weighting='sequence'``: over the group's trajectories, one value each
    (raw must be constant per trajectory, e.g. reward broadcast).
    adv = (raw - mean) / (std + eps); std + eps == 0 -> 0.
    """
    raw = np.asarray(raw, dtype=np.float64)
    bounds = np.asarray(traj_bounds, dtype=np.int64)
    gids = np.asarray(group_ids, dtype=np.int64)
    out = np.zeros_like(raw)
    for g in np.unique(gids):
        members = np.nonzero(gids == g)[0]
        if weighting == "token":
            idx = np.concatenate([np.arange(bounds[k], bounds[k + 1]) for k in members]) \
                if len(members) else np.zeros(0, dtype=np.int64)
            if idx.size == 0:
                continue
            vals = raw[idx]
            mean = float(np.mean(vals))
            std = float(np.std(vals))
            denom = std + eps
            out[idx] = 0.0 if denom == 0.0 else (vals - mean) / denom
        elif weighting == "sequence":
            nonempty = [k for k in members if bounds[k + 1] > bounds[k]]
            if not nonempty:
                continue
            seq = np.array([raw[bounds[k]] for k in nonempty])
            mean = float(np.mean(seq))
            std = float(np.std(seq))
            denom = std + eps
            for k in nonempty:
                s, e = bounds[k], bounds[k + 1]
                out[s:e] = 0.0 if denom == 0.0 else (raw[s:e] - mean) / denom
        else:
            raise OracleBatchError(f"unknown weighting {weighting!r}")
    return out


def advantages(rewards, traj_bounds, mode="reference", gamma=1.0, lam=1.0, values=None,
               norm="global", group_ids=None, eps=0.0, weighting="token"):
    """Front door for all advantage variants (reference mode = trainer.py:114-125)."""
    if mode == "reference":
        return compute_advantages_ref(rewards, traj_bounds)
    raw = gae_raw(rewards, traj_bounds, gamma, lam, values)
    if norm == "global":
        return normalize_global(raw)
    if norm == "group":
        return normalize_group(raw, traj_bounds, group_ids, eps, weighting)
    if norm == "none":
        return raw
    raise OracleBatchError(f"unknown norm {norm!r}")


# ---------------------------------------------------------------------------
# dynamic micro-batch allocation  (trainer.py:235-270; PAPER Alg. 1)
# ---------------------------------------------------------------------------

def allocate_microbatches(lengths, capacity, min_groups=1):
    """Alg. 1 restated: longest first (stable, trainer.py:253); open a new group
    while fewer than min_groups exist or none fits (259-261); else join the
    fitting group with the fewest members, lowest index on ties (263-265)."""
    lengths = [int(s) for s in lengths]
    if min_groups < 1:
        raise OracleBatchError("min_groups must be >= 1")
    for s in lengths:
        if s < 1:
            raise OracleBatchError(f"sequence lengths must be positive, got {s}")
        if s > capacity:
            raise OracleBatchError(f"sequence length {s} exceeds capacity {capacity}")
    order = sorted(range(len(lengths)), key=lambda i: (-lengths[i], i))
    groups, totals = [], []
    for i in order:
        s = lengths[i]
        best = None
        for g in range(len(groups)):
            if totals[g] + s <= capacity:
                key = (len(groups[g]), g)
                if best is None or key < best[0]:
                    best = (key, g)
        if len(groups) < min_groups or best is None:
            groups.append([i])
            totals.append(s)
        else:
            groups[best[1]].append(i)
            totals[best[1]] += s
    return tuple(tuple(g) for g in groups)


def minibatch_splits(n_traj, minibatches):
    """np.array_split(arange(n), k) with empty chunks dropped (trainer.py:300-301)."""
    return [s for s in np.array_split(np.arange(n_traj), minibatches) if len(s) > 0]


def train_step_plan(traj_bounds, minibatches, capacity, min_groups):
    """Minibatch/micro-batch structure of train_step (trainer.py:299-320).

    Returns a list (one per non-empty minibatch) of dicts with ``traj_ids``
    (non-empty trajectories, trainer.py:310), ``groups`` (local indices) and
    ``gather`` (per group: packed token indices in placement order, 320).
    """
    bounds = np.asarray(traj_bounds, dtype=np.int64)
    out = []
    for mb in minibatch_splits(len(bounds) - 1, minibatches):
        traj_ids = [int(k) for k in mb if bounds[k + 1] > bounds[k]]
        if not traj_ids:
            continue
        lengths = [int(bounds[k + 1] - bounds[k]) for k in traj_ids]
        groups = allocate_microbatches(lengths, capacity, min_groups)
        gathers = [np.concatenate([np.arange(bounds[traj_ids[j]], bounds[traj_ids[j] + 1])
                                   for j in g]) for g in groups]
        out.append({"traj_ids": traj_ids, "groups": groups, "gather": gathers})
    return out


# ---------------------------------------------------------------------------
# linear-policy train step, for drop-in parity with the reference
# (trainer.py:285-346, policy.py:216-258)
# ---------------------------------------------------------------------------

@dataclass
class AdamCfg:
    """Same defaults as policy.AdamConfig (policy.py:186-195)."""
    lr: float = 2e-2
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-5
    weight_decay: float = 0.05
    clip_norm: float = 1.0


def linear_logits(features, W, b):
    """feats @ W.T + b (trainer.py:163; policy.py:162)."""
    return np.asarray(features) @ np.asarray(W).T + np.asarray(b)


def linear_loss(features, tokens, behav, prox, adv, W, b, clip_eps=0.2, decoupled=True):
    """_ppo_loss over the whole batch (trainer.py:198-213)."""
    t = surrogate_terms(linear_logits(features, W, b), tokens, behav, prox, adv,
                        clip_eps, decoupled)
    s = t["stats"]
    n = max(int(s[1]), 1)
    d = t["dlogits"] / n  # d(loss)/d(logits)
    gw = d.T @ np.asarray(features)
    gb = d.sum(axis=0)
    return {"loss": -s[0] / n, "grad_w": gw, "grad_b": gb, "n_tokens": int(s[1]),
            "clip_fraction": s[2] / n, "mean_ratio": s[3] / n, "excluded": int(s[4])}


def adam_update(W, b, gw, gb, m_w, v_w, m_b, v_b, step, cfg: AdamCfg):
    """apply_update restated (policy.py:215-258): non-finite check, clip_by_global_norm,
    Adam with decoupled weight decay; grads already scaled by -1/n (trainer.py:330)."""
    if not (np.all(np.isfinite(gw)) and np.all(np.isfinite(gb))):
        raise FloatingPointError("non-finite gradient")
    norm = math.sqrt(float(np.sum(gw ** 2) + np.sum(gb ** 2)))
    if cfg.clip_norm > 0 and norm > cfg.clip_norm:
        f = cfg.clip_norm / norm
        gw, gb = gw * f, gb * f
    step += 1
    b1, b2 = cfg.beta1, cfg.beta2
    m_w = b1 * m_w + (1 - b1) * gw
    v_w = b2 * v_w + (1 - b2) * gw ** 2
    m_b = b1 * m_b + (1 - b1) * gb
    v_b = b2 * v_b + (1 - b2) * gb ** 2
    c1, c2 = 1 - b1 ** step, 1 - b2 ** step
    W = W - cfg.lr * ((m_w / c1) / (np.sqrt(v_w / c2) + cfg.eps) + cfg.weight_decay * W)
    b = b - cfg.lr * ((m_b / c1) / (np.sqrt(v_b / c2) + cfg.eps) + cfg.weight_decay * b)
    return W, b, m_w, v_w, m_b, v_b, step


def linear_train_step(features, tokens, behav, traj_bounds, rewards, W, b, adam_state=None,
                      clip_eps=0.2, minibatches=4, capacity=512, min_groups=1,
                      decoupled=True, adam: AdamCfg | None = None):
    """train_step restated for the linear policy (trainer.py:285-346)."""
    adam = adam or AdamCfg()
    W = np.array(W, dtype=np.float64)
    b = np.array(b, dtype=np.float64)
    if adam_state is None:
        adam_state = (np.zeros_like(W), np.zeros_like(W), np.zeros_like(b), np.zeros_like(b), 0)
    m_w, v_w, m_b, v_b, step = adam_state
    feats = np.asarray(features, dtype=np.float64)
    prox = token_logprobs(linear_logits(feats, W, b), tokens)  # 295
    adv = compute_advantages_ref(rewards, traj_bounds)  # 296
    loss_sum = clip_sum = ratio_sum = 0.0
    token_total = excluded = micro = updates = 0
    for mb in train_step_plan(traj_bounds, minibatches, capacity, min_groups):
        gw = np.zeros_like(W)
        gb = np.zeros_like(b)
        obj = 0.0
        n_valid = 0
        for idx in mb["gather"]:
            t = surrogate_terms(linear_logits(feats[idx], W, b), np.asarray(tokens)[idx],
                                np.asarray(behav)[idx], prox[idx], adv[idx], clip_eps, decoupled)
            s = t["stats"]
            gw += t["dlogits"].T @ feats[idx]
            gb += t["dlogits"].sum(axis=0)
            obj += s[0]
            n_valid += int(s[1])
            clip_sum += s[2]
            ratio_sum += s[3]
            excluded += int(s[4])
            micro += 1
        n = max(n_valid, 1)
        gw /= n
        gb /= n
        W, b, m_w, v_w, m_b, v_b, step = adam_update(W, b, gw, gb, m_w, v_w, m_b, v_b, step, adam)
        updates += 1
        loss_sum += -obj
        token_total += n_valid
    d = max(token_total, 1)
    stats = {"loss": loss_sum / d, "clip_fraction": clip_sum / d, "mean_ratio": ratio_sum / d,
             "tokens": int(np.asarray(tokens).size), "minibatch_updates": updates,
             "microbatches": micro, "excluded_tokens": excluded}
    return W, b, (m_w, v_w, m_b, v_b, step), stats, prox, adv
