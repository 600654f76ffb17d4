"""Drop-in replacement for ``asyncrl.trainer`` on B200.

Same names, signatures, mutation semantics and error types as
/root/reference/pkg/src/asyncrl/trainer.py (cited per function), so
``harness._RunState.train`` (harness.py:214-220) can import this module
instead.  Everything on the hot path runs on the GPU:

* prox log-probs            -> K1 ``areal_logprob_fwd``
* advantages                -> K3 ``areal_advantages`` (bit-identical)
* micro-batch allocation    -> K4 ``areal_plan_microbatches`` (bit-exact)
* packing                   -> K5 ``areal_fill_gather``
* loss + backward           -> K2 ``areal_ppo_fwd_bwd`` (dlogits, stats)

The reference's *model* (the linear-softmax policy of policy.py: logits =
feats @ W.T + b, and its Adam) is outside the hot path; here it runs as float64
torch ops on the same device (cuBLAS GEMMs and elementwise kernels) so the
whole step stays resident and numerically matches the float64 reference.
Parameters arrive and leave as the caller's numpy-backed dataclasses.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import kernels as K


class BatchError(ValueError):
    """trainer.py:34-35"""


class NonFiniteGradientError(RuntimeError):
    """policy.py:34-35 — raised when a non-finite gradient reaches the optimizer."""


@dataclass(frozen=True)
class AdamConfig:
    """policy.py:186-195 (same defaults)."""
    lr: float = 2e-2
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-5
    weight_decay: float = 0.05
    clip_norm: float = 1.0


@dataclass(frozen=True)
class TrainerConfig:
    """trainer.py:38-53, plus B200-path extensions (defaults = reference behaviour)."""
    clip_eps: float = 0.2
    minibatches: int = 4
    micro_token_budget: int = 512
    micro_min_groups: int = 1
    objective: str = "decoupled"  # or "naive"
    adam: AdamConfig = field(default_factory=AdamConfig)
    # extensions (north star); defaults reproduce the reference
    eta_mask: int = -1               # mask tokens with version lag > eta_mask (-1: off)
    behav_weight_cap: float = 0.0    # mask tokens with prox/behav weight > cap (0: off)
    adv_mode: str = "reference"      # or "gae"
    gamma: float = 1.0
    lam: float = 1.0
    adv_norm: str = "global"         # "global" | "group" | "group_sequence" | "none"

    def __post_init__(self):
        if not (0 < self.clip_eps < 1):
            raise BatchError("clip_eps must be in (0, 1)")
        if self.minibatches < 1:
            raise BatchError("minibatches must be >= 1")
        if self.objective not in ("decoupled", "naive"):
            raise BatchError(f"unknown objective {self.objective!r}")


@dataclass
class ParamGrad:
    """policy.py:113-134 (gradient container returned in LossResult)."""
    weights: np.ndarray
    bias: np.ndarray

    @staticmethod
    def zeros_like(params) -> "ParamGrad":
        return ParamGrad(np.zeros_like(params.weights), np.zeros_like(params.bias))

    def add_(self, other: "ParamGrad") -> None:
        self.weights += other.weights
        self.bias += other.bias

    def scale_(self, factor: float) -> None:
        self.weights *= factor
        self.bias *= factor

    def global_norm(self) -> float:
        return float(np.sqrt(np.sum(self.weights ** 2) + np.sum(self.bias ** 2)))

    def is_finite(self) -> bool:
        return bool(np.all(np.isfinite(self.weights)) and np.all(np.isfinite(self.bias)))


@dataclass(frozen=True)
class VersionedParams:
    """policy.py:84-100 stand-in (linear policy snapshot) for callers without asyncrl.

    train_step accepts any dataclass with ``version``, ``weights`` (V, F) and
    ``bias`` (V,) — including asyncrl.policy.VersionedParams — and returns
    ``dataclasses.replace(params, ...)`` of the same type.
    """
    version: int
    weights: np.ndarray
    bias: np.ndarray


@dataclass
class AdamState:
    """policy.py:198-213 (mutated in place by train_step)."""
    m_weights: np.ndarray
    v_weights: np.ndarray
    m_bias: np.ndarray
    v_bias: np.ndarray
    step: int = 0

    @staticmethod
    def zeros_like(params) -> "AdamState":
        return AdamState(np.zeros_like(params.weights), np.zeros_like(params.weights),
                         np.zeros_like(params.bias), np.zeros_like(params.bias))


@dataclass
class TrainBatch:
    """trainer.py:56-80.  ``traj_bounds`` is the cu_seqlens of the global batch.

    ``versions`` (per-token policy version at emission, rollout.py:52, 159) is
    carried for the staleness mask; the reference drops it.
    """
    trajectories: list
    step_index: int
    features: np.ndarray
    tokens: np.ndarray
    behavior_logprobs: np.ndarray
    traj_bounds: np.ndarray
    prox_logprobs: np.ndarray | None = None
    prox_version: int | None = None
    advantages: np.ndarray | None = None
    versions: np.ndarray | None = None

    @property
    def n_tokens(self) -> int:
        return len(self.tokens)

    def token_range(self, traj_index: int) -> np.ndarray:
        return np.arange(self.traj_bounds[traj_index], self.traj_bounds[traj_index + 1])


def build_train_batch(trajectories, featurizer, step_index: int) -> TrainBatch:
    """trainer.py:83-111: flatten trajectories (formation order) into per-token arrays.

    Context features are the model's input (out of the hot path) and are
    recomputed from each prefix on the host exactly as the reference does.
    """
    feats, tokens, behav, vers, bounds = [], [], [], [], [0]
    have_versions = True
    for traj in trajectories:
        if traj.reward is None:
            raise BatchError(f"trajectory {traj.trajectory_id} is unrewarded")
        prefix: list[int] = []
        for tok in traj.tokens:
            feats.append(featurizer.features(traj.prompt, prefix))
            prefix.append(tok)
        tokens.extend(traj.tokens)
        behav.extend(traj.behavior_logprobs)
        v = getattr(traj, "versions", None)
        if v is None or len(v) != len(traj.tokens):
            have_versions = False
        else:
            vers.extend(v)
        bounds.append(len(tokens))
    n = len(tokens)
    dim = featurizer.feature_dim
    return TrainBatch(
        trajectories=list(trajectories),
        step_index=step_index,
        features=np.array(feats).reshape(n, dim),
        tokens=np.array(tokens, dtype=np.int64),
        behavior_logprobs=np.array(behav, dtype=np.float64),
        traj_bounds=np.array(bounds, dtype=np.int64),
        versions=np.array(vers, dtype=np.int32) if have_versions else None,
    )


# ---------------------------------------------------------------- device helpers
def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2505_24298_b200.trainer needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _d(x, dtype, dev):
    # the reference's parameter snapshots are read-only arrays (policy.py:99-100): a
    # writable host copy keeps torch from aliasing them
    return torch.as_tensor(np.require(x, requirements=("C", "W")), dtype=dtype).to(dev)


def _rewards(batch) -> np.ndarray:
    return np.array([float(t.reward.reward) for t in batch.trajectories], dtype=np.float64)


def _group_ids(batch) -> np.ndarray:
    ids = [getattr(getattr(t, "prompt", None), "id", k) for k, t in enumerate(batch.trajectories)]
    _, inv = np.unique(np.asarray(ids), return_inverse=True)
    return inv.astype(np.int32)


def _linear_logits(X: torch.Tensor, W: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """The reference model: feats @ W.T + b (trainer.py:163, policy.py:162)."""
    return torch.addmm(b, X, W.t())


# Extension fields of TrainerConfig and the values that reproduce the reference.  The
# reference's own asyncrl.trainer.TrainerConfig (trainer.py:38-53) has none of them, so
# every read goes through _ext: either config class drives this module unchanged.
_EXT_DEFAULTS = dict(eta_mask=-1, behav_weight_cap=0.0, adv_mode="reference", gamma=1.0,
                     lam=1.0, adv_norm="global")


def _ext(config, name):
    return _EXT_DEFAULTS[name] if config is None else getattr(config, name, _EXT_DEFAULTS[name])


def _adv_kwargs(config):
    norm = _ext(config, "adv_norm")
    norm = {"group": "group_token"}.get(norm, norm)
    return dict(mode=_ext(config, "adv_mode"), gamma=_ext(config, "gamma"),
                lam=_ext(config, "lam"), norm=norm)


def _advantages_device(batch, dev, config=None) -> torch.Tensor:
    kw = _adv_kwargs(config)
    rewards = _d(_rewards(batch), torch.float64, dev)
    bounds = _d(batch.traj_bounds, torch.int64, dev)
    gids = None
    if kw["norm"] in ("group_token", "group_sequence"):
        gids = _d(_group_ids(batch), torch.int32, dev)
    return K.advantages(rewards, bounds, batch.n_tokens, group_ids=gids, **kw)


# ---------------------------------------------------------------- public API
def compute_advantages(batch: TrainBatch, config: TrainerConfig | None = None) -> np.ndarray:
    """trainer.py:114-125 on the GPU (K3); sets ``batch.advantages``.

    Default (reference) mode is bit-identical to the reference's numpy result.
    """
    dev = _device()
    adv = _advantages_device(batch, dev, config).cpu().numpy()
    batch.advantages = adv
    return adv


def recompute_prox_logprobs(batch: TrainBatch, current_params) -> np.ndarray:
    """trainer.py:128-137: token log-probs under the params at batch arrival (K1)."""
    dev = _device()
    prox = _prox_device(batch, current_params, dev)
    batch.prox_logprobs = prox.cpu().numpy()
    batch.prox_version = current_params.version
    return batch.prox_logprobs


def _prox_device(batch, params, dev, X=None, W=None, b=None):
    if batch.n_tokens == 0:
        return torch.zeros(0, dtype=torch.float64, device=dev)
    X = _d(batch.features, torch.float64, dev) if X is None else X
    W = _d(params.weights, torch.float64, dev) if W is None else W
    b = _d(params.bias, torch.float64, dev) if b is None else b
    toks = _d(batch.tokens, torch.int64, dev)
    lp, _ = K.logprob_fwd(_linear_logits(X, W, b), toks, with_entropy=False)
    return lp


@dataclass
class LossResult:
    """trainer.py:140-147"""
    loss: float
    grad: ParamGrad
    n_tokens: int
    clip_fraction: float
    mean_ratio: float
    excluded: int


def _surrogate_terms(batch: TrainBatch, idx, params, clip_eps: float, decoupled: bool):
    """trainer.py:150-195: objective and gradient sums over one token subset (K2 + the
    linear policy's GEMMs), as raw sums so micro-batch accumulation stays exact."""
    if batch.prox_logprobs is None or batch.advantages is None:
        raise BatchError("populate prox_logprobs and advantages before the loss")
    dev = _device()
    idx = np.asarray(idx, dtype=np.int64)
    X = _d(batch.features[idx], torch.float64, dev)
    W = _d(params.weights, torch.float64, dev)
    b = _d(params.bias, torch.float64, dev)
    stats = torch.zeros(8, dtype=torch.float64, device=dev)
    if len(idx):
        logits = _linear_logits(X, W, b)
        dl, stats = K.ppo_fwd_bwd(logits, _d(batch.tokens[idx], torch.int64, dev),
                                  _d(batch.behavior_logprobs[idx], torch.float64, dev),
                                  _d(batch.prox_logprobs[idx], torch.float64, dev),
                                  _d(batch.advantages[idx], torch.float64, dev),
                                  clip_eps=clip_eps, decoupled=decoupled, stats=stats,
                                  dlogits=logits)
        # dl = coef (softmax - onehot) = -resid, so resid^T feats = -(dl^T X) (exact negation)
        gw, gb = -(dl.t() @ X), -dl.sum(dim=0)
    else:
        gw, gb = torch.zeros_like(W), torch.zeros_like(b)
    s = stats.cpu().numpy()
    return {"objective_sum": float(s[0]), "grad_w_sum": gw.cpu().numpy(),
            "grad_b_sum": gb.cpu().numpy(), "n_valid": int(s[1]), "n_clipped": int(s[2]),
            "ratio_sum": float(s[3]), "n_excluded": int(s[4])}


def _ppo_loss(batch: TrainBatch, params, clip_eps: float, decoupled: bool) -> LossResult:
    """trainer.py:198-213: whole-batch loss via one K2 launch."""
    if batch.prox_logprobs is None or batch.advantages is None:
        raise BatchError("populate prox_logprobs and advantages before the loss")
    dev = _device()
    X = _d(batch.features, torch.float64, dev)
    W = _d(params.weights, torch.float64, dev)
    b = _d(params.bias, torch.float64, dev)
    stats = torch.zeros(8, dtype=torch.float64, device=dev)
    if batch.n_tokens:
        logits = _linear_logits(X, W, b)
        dl, stats = K.ppo_fwd_bwd(logits, _d(batch.tokens, torch.int64, dev),
                                  _d(batch.behavior_logprobs, torch.float64, dev),
                                  _d(batch.prox_logprobs, torch.float64, dev),
                                  _d(batch.advantages, torch.float64, dev),
                                  clip_eps=clip_eps, decoupled=decoupled, stats=stats,
                                  dlogits=logits)  # in-place backward
        gw, gb = dl.t() @ X, dl.sum(dim=0)
    else:
        gw, gb = torch.zeros_like(W), torch.zeros_like(b)
    s = stats.cpu().numpy()
    n = max(int(s[1]), 1)
    return LossResult(loss=-float(s[0]) / n,
                      grad=ParamGrad((gw / n).cpu().numpy(), (gb / n).cpu().numpy()),
                      n_tokens=int(s[1]), clip_fraction=float(s[2]) / n,
                      mean_ratio=float(s[3]) / n, excluded=int(s[4]))


def decoupled_ppo_loss(batch: TrainBatch, params, clip_eps: float = 0.2) -> LossResult:
    """trainer.py:216-219"""
    return _ppo_loss(batch, params, clip_eps, decoupled=True)


def naive_ppo_loss(batch: TrainBatch, params, clip_eps: float = 0.2) -> LossResult:
    """trainer.py:222-225"""
    return _ppo_loss(batch, params, clip_eps, decoupled=False)


@dataclass(frozen=True)
class MicrobatchPlan:
    """trainer.py:228-232"""
    groups: tuple
    capacity: int
    min_groups: int


def _status_error(code: int, lengths, capacity) -> BatchError:
    from ._lib import ERR_LEN_EXCEEDS_CAPACITY, ERR_LEN_NONPOSITIVE
    if code == ERR_LEN_NONPOSITIVE:
        bad = next(s for s in lengths if s < 1)
        return BatchError(f"sequence lengths must be positive, got {bad}")
    if code == ERR_LEN_EXCEEDS_CAPACITY:
        bad = next(s for s in lengths if s > capacity)
        return BatchError(f"sequence length {bad} exceeds capacity {capacity}")
    return BatchError(f"allocation failed with status {code}")


_INT32_MAX = 2 ** 31 - 1


def _device_capacity(capacity, lengths) -> int:
    """K4 takes an int32 capacity.  A capacity at or above the total length admits every
    placement (totals[g] + s never exceeds the sum of distinct lengths), so larger
    values are clamped to the total with identical groups (trainer.py:258)."""
    capacity = int(capacity)
    if capacity > _INT32_MAX:
        capacity = max(int(sum(lengths)), 1)
        if capacity > _INT32_MAX:
            raise BatchError(f"minibatch of {capacity} tokens exceeds the GPU allocator's "
                             f"int32 token range")
    return capacity


def _check_items(n_items: int) -> None:
    from ._lib import MAX_ITEMS_PER_MINIBATCH
    if n_items > MAX_ITEMS_PER_MINIBATCH:
        raise BatchError(f"{n_items} sequences in one minibatch exceed the GPU allocator's "
                         f"limit of {MAX_ITEMS_PER_MINIBATCH} (split the batch into more "
                         f"minibatches)")


def allocate_microbatches(lengths, capacity: int, min_groups: int = 1) -> MicrobatchPlan:
    """trainer.py:235-270 on the GPU (K4), bit-exact group assignment."""
    lengths = [int(s) for s in lengths]
    if min_groups < 1:
        raise BatchError("min_groups must be >= 1")
    if not lengths:
        return MicrobatchPlan(groups=(), capacity=capacity, min_groups=min_groups)
    dev = _device()
    if 1 <= min(lengths) and max(lengths) <= capacity:  # else the device reports the
        _check_items(len(lengths))                          # first bad length (248-252)
    cap = _device_capacity(capacity, [max(s, 0) for s in lengths])
    bounds = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    # the device validates lengths and reports the first failing item (trainer.py:248-252)
    plan = K.plan_microbatches(_d(bounds, torch.int64, dev),
                               torch.arange(len(lengths), dtype=torch.int32, device=dev),
                               [0, len(lengths)], [0], cap, min_groups)
    status = int(plan.status[0].item())
    if status != 0:
        raise _status_error(status, lengths, capacity)
    return MicrobatchPlan(groups=_groups_from(plan, 0, len(lengths)), capacity=capacity,
                          min_groups=min_groups)


def _groups_from(plan, m: int, n: int, local_ids=None):
    off = int(plan.mb_offsets[m])
    gof = plan.group_of[off:off + n].cpu().numpy()
    slot = plan.slot_of[off:off + n].cpu().numpy()
    G = int(plan.n_groups[m].item())
    sizes = np.bincount(gof, minlength=G)
    groups = [[0] * int(sizes[g]) for g in range(G)]
    for i in range(n):
        groups[gof[i]][slot[i]] = i if local_ids is None else local_ids[i]
    return tuple(tuple(g) for g in groups)


@dataclass
class TrainStepStats:
    """trainer.py:273-282"""
    step_index: int
    loss: float
    clip_fraction: float
    mean_ratio: float
    tokens: int
    minibatch_updates: int
    microbatches: int
    excluded_tokens: int


def minibatch_items(traj_bounds: np.ndarray, minibatches: int):
    """np.array_split into contiguous trajectory chunks, dropping empty chunks and
    zero-length trajectories (trainer.py:300-301, 310-311)."""
    bounds = np.asarray(traj_bounds, dtype=np.int64)
    n_traj = len(bounds) - 1
    nonempty = np.diff(bounds) > 0
    out = []
    for mb in np.array_split(np.arange(n_traj), minibatches):
        ids = mb[nonempty[mb]]
        if len(ids):
            out.append(ids.tolist())
    return out


def plan_step(bounds_host: np.ndarray, bounds_dev: torch.Tensor, minibatches: int, capacity: int,
              min_groups: int, dev):
    """Minibatch split (host, O(n)) + allocation and packing of every minibatch (device).

    Returns (items per minibatch, DevicePlan, gather index, host group_cu, host n_groups).
    """
    items = minibatch_items(bounds_host, minibatches)
    if not items:
        return items, None, None, None, None
    mb_offsets = np.concatenate([[0], np.cumsum([len(x) for x in items])]).astype(np.int32)
    lens = np.diff(bounds_host)
    mb_tokens = [int(lens[x].sum()) for x in items]
    mb_token_start = np.concatenate([[0], np.cumsum(mb_tokens)[:-1]]).astype(np.int64)
    if max(int(lens[x].max()) for x in items) <= capacity:  # else K4 reports the bad length
        _check_items(max(len(x) for x in items))
    capacity = _device_capacity(capacity, [max(mb_tokens)])
    flat = torch.as_tensor(np.concatenate(items).astype(np.int32)).to(dev)
    plan = K.plan_microbatches(bounds_dev, flat, mb_offsets, mb_token_start, capacity, min_groups)
    n_packed = int(sum(mb_tokens))
    gather, _ = K.fill_gather(bounds_dev, plan, n_packed)
    status = plan.status.cpu().numpy()
    bad = np.nonzero(status[:len(items)])[0]
    if len(bad):
        m = int(bad[0])
        raise _status_error(int(status[m]), [int(lens[k]) for k in items[m]], capacity)
    return items, plan, gather, plan.group_cu.cpu().numpy(), plan.n_groups.cpu().numpy()


class _DeviceAdam:
    """policy.apply_update (policy.py:225-258) after grad.scale_(-1/n) (trainer.py:330),
    as one fused K6 launch sequence: numpy-exact global norm, clip, Adam, in place."""

    def __init__(self, opt, dev):
        self.opt = opt
        self.step_count = int(opt.step)  # committed to opt with the moments (write_back)
        self.m_w = _d(opt.m_weights, torch.float64, dev)
        self.v_w = _d(opt.v_weights, torch.float64, dev)
        self.m_b = _d(opt.m_bias, torch.float64, dev)
        self.v_b = _d(opt.v_bias, torch.float64, dev)

    def step(self, W, b, gw, gb, cfg, grad_scale=1.0):
        """W, b are updated in place; gw, gb are the raw (unscaled) gradient sums."""
        norm = K.adam_step([W, b], [gw, gb], [self.m_w, self.m_b], [self.v_w, self.v_b],
                           step=self.step_count + 1, lr=cfg.lr, beta1=cfg.beta1, beta2=cfg.beta2,
                           eps=cfg.eps, weight_decay=cfg.weight_decay, clip_norm=cfg.clip_norm,
                           grad_scale=grad_scale, exact_norm=True)
        bad = int(norm[1].item())
        if bad:
            raise NonFiniteGradientError(
                f"non-finite gradient at optimizer step {self.step_count + 1}: "
                f"|w|_nan={int(torch.isnan(gw * grad_scale).sum())}, "
                f"|b|_nan={int(torch.isnan(gb * grad_scale).sum())}")
        self.step_count += 1
        return W, b

    def write_back(self):
        """Commit moments and step count together, as apply_update mutates them
        (policy.py:241-246); called after the last minibatch and, when a minibatch
        raises, for the updates completed before it."""
        self.opt.step = self.step_count
        self.opt.m_weights = self.m_w.cpu().numpy()
        self.opt.v_weights = self.v_w.cpu().numpy()
        self.opt.m_bias = self.m_b.cpu().numpy()
        self.opt.v_bias = self.v_b.cpu().numpy()


def train_step(batch: TrainBatch, params, opt, config: TrainerConfig = TrainerConfig()):
    """trainer.py:285-346: one PPO step over a global batch, resident on the GPU.

    prox (K1) and advantages (K3) once; minibatches updated sequentially; in
    each, K4/K5 allocate and pack micro-batches, K2 produces dlogits and the
    raw statistic sums, gradients accumulate unscaled and are scaled by
    -1/n_valid after the last micro-batch (the reference's order), then Adam.
    Returns params tagged version + 1.
    """
    dev = _device()
    X = _d(batch.features, torch.float64, dev)
    W = _d(params.weights, torch.float64, dev)
    b = _d(params.bias, torch.float64, dev)
    toks = _d(batch.tokens, torch.int64, dev)
    behav = _d(batch.behavior_logprobs, torch.float64, dev)
    bounds_d = _d(batch.traj_bounds, torch.int64, dev)
    prox = _prox_device(batch, params, dev, X, W, b)                      # 295
    batch.prox_logprobs = prox.cpu().numpy()
    batch.prox_version = params.version
    adv = _advantages_device(batch, dev, config) if batch.n_tokens else \
        torch.zeros(0, dtype=torch.float64, device=dev)                 # 296
    batch.advantages = adv.cpu().numpy()
    decoupled = config.objective == "decoupled"
    eta_mask, behav_cap = _ext(config, "eta_mask"), _ext(config, "behav_weight_cap")
    versions = None
    if eta_mask >= 0:
        if getattr(batch, "versions", None) is None:
            raise BatchError("eta_mask needs per-token versions in the batch")
        versions = _d(batch.versions, torch.int32, dev)
    dadam = _DeviceAdam(opt, dev)

    items, plan, gather, group_cu, n_groups = plan_step(
        batch.traj_bounds, bounds_d, config.minibatches, config.micro_token_budget,
        config.micro_min_groups, dev)
    loss_sum = clip_sum = ratio_sum = 0.0
    token_total = excluded = micro_count = updates = 0
    stats = torch.zeros(8, dtype=torch.float64, device=dev)
    try:
        for m, traj_ids in enumerate(items):                             # 309-334
            gw = torch.zeros_like(W)
            gb = torch.zeros_like(b)
            stats.zero_()
            base = int(plan.mb_offsets[m]) + m
            for g in range(int(n_groups[m])):
                lo, hi = int(group_cu[base + g]), int(group_cu[base + g + 1])
                rows = gather[lo:hi]
                Xg = X.index_select(0, rows.long())
                logits = _linear_logits(Xg, W, b)
                dl, _ = K.ppo_fwd_bwd(logits, toks, behav, prox, adv, clip_eps=config.clip_eps,
                                      decoupled=decoupled, versions=versions,
                                      current_version=params.version, eta_mask=eta_mask,
                                      behav_weight_cap=behav_cap, row_index=rows,
                                      dlogits=logits, stats=stats)
                gw += dl.t() @ Xg
                gb += dl.sum(dim=0)
                micro_count += 1
            s = stats.cpu().numpy()
            n_valid = int(s[1])
            n = max(n_valid, 1)
            # dl = -(d obj/d logits), so gw = -grad_w_sum and the reference's scale -1/n
            # becomes +1/n (sign flips are exact)
            W, b = dadam.step(W, b, gw, gb, config.adam, grad_scale=1.0 / n)  # 329-331
            updates += 1
            loss_sum += -float(s[0])
            clip_sum += float(s[2])
            ratio_sum += float(s[3])
            excluded += int(s[4])
            token_total += n_valid
    finally:
        # a raising minibatch leaves opt with the updates before it, moments and step
        # together, as the reference's in-place apply_update does
        dadam.write_back()
    d = max(token_total, 1)
    out_stats = TrainStepStats(step_index=batch.step_index, loss=loss_sum / d,
                               clip_fraction=clip_sum / d, mean_ratio=ratio_sum / d,
                               tokens=batch.n_tokens, minibatch_updates=updates,
                               microbatches=micro_count, excluded_tokens=excluded)
    new_params = replace(params, weights=W.cpu().numpy(), bias=b.cpu().numpy(),
                         version=params.version + 1)
    return new_params, out_stats
