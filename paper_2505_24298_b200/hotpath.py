"""LM-scale decoupled-PPO hot path: packed rollouts -> advantages -> prox log-probs
-> micro-batch allocation/packing -> fused loss+backward, with data parallelism.

This is ``asyncrl.trainer.train_step`` (trainer.py:285-346) restated for a real
language model whose logits live on the GPU: the model is abstracted as two
callbacks, so this module owns exactly the hot path and nothing else.

    logits_fn(phase, minibatch, micro, rows) -> logits [len(rows), V] (CUDA)
        phase 'prox'  : forward under the params at batch arrival (K1 consumes it)
        phase 'train' : forward under the current params (K2 consumes it)
        rows          : int32 CUDA tensor, global token index of each packed row
    prox_head_fn(minibatch, micro, rows) -> (hidden [len(rows), d], W [V, d], bias|None)
        optional replacement of logits_fn for the 'prox' phase: the model hands over
        its final hidden states and LM head and K7 (tcgen05) computes the prox
        log-probs without materialising the [rows, V] logits
    backward_fn(minibatch, micro, dlogits)   -> model backward from dlogits (optional)
    update_fn(minibatch, stats)              -> optimizer step; stats is the
        all-reduced float64[8] device tensor of the minibatch, so the caller
        scales its accumulated gradients by 1 / max(stats[1], 1) (trainer.py:329-330)

Data parallelism: every rank computes the same plan (K4 is
deterministic, so no broadcast), the micro-batches of each minibatch are dealt
to ranks longest-processing-time first by token count, and the only collective
is one NCCL all-reduce of the 8 statistics per minibatch.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import kernels as K
from .trainer import BatchError, minibatch_items, _status_error, _check_items, _device_capacity

ADV_NORM_ALIASES = {"group": "group_token"}


@dataclass(frozen=True)
class HotPathConfig:
    """TrainerConfig (trainer.py:38-53) fields that the hot path reads, + extensions."""
    clip_eps: float = 0.2
    minibatches: int = 4
    micro_token_budget: int = 32768
    micro_min_groups: int = 1
    objective: str = "decoupled"
    eta_mask: int = -1
    behav_weight_cap: float = 0.0
    adv_mode: str = "reference"
    gamma: float = 1.0
    lam: float = 1.0
    adv_norm: str = "global"
    adv_eps: float = 0.0
    algo: str = "auto"
    # minibatch 0 trains under the batch-arrival params that define prox (trainer.py:295,
    # no update precedes it), so its prox log-probs ARE its current log-probs: K2
    # computes them in the same read of the logits (and the model skips that prox forward)
    fuse_first_prox: bool = True

    def __post_init__(self):
        if not (0 < self.clip_eps < 1):
            raise BatchError("clip_eps must be in (0, 1)")
        if self.minibatches < 1:
            raise BatchError("minibatches must be >= 1")
        if self.micro_min_groups < 1:
            raise BatchError("min_groups must be >= 1")
        if self.objective not in ("decoupled", "naive"):
            raise BatchError(f"unknown objective {self.objective!r}")


@dataclass
class PackedRollouts:
    """One global batch in formation order (controller.form_batch order), on device.

    traj_bounds is cu_seqlens (trainer.py:56-80 ``traj_bounds``); per-token
    arrays are indexed by global token; group_ids (GRPO) by trajectory.
    """
    traj_bounds: torch.Tensor
    traj_bounds_host: np.ndarray
    tokens: torch.Tensor
    behav: torch.Tensor
    rewards: torch.Tensor
    versions: torch.Tensor | None = None
    group_ids: torch.Tensor | None = None
    values: torch.Tensor | None = None

    @property
    def n_tokens(self) -> int:
        return int(self.traj_bounds_host[-1])

    @property
    def n_traj(self) -> int:
        return len(self.traj_bounds_host) - 1

    def h2d_bytes(self) -> int:
        ts = [self.traj_bounds, self.tokens, self.behav, self.rewards, self.versions,
              self.group_ids, self.values]
        return int(sum(t.numel() * t.element_size() for t in ts if t is not None))

    @staticmethod
    def from_host(traj_bounds, tokens, behav, rewards, versions=None, group_ids=None, values=None,
                  device=None, non_blocking=True):
        """Host (ideally pinned) arrays/tensors -> device copies on the current stream."""
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device

        def up(x, dtype):
            if x is None:
                return None
            t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
            return t.to(dtype).to(dev, non_blocking=non_blocking)

        bh = np.asarray(traj_bounds.numpy() if isinstance(traj_bounds, torch.Tensor)
                        else traj_bounds, dtype=np.int64)
        return PackedRollouts(up(traj_bounds, torch.int64), bh, up(tokens, torch.int64),
                              up(behav, torch.float64), up(rewards, torch.float64),
                              up(versions, torch.int32), up(group_ids, torch.int32),
                              up(values, torch.float64))


    @staticmethod
    def from_host_meta(host: "HostRollouts", device=None):
        """The trajectory-level arrays (cu_seqlens, rewards, group ids; GAE values whole,
        K3 scans every trajectory) uploaded; the per-token arrays allocated on the device
        and left for ``upload_token_ranges`` (a rank fills only the tokens it trains on)."""
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        up = lambda t, dt: None if t is None else t.to(dt).to(dev, non_blocking=True)
        T = int(host.traj_bounds[-1]) if host.traj_bounds.numel() else 0
        emp = lambda t, dt: None if t is None else torch.empty(T, dtype=dt, device=dev)
        return PackedRollouts(up(host.traj_bounds, torch.int64),
                              host.traj_bounds.numpy().astype(np.int64),
                              emp(host.tokens, torch.int64), emp(host.behav, torch.float64),
                              up(host.rewards, torch.float64), emp(host.versions, torch.int32),
                              up(host.group_ids, torch.int32), up(host.values, torch.float64))

    def upload_token_ranges(self, host: "HostRollouts", ranges) -> int:
        """Async H2D of the per-token arrays for global token ranges [(lo, hi)] only, at the
        same offsets (the device arrays stay indexed by global token).  Returns bytes."""
        n = 0
        for name in ("tokens", "behav", "versions"):
            src, dst = getattr(host, name), getattr(self, name)
            if src is None or dst is None:
                continue
            for lo, hi in ranges:
                dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
                n += (hi - lo) * dst.element_size()
        return n


@dataclass
class HostRollouts:
    """One global batch in formation order on the host (pinned tensors; the output of the
    native packer, ``pack_trajectories(..., device=None)``).  ``DecoupledPPOStep.run``
    uploads the trajectory-level arrays whole and the per-token arrays only for the
    trajectories of this rank's micro-batches (all of them on one GPU)."""
    traj_bounds: torch.Tensor
    tokens: torch.Tensor
    behav: torch.Tensor
    rewards: torch.Tensor
    versions: torch.Tensor | None = None
    group_ids: torch.Tensor | None = None
    values: torch.Tensor | None = None

    @staticmethod
    def from_arrays(traj_bounds, tokens, behav, rewards, versions=None, group_ids=None,
                    values=None, pin: bool = True):
        def h(x, dt):
            if x is None:
                return None
            t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
            t = t.to(dt).contiguous()
            return t.pin_memory() if pin and not t.is_pinned() else t
        return HostRollouts(h(traj_bounds, torch.int64), h(tokens, torch.int64),
                            h(behav, torch.float64), h(rewards, torch.float64),
                            h(versions, torch.int32), h(group_ids, torch.int32),
                            h(values, torch.float64))

    def h2d_bytes(self) -> int:
        ts = [self.traj_bounds, self.tokens, self.behav, self.rewards, self.versions,
              self.group_ids, self.values]
        return int(sum(t.numel() * t.element_size() for t in ts if t is not None))


def _packer():
    try:
        from . import _packer as P  # built by paper_2505_24298_b200.build (gcc)
    except ImportError as e:
        raise ImportError("the native rollout packer is not built: run "
                          "`python -m paper_2505_24298_b200.build`") from e
    return P


def pack_trajectories(trajectories, device=None, pin: bool = True, with_groups: bool = True,
                      upload: bool = True):
    """Replay-buffer trajectories (formation order) -> PackedRollouts on the GPU.

    build_train_batch (trainer.py:83-111) without the per-token Python loop: the
    native packer (csrc/packer.c) writes tokens / behaviour log-probs / per-token
    versions / cu_seqlens / rewards straight into pinned host tensors, which are
    copied to the device asynchronously on the current stream.  GRPO group ids are
    the dense ids of ``traj.prompt.id`` in first-appearance order (tasks.py:80, the
    harness's n_prompts x n_responses batch, harness.py:93-95).  Returns
    (PackedRollouts, host tensors) — keep the host tensors alive until the copies
    have completed (e.g. reuse them for the next batch).  ``upload=False`` returns
    (HostRollouts, host tensors) instead: ``DecoupledPPOStep.run`` then uploads only the
    tokens of this rank's micro-batches.
    """
    P = _packer()
    trajs = list(trajectories)
    T, n = P.count(trajs)
    alloc = (lambda *a, **k: torch.empty(*a, **k).pin_memory()) if pin else torch.empty
    host = dict(tokens=alloc(T, dtype=torch.int64), behav=alloc(T, dtype=torch.float64),
                versions=alloc(T, dtype=torch.int32), traj_bounds=alloc(n + 1, dtype=torch.int64),
                rewards=alloc(n, dtype=torch.float64))
    have_versions = P.fill(trajs, host["tokens"].data_ptr(), host["behav"].data_ptr(),
                           host["versions"].data_ptr(), host["traj_bounds"].data_ptr(),
                           host["rewards"].data_ptr(), T)
    if not have_versions:
        host["versions"] = None
    if with_groups:
        ids: dict = {}
        g = [ids.setdefault(getattr(getattr(t, "prompt", None), "id", k), len(ids))
             for k, t in enumerate(trajs)]
        host["group_ids"] = torch.tensor(g, dtype=torch.int32)
        if pin:
            host["group_ids"] = host["group_ids"].pin_memory()
    if not upload:
        return HostRollouts(**host), host
    ro = PackedRollouts.from_host(**host, device=device)
    return ro, host


@dataclass
class StepPlan:
    """Output of K4/K5 for one global batch plus this rank's share."""
    items: list                 # non-empty trajectory ids per minibatch
    device_plan: K.DevicePlan
    gather: torch.Tensor        # int32 [n_packed]: packed position -> global token
    group_cu: np.ndarray        # host copy of micro-batch token boundaries
    n_groups: np.ndarray        # host, per minibatch
    micro: list = field(default_factory=list)     # [(m, g, lo, hi)] all micro-batches
    mine: list = field(default_factory=list)      # per minibatch: this rank's [(g, lo, hi)]
    load: np.ndarray | None = None                # [M, world] tokens dealt to each rank
    host_seq: tuple | None = None                 # (group_seq_cu, packed_traj) host copies

    @property
    def n_micro(self) -> int:
        return len(self.micro)


def lpt_assign(sizes, world_size: int):
    """Longest-processing-time-first: deal items (by descending size, ties by index)
    to the least-loaded rank (ties by rank).  Deterministic on every rank."""
    order = sorted(range(len(sizes)), key=lambda i: (-int(sizes[i]), i))
    heap = [(0, r) for r in range(world_size)]
    owner = [0] * len(sizes)
    for i in order:
        load, r = heapq.heappop(heap)
        owner[i] = r
        heapq.heappush(heap, (load + int(sizes[i]), r))
    return owner


def shard_micro_batches(group_cu, n_groups, mb_offsets, world_size: int, rank: int,
                        with_load: bool = False):
    """Host-side DP sharding of a replicated plan.

    group_cu / n_groups / mb_offsets use the layout of areal_plan_microbatches.
    Returns (all micro-batches [(m, g, lo, hi)], this rank's [(g, lo, hi)] per
    minibatch), micro-batches dealt LPT by token count within each minibatch; with
    ``with_load`` also the [M, world] token load of every rank (identical on all ranks).
    """
    micro, mine = [], []
    load = np.zeros((len(n_groups), world_size), dtype=np.int64)
    for m in range(len(n_groups)):
        base = int(mb_offsets[m]) + m
        groups = [(g, int(group_cu[base + g]), int(group_cu[base + g + 1]))
                  for g in range(int(n_groups[m]))]
        micro.extend((m, g, lo, hi) for g, lo, hi in groups)
        owner = lpt_assign([hi - lo for _, lo, hi in groups], world_size)
        mine.append([grp for grp, r in zip(groups, owner) if r == rank])
        for (g, lo, hi), r in zip(groups, owner):
            load[m, r] += hi - lo
    return (micro, mine, load) if with_load else (micro, mine)


def load_summary(load: np.ndarray) -> dict:
    """Data-parallel balance of a plan: the step waits, minibatch by minibatch, for the
    busiest rank (the statistics all-reduce), so sum_m mean / sum_m max bounds the
    scaling efficiency the dealing allows."""
    if load is None or load.size == 0:
        return dict(rank_tokens=[], max_over_mean=1.0, efficiency_bound=1.0)
    per_rank = load.sum(axis=0)
    mx = load.max(axis=1).sum()
    return dict(rank_tokens=[int(x) for x in per_rank],
                max_over_mean=float(per_rank.max() / max(per_rank.mean(), 1e-9)),
                per_minibatch_max_over_mean=[float(r.max() / max(r.mean(), 1e-9)) for r in load],
                efficiency_bound=float(load.mean(axis=1).sum() / max(mx, 1)))


@dataclass
class StepResult:
    """TrainStepStats (trainer.py:273-282) fields + the raw per-minibatch sums."""
    loss: float
    clip_fraction: float
    mean_ratio: float
    tokens: int
    minibatch_updates: int
    microbatches: int
    excluded_tokens: int
    masked_tokens: int
    entropy: float
    minibatch_stats: np.ndarray   # [M, 8] all-reduced sums


class DecoupledPPOStep:
    """The hot path of one PPO step over a packed global batch (see module doc)."""

    def __init__(self, config: HotPathConfig = HotPathConfig(), device=None, group=None):
        self.cfg = config
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.world = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0
        self.launches = 0  # kernels launched by this object (K1-K5)
        self.k1_events: list = []
        self.k2_events: list = []
        self.k3_events: list = []   # advantages
        self.k45_events: list = []  # allocation + packing plan (incl. its one host read)
        self.k2_bytes = 0
        self.k1_bytes = 0
        self.k7_flops = 0
        self.record_events = False
        self._ev_pool: list = []  # reused timing events (no event creation per launch)
        self._ev_next = 0
        self._readback = None  # pinned buffer for the plan's host read
        self.h2d_bytes = 0     # host->device bytes of the last run() from HostRollouts
        self.last_plan = None

    # ---- K3
    def advantages(self, ro: PackedRollouts) -> torch.Tensor:
        c = self.cfg
        norm = ADV_NORM_ALIASES.get(c.adv_norm, c.adv_norm)
        adv = K.advantages(ro.rewards, ro.traj_bounds, ro.n_tokens, mode=c.adv_mode,
                           gamma=c.gamma, lam=c.lam, values=ro.values, norm=norm,
                           group_ids=ro.group_ids, eps=c.adv_eps)
        # global norm: one fused cooperative launch (+ the GAE scan before it)
        if norm == "global":
            self.launches += 1 if c.adv_mode == "reference" else 2
        else:
            self.launches += 1 + (1 if norm.startswith("group") else 0)
        return adv

    # ---- K4 + K5
    def plan(self, ro: PackedRollouts) -> StepPlan:
        return self._plan_finish(self._plan_launch(ro))

    def _plan_launch(self, ro: PackedRollouts, with_seq: bool = False):
        """Host split + K4, an async read of the plan's sizes into pinned memory, then
        K5: the host later waits for K4 and that read only (K5 and whatever the caller
        queues next, e.g. K3, run while it deals the micro-batches)."""
        c = self.cfg
        items = minibatch_items(ro.traj_bounds_host, c.minibatches)
        if not items:
            return items, None
        lens = np.diff(ro.traj_bounds_host)
        mb_offsets = np.concatenate([[0], np.cumsum([len(x) for x in items])]).astype(np.int32)
        mb_tokens = [int(lens[x].sum()) for x in items]
        mb_token_start = np.concatenate([[0], np.cumsum(mb_tokens)[:-1]]).astype(np.int64)
        flat = np.concatenate(items).astype(np.int32)  # staged with the offsets, one copy
        cap = c.micro_token_budget
        if max(int(lens[x].max()) for x in items) <= cap:  # else K4 reports the bad length
            _check_items(max(len(x) for x in items))
        dplan = K.plan_microbatches(ro.traj_bounds, flat, mb_offsets, mb_token_start,
                                    _device_capacity(cap, [max(mb_tokens)]), c.micro_min_groups)
        # the single host read of the plan: micro-batch sizes drive the model's shapes
        # (+ which trajectories each micro-batch packs, when the rank uploads only its own)
        M, n_gc = len(items), dplan.group_cu.numel()
        n_it = dplan.packed_traj.numel()
        need = 16 * M + 8 * n_gc + (4 * (n_gc + n_it) + 16 if with_seq else 0)
        if self._readback is None or self._readback.numel() < need:
            self._readback = torch.empty(max(2 * need, 4096), dtype=torch.uint8).pin_memory()
        rb = self._readback
        gcu = rb[:8 * n_gc].view(torch.int64)
        st = rb[8 * n_gc:8 * n_gc + 4 * M].view(torch.int32)
        ng = rb[8 * n_gc + 8 * M:8 * n_gc + 12 * M].view(torch.int32)
        gcu.copy_(dplan.group_cu, non_blocking=True)
        st.copy_(dplan.status[:M], non_blocking=True)
        ng.copy_(dplan.n_groups[:M], non_blocking=True)
        seq = None
        if with_seq:
            o = 8 * n_gc + 16 * M
            gsc = rb[o:o + 4 * n_gc].view(torch.int32)
            ptr = rb[o + 4 * n_gc:o + 4 * (n_gc + n_it)].view(torch.int32)
            gsc.copy_(dplan.group_seq_cu, non_blocking=True)
            ptr.copy_(dplan.packed_traj, non_blocking=True)
            seq = (gsc, ptr)
        ready = torch.cuda.Event()
        ready.record()
        gather, _ = K.fill_gather(ro.traj_bounds, dplan, int(sum(mb_tokens)))
        self.launches += 2
        return items, (dplan, gather, mb_offsets, lens, gcu, st, ng, ready, seq)

    def _plan_finish(self, pending) -> StepPlan:
        items, rest = pending
        if rest is None:
            return StepPlan(items, None, None, None, None)
        dplan, gather, mb_offsets, lens, gcu, st, ng, ready, seq = rest
        ready.synchronize()
        status, n_groups, group_cu = st.numpy().copy(), ng.numpy().astype(np.int64), \
            gcu.numpy().copy()
        bad = np.nonzero(status)[0]
        if len(bad):
            m = int(bad[0])
            raise _status_error(int(status[m]), [int(lens[k]) for k in items[m]],
                                self.cfg.micro_token_budget)
        sp = StepPlan(items, dplan, gather, group_cu, n_groups)
        sp.micro, sp.mine, sp.load = shard_micro_batches(group_cu, n_groups, mb_offsets,
                                                         self.world, self.rank, with_load=True)
        if seq is not None:
            sp.host_seq = (seq[0].numpy().copy(), seq[1].numpy().copy())
        self.last_plan = sp
        return sp

    def own_token_ranges(self, ro: PackedRollouts, sp: StepPlan):
        """Global token ranges of the trajectories in this rank's micro-batches, sorted and
        coalesced (consecutive trajectories merge into one copy)."""
        gsc, ptraj = sp.host_seq
        mb_off = sp.device_plan.mb_offsets
        trajs = []
        for m, groups in enumerate(sp.mine):
            base = int(mb_off[m]) + m
            for g, _, _ in groups:
                trajs.extend(ptraj[gsc[base + g]:gsc[base + g + 1]].tolist())
        trajs.sort()
        b = ro.traj_bounds_host
        ranges = []
        for k in trajs:
            lo, hi = int(b[k]), int(b[k + 1])
            if ranges and ranges[-1][1] == lo:
                ranges[-1] = (ranges[-1][0], hi)
            elif hi > lo:
                ranges.append((lo, hi))
        return ranges

    def reset_events(self) -> None:
        """Start a timed region: clear the per-kernel event lists; the pooled events are
        reused (read every elapsed_time of the previous region first)."""
        self.k1_events, self.k2_events, self.k3_events, self.k45_events = [], [], [], []
        self._ev_next = 0

    def _event(self):
        if self._ev_next == len(self._ev_pool):
            self._ev_pool.append(torch.cuda.Event(enable_timing=True))
        ev = self._ev_pool[self._ev_next]
        self._ev_next += 1
        return ev

    def _timed(self, events, fn):
        if not self.record_events:
            return fn()
        s, e = self._event(), self._event()
        s.record()
        out = fn()
        e.record()
        events.append((s, e))
        return out

    # ---- K1 (or fused K7) over this rank's micro-batches (prox, once per global batch)
    def prox_logprobs(self, ro: PackedRollouts, sp: StepPlan, logits_fn=None,
                      head_fn=None, skip_minibatches=()) -> torch.Tensor:
        # zeros: under DP each token's prox is written by exactly one rank, so a SUM
        # all-reduce (if a caller needs the full vector) reconstructs it
        prox = torch.zeros(ro.n_tokens, dtype=torch.float64, device=self.device)
        for m, groups in enumerate(sp.mine):
            if m in skip_minibatches:  # filled by K2 (prox_from_lp) instead
                continue
            for g, lo, hi in groups:
                rows = sp.gather[lo:hi]
                if head_fn is not None:  # trainer.py:128-137 with the output layer fused in
                    hidden, weight, bias = head_fn(m, g, rows)
                    self._timed(self.k1_events, lambda: K.linear_logprob_fwd(
                        hidden, weight, ro.tokens, bias=bias, row_index=rows, lp_out=prox))
                    self.k7_flops += 2 * (hi - lo) * weight.shape[0] * weight.shape[1]
                    self.launches += 2
                    continue
                logits = logits_fn("prox", m, g, rows)
                self._timed(self.k1_events, lambda: K.logprob_fwd(
                    logits, ro.tokens, row_index=rows, lp_out=prox, with_entropy=False,
                    algo=self.cfg.algo))
                self.k1_bytes += (hi - lo) * (logits.shape[1] * logits.element_size() + 16)
                self.launches += 1
        return prox

    # ---- full step
    def run(self, ro, logits_fn, backward_fn=None, update_fn=None,
            current_version: int = 0, dlogits_fn=None, prox_head_fn=None) -> StepResult:
        """``ro`` is a device-resident PackedRollouts, or a HostRollouts (pinned host
        arrays): then the trajectory-level arrays are uploaded whole and the per-token
        arrays only for the trajectories this rank trains on (``self.h2d_bytes``)."""
        c = self.cfg
        host = None
        if isinstance(ro, HostRollouts):
            host = ro
            ro = PackedRollouts.from_host_meta(host, self.device)
            self.h2d_bytes = sum(t.numel() * t.element_size() for t in (
                host.traj_bounds, host.rewards, host.group_ids, host.values) if t is not None)
        # K4 first: the plan's one host read waits for K4 only; K5 and K3 run
        # behind it while the host deals the micro-batches and launches the prox pass
        pending = self._timed(self.k45_events,
                              lambda: self._plan_launch(ro, with_seq=host is not None))  # 300-315
        adv = self._timed(self.k3_events, lambda: self.advantages(ro))  # trainer.py:296
        sp = self._plan_finish(pending)
        if host is not None and sp.device_plan is not None:
            self.h2d_bytes += ro.upload_token_ranges(host, self.own_token_ranges(ro, sp))
        decoupled = c.objective == "decoupled"
        M = len(sp.items)
        fuse0 = c.fuse_first_prox and decoupled and M > 0
        prox = self.prox_logprobs(ro, sp, logits_fn, prox_head_fn,       # 295 (before any update)
                                  skip_minibatches=(0,) if fuse0 else ())
        self.last_prox = prox
        mstats = torch.zeros((max(M, 1), K._lib.N_STATS), dtype=torch.float64, device=self.device)
        micro_count = 0
        pending_reduce = []
        for m in range(M):
            st = mstats[m]
            for g, lo, hi in sp.mine[m]:
                rows = sp.gather[lo:hi]
                logits = logits_fn("train", m, g, rows)
                dl_buf = dlogits_fn(m, g, logits) if dlogits_fn else None
                first = fuse0 and m == 0
                dl, _ = self._timed(self.k2_events, lambda: K.ppo_fwd_bwd(
                    logits, ro.tokens, ro.behav, prox, adv, clip_eps=c.clip_eps,
                    decoupled=decoupled, versions=ro.versions, current_version=current_version,
                    eta_mask=c.eta_mask, behav_weight_cap=c.behav_weight_cap, row_index=rows,
                    dlogits=dl_buf, stats=st, algo=c.algo, prox_from_lp=first,
                    lp_out=prox if first else None))
                self.k2_bytes += (hi - lo) * (2 * logits.shape[1] * logits.element_size() + 52)
                self.launches += 1
                if backward_fn is not None:
                    backward_fn(m, g, dl)
            micro_count += int(sp.n_groups[m])
            if self.world > 1:
                # the one collective; only the parameter update needs its result (its n_valid
                # normaliser, trainer.py:329), so without one the next minibatch's kernels
                # do not wait for it
                work = dist.all_reduce(st, group=self.group, async_op=True)
                if update_fn is not None:
                    work.wait()
                else:
                    pending_reduce.append(work)
            if update_fn is not None:
                update_fn(m, st)                                # 329-331
        for work in pending_reduce:
            work.wait()
        s = mstats[:M].cpu().numpy() if M else np.zeros((0, 8))
        tot = s.sum(axis=0) if M else np.zeros(8)
        d = max(int(tot[1]), 1)
        return StepResult(loss=-float(tot[0]) / d, clip_fraction=float(tot[2]) / d,
                          mean_ratio=float(tot[3]) / d, tokens=ro.n_tokens,
                          minibatch_updates=M, microbatches=micro_count,
                          excluded_tokens=int(tot[4]), masked_tokens=int(tot[5]),
                          entropy=float(tot[6]) / d, minibatch_stats=s)


def emission_logprobs(tokens: torch.Tensor, logits: torch.Tensor | None = None,
                      hidden: torch.Tensor | None = None, weight: torch.Tensor | None = None,
                      bias: torch.Tensor | None = None) -> torch.Tensor:
    """Behaviour log-probs recorded at emission (rollout.py:154-159: ``P.log_prob``
    of each sampled token under the generating params), for one decode step of a
    batch of sequences.  Either the step's logits [B, V] (K1) or the final hidden
    states [B, d] + LM head [V, d] (+ bias) (K7, no logits) are given.  Returns
    float64 [B].  ``EmissionRecorder`` keeps whole trajectories (tokens, log-probs,
    versions) on the device."""
    if (logits is None) == (hidden is None):
        raise ValueError("pass exactly one of logits or hidden (+ weight)")
    if logits is not None:
        lp, _ = K.logprob_fwd(logits, tokens, with_entropy=False)
        return lp
    if weight is None:
        raise ValueError("hidden needs the LM-head weight")
    lp, _ = K.linear_logprob_fwd(hidden, weight, tokens, bias=bias)
    return lp


class EmissionRecorder:
    """Device-resident provenance record of live sequences: RolloutWorker.step
    (rollout.py:140-165) appends, per emitted token, the token, its behaviour
    log-prob ``P.log_prob(params, features, token)`` and ``params.version`` to the
    sequence's Trajectory (``tokens``, ``behavior_logprobs``, ``versions``).

    ``step(slots, tokens, version, logits=... | hidden=..., weight=...)`` records one
    decode step of len(slots) sequences in 2 launches (areal_emission_append, then K1
    or K7 writing the log-probs in place through the row map), with no host sync; the
    version lives on the device (``set_version``), so with version=None a step can be
    captured once in a CUDA graph and replayed.
    ``trajectory(slot)`` returns the three lists' arrays for that slot (one D2H copy),
    ``release(slot)`` empties it for the next request.  Slots in one step must be
    distinct; overflow (more than ``max_len`` tokens) or a bad slot is reported by
    ``check()`` / ``trajectory()`` as the reference's worker would refuse the step.
    """

    def __init__(self, n_slots: int, max_len: int, device=None):
        if n_slots < 1 or max_len < 1:
            raise ValueError("n_slots and max_len must be >= 1")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device, self.n_slots, self.max_len = dev, int(n_slots), int(max_len)
        n = self.n_slots * self.max_len + 1  # + the sink entry
        self.tokens = torch.zeros(n, dtype=torch.int64, device=dev)
        self.versions = torch.zeros(n, dtype=torch.int32, device=dev)
        self.logprobs = torch.zeros(n, dtype=torch.float64, device=dev)
        self.lengths = torch.zeros(self.n_slots, dtype=torch.int32, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.version = torch.zeros(1, dtype=torch.int32, device=dev)  # generating params' version
        self._version_host = 0
        self._rows = torch.empty(0, dtype=torch.int32, device=dev)
        self.launches = 0

    def set_version(self, version: int) -> None:
        """update_weights (rollout.py:180-208): later emissions record ``version``."""
        if int(version) != self._version_host:
            self.version.fill_(int(version))
            self._version_host = int(version)

    def step(self, slots: torch.Tensor, tokens: torch.Tensor, version: int | None = None, *,
             logits: torch.Tensor | None = None, hidden: torch.Tensor | None = None,
             weight: torch.Tensor | None = None, bias: torch.Tensor | None = None) -> None:
        if (logits is None) == (hidden is None):
            raise ValueError("pass exactly one of logits or hidden (+ weight)")
        B = slots.numel()
        if tokens.numel() != B:
            raise ValueError("one sampled token per slot")
        if slots.dtype != torch.int32 or tokens.dtype != torch.int64:
            raise TypeError("slots int32, tokens int64")
        if self._rows.numel() < B:
            self._rows = torch.empty(B, dtype=torch.int32, device=self.device)
        rows = self._rows[:B]
        if version is not None:
            self.set_version(version)
        lib = K._lib.load()
        K.check(lib.areal_emission_append(
            K._ptr(slots), K._ptr(tokens), B, K._ptr(self.version), self.n_slots, self.max_len,
            K._ptr(self.lengths), K._ptr(self.tokens), K._ptr(self.versions), K._ptr(rows),
            K._ptr(self.status), K._stream()), "areal_emission_append")
        if logits is not None:
            K.logprob_fwd(logits, self.tokens, row_index=rows, lp_out=self.logprobs,
                          with_entropy=False)
            self.launches += 2
        else:
            if weight is None:
                raise ValueError("hidden needs the LM-head weight")
            K.linear_logprob_fwd(hidden, weight, self.tokens, bias=bias, row_index=rows,
                                 lp_out=self.logprobs)
            self.launches += 3

    def check(self) -> None:
        st = int(self.status.item())
        if st != 0:
            raise K._lib.ArealError(st, "EmissionRecorder.step")

    def trajectory(self, slot: int):
        """(tokens int64, behavior_logprobs float64, versions int32) of ``slot``."""
        self.check()
        n = int(self.lengths[slot].item())
        lo = slot * self.max_len
        return (self.tokens[lo:lo + n].cpu().numpy(), self.logprobs[lo:lo + n].cpu().numpy(),
                self.versions[lo:lo + n].cpu().numpy())

    def release(self, slot: int) -> None:
        self.lengths[slot] = 0


def linear_ppo_fwd_bwd(hidden: torch.Tensor, weight: torch.Tensor, tokens: torch.Tensor,
                       behav: torch.Tensor, prox: torch.Tensor, adv: torch.Tensor, *,
                       bias: torch.Tensor | None = None, row_index: torch.Tensor | None = None,
                       clip_eps: float = 0.2, decoupled: bool = True, versions=None,
                       current_version: int = 0, eta_mask: int = -1,
                       behav_weight_cap: float = 0.0, grad_scale: float = 1.0,
                       chunk_tokens: int = 8192, stats: torch.Tensor | None = None,
                       grad_weight: torch.Tensor | None = None,
                       grad_bias: torch.Tensor | None = None, algo: str = "auto",
                       prox_from_lp: bool = False, lp_out: torch.Tensor | None = None):
    """Decoupled-PPO loss + backward THROUGH the LM head on the tensor cores, the
    micro-batch's rows in chunks of ``chunk_tokens`` (only one chunk's [rows, V] logits
    exist at a time).

    _surrogate_terms (trainer.py:150-195) including its model GEMMs, per chunk:
    logits = h W^T + b (areal_lm_head_gemm LOGITS, tcgen05, fp32 accumulate, bf16 out)
    -> K2 in place -> dlogits dL, then one grouped launch (areal_lm_head_backward):
    dH = dL W (trainer.py:183's residual^T features, transposed) and dW += dL^T h (fp32,
    accumulated across chunks in the epilogue), and db += sum(dL) (areal_colsum,
    trainer.py:184).  Four launches per chunk (3 without a bias), all of them this
    library's kernels.  Peak extra memory is
    chunk_tokens x V x 2 bytes (2.5 GB at 8,192 x 151,936).

    ``prox_from_lp`` / ``lp_out``: as in kernels.ppo_fwd_bwd (first minibatch of a step).

    Returns (grad_hidden [T, d] in hidden's dtype, grad_weight [V, d] fp32,
    grad_bias [V] fp32 or None, stats float64[8]); all gradients are of
    grad_scale * (-sum objective), like K2's dlogits.
    """
    if hidden.dim() != 2 or weight.dim() != 2 or hidden.shape[1] != weight.shape[1]:
        raise ValueError("hidden [T, d] and weight [V, d] must share d")
    if hidden.dtype != weight.dtype or hidden.dtype not in (torch.bfloat16, torch.float16):
        raise TypeError("hidden and weight must both be bfloat16 or float16")
    dev = hidden.device
    T, d = hidden.shape
    V = weight.shape[0]
    if stats is None:
        stats = torch.zeros(K._lib.N_STATS, dtype=torch.float64, device=dev)
    fresh_w = grad_weight is None
    if fresh_w:
        grad_weight = torch.empty(V, d, dtype=torch.float32, device=dev)
    fresh_b = bias is not None and grad_bias is None
    if fresh_b:
        grad_bias = torch.empty(V, dtype=torch.float32, device=dev)
    grad_hidden = torch.empty_like(hidden)
    bias32 = bias.float().contiguous() if bias is not None else None
    chunk = max(1, int(chunk_tokens))
    ldv = (V + 7) // 8 * 8  # 16-byte row stride for the tensor maps
    buf = torch.empty((min(chunk, max(T, 1)), ldv), dtype=hidden.dtype, device=dev)
    # one accumulate flag drives grad_w and grad_b: the first chunk may overwrite only
    # when both are fresh; otherwise fresh ones start from zero
    acc0 = not fresh_w or (grad_bias is not None and not fresh_b)
    if (acc0 or T == 0) and fresh_w:
        grad_weight.zero_()
    if (acc0 or T == 0) and fresh_b:
        grad_bias.zero_()
    for lo in range(0, T, chunk):
        hi = min(T, lo + chunk)
        h = hidden[lo:hi]
        lg = buf[: hi - lo, :V]
        K.lm_head_gemm("logits", h, weight, lg, bias=bias32)                    # trainer.py:163
        ri = row_index[lo:hi] if row_index is not None else \
            torch.arange(lo, hi, dtype=torch.int32, device=dev)
        K.ppo_fwd_bwd(lg, tokens, behav, prox, adv, clip_eps=clip_eps, decoupled=decoupled,
                      versions=versions, current_version=current_version, eta_mask=eta_mask,
                      behav_weight_cap=behav_weight_cap, grad_scale=grad_scale, row_index=ri,
                      dlogits=lg, stats=stats, algo=algo, prox_from_lp=prox_from_lp,
                      lp_out=lp_out)                                              # 164-182
        # dH = dL W, dW (+)= dL^T h (trainer.py:183-184): one grouped launch; db (+)= sum dL
        # (184) by the column-sum kernel (measured faster than summing inside the GEMM,
        # DESIGN.md §8.1)
        acc = acc0 or lo > 0
        K.lm_head_backward(lg, h, weight, grad_hidden[lo:hi], grad_weight, None,
                           accumulate=acc, with_bias=False)
        if grad_bias is not None:
            K.colsum(lg, grad_bias, accumulate=acc)
    return grad_hidden, grad_weight, grad_bias, stats
