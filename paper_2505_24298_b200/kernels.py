"""Torch-tensor front end of the C-ABI kernels (K1-K5).

Every function takes CUDA tensors, validates dtype / device / contiguity,
passes raw pointers plus ``torch.cuda.current_stream()`` to libareal_b200.so
and returns CUDA tensors.  Launches are asynchronous; nothing here
synchronises except ``MicrobatchPlan``-style host reads done by callers.
"""
from __future__ import annotations

import contextlib
import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import AdvParams, PpoParams, check

STAT_NAMES = ("objective_sum", "n_valid", "n_clipped", "ratio_sum", "n_excluded", "n_masked",
              "entropy_sum", "n_tokens")
ADV_MODES = {"reference": 0, "gae": 1}
NORMS = {"none": 0, "global": 1, "group": 2, "group_token": 2, "group_sequence": 3}

_WORKSPACES: dict = {}
_STAGES: dict = {}


class _HostStage:
    """Reusable pinned host buffer for small per-step host->device inputs: several
    arrays go over in ONE async copy (pageable ``.to(dev)`` copies stage through a
    driver bounce buffer and block the host).  An event guards reuse until the
    previous copy has executed."""

    def __init__(self):
        self.buf = None
        self.event = None

    def upload(self, arrays, device):
        offs, n = [], 0
        for a in arrays:
            offs.append(n)
            n += (a.nbytes + 15) // 16 * 16
        if self.event is not None:
            self.event.synchronize()
        if self.buf is None or self.buf.numel() < n:
            self.buf = torch.empty(max(n, 4096) * 2, dtype=torch.uint8).pin_memory()
        host = self.buf.numpy()
        for a, o in zip(arrays, offs):
            host[o:o + a.nbytes] = a.reshape(-1).view(np.uint8)
        dev = torch.empty(max(n, 16), dtype=torch.uint8, device=device)
        dev[:n].copy_(self.buf[:n], non_blocking=True)
        self.event = torch.cuda.Event()
        self.event.record()
        return [dev[o:o + a.nbytes].view(torch.from_numpy(a[:0]).dtype)
                for a, o in zip(arrays, offs)]


def set_tuning(knob: str, value: int) -> int:
    """Override one kernel-selection rule (areal_set_tuning; include/areal_b200.h
    areal_tune_t).  ``value`` -1 restores the shipped rule.  Returns the previous value."""
    lib = _lib.load()
    if knob not in _lib.TUNE_KNOBS:
        raise ValueError(f"unknown tuning knob {knob!r}; known: {sorted(_lib.TUNE_KNOBS)}")
    k = _lib.TUNE_KNOBS[knob]
    old = ctypes.c_int64()
    check(lib.areal_get_tuning(k, ctypes.byref(old)), "areal_get_tuning")
    check(lib.areal_set_tuning(k, int(value)), f"areal_set_tuning({knob}={value})")
    return int(old.value)


@contextlib.contextmanager
def tuning(**knobs):
    """``with tuning(k2_tmem=0): ...`` — scoped kernel-selection overrides (A/B, tests)."""
    prev = {}
    try:
        for k, v in knobs.items():
            prev[k] = set_tuning(k, v)
        yield
    finally:
        for k, v in prev.items():
            set_tuning(k, v)


def _upload(arrays, device):
    key = (device.index, torch.cuda.current_stream(device).cuda_stream)
    st = _STAGES.get(key)
    if st is None:
        st = _STAGES[key] = _HostStage()
    return st.upload([np.ascontiguousarray(a) for a in arrays], device)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def workspace(device=None) -> torch.Tensor:
    """Zero-initialised per-(device, stream) workspace (AREAL_WORKSPACE_BYTES)."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    key = (dev.index, torch.cuda.current_stream(dev).cuda_stream)
    ws = _WORKSPACES.get(key)
    if ws is None:
        ws = torch.zeros(_lib.WORKSPACE_BYTES, dtype=torch.uint8, device=dev)
        _WORKSPACES[key] = ws
    return ws


def _need(t, name, dtype, device=None, numel=None):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    if numel is not None and t.numel() < numel:
        raise ValueError(f"{name} has {t.numel()} elements, needs >= {numel}")
    return t


def _logits_info(logits):
    if not isinstance(logits, torch.Tensor) or not logits.is_cuda or logits.dim() != 2:
        raise ValueError("logits must be a 2-D CUDA tensor [rows, vocab]")
    if logits.dtype not in _lib.DTYPE_CODES:
        raise TypeError(f"unsupported logits dtype {logits.dtype}")
    if logits.stride(1) != 1:
        raise ValueError("logits rows must be contiguous (stride(1) == 1)")
    n, v = logits.shape
    ld = logits.stride(0) if n > 1 else v
    return n, v, ld, _lib.DTYPE_CODES[logits.dtype]


# ---------------------------------------------------------------- K1
def logprob_fwd(logits: torch.Tensor, tokens: torch.Tensor, row_index: torch.Tensor | None = None,
                lp_out: torch.Tensor | None = None, entropy_out: torch.Tensor | None = None,
                with_entropy: bool = True, algo: str = "auto"):
    """Per-token log-prob (and entropy) of ``tokens`` under ``logits`` (K1).

    Row r of ``logits`` belongs to global token ``row_index[r]`` (identity if
    None); ``tokens``/``lp_out``/``entropy_out`` are indexed by global token.
    Replaces trainer.recompute_prox_logprobs -> policy.batch_token_log_probs.
    """
    lib = _lib.load()
    n, v, ld, dt = _logits_info(logits)
    dev = logits.device
    n_glob = tokens.numel()
    _need(tokens, "tokens", torch.int64, dev)
    if row_index is not None:
        _need(row_index, "row_index", torch.int32, dev, n)
    elif n_glob < n:
        raise ValueError("tokens shorter than the number of logits rows")
    if lp_out is None:
        lp_out = torch.empty(n_glob, dtype=torch.float64, device=dev)
    _need(lp_out, "lp_out", torch.float64, dev, n_glob)
    if with_entropy and entropy_out is None:
        entropy_out = torch.empty(n_glob, dtype=torch.float64, device=dev)
    if entropy_out is not None:
        _need(entropy_out, "entropy_out", torch.float64, dev, n_glob)
    ws = workspace(dev)
    check(lib.areal_logprob_fwd(_ptr(logits), ld, dt, n, v, _ptr(tokens), _ptr(row_index),
                                _ptr(lp_out), _ptr(entropy_out), _lib.ALGO_CODES[algo],
                                _ptr(ws), ws.numel(), _stream()), "areal_logprob_fwd")
    return lp_out, entropy_out


# ---------------------------------------------------------------- K2
def ppo_fwd_bwd(logits, tokens, behav, prox, adv, *, clip_eps=0.2, decoupled=True,
                versions=None, current_version=0, eta_mask=-1, behav_weight_cap=0.0,
                grad_scale=1.0, row_index=None, dlogits=None, lp_out=None, entropy_out=None,
                stats=None, algo="auto", prox_from_lp=False):
    """Fused decoupled/naive PPO loss + backward (K2).

    Returns ``(dlogits, stats)``: dlogits = grad_scale * coef * (softmax - onehot)
    (the gradient of -sum(objective) scaled), stats a float64[8] device tensor
    accumulated with += (order: ``STAT_NAMES``).  ``dlogits`` may be ``logits``
    itself (in-place backward).  Per-token arrays are float64 indexed by global
    token (see ``row_index``).  Replaces trainer._surrogate_terms.

    ``prox_from_lp=True`` (first minibatch of a step, whose params are the ones prox
    is defined under, trainer.py:295): prox := the lp this kernel computes (``prox``
    may be None; pass ``lp_out`` = the prox vector to record it), so the prox pass
    and the loss share one read of the logits.
    """
    lib = _lib.load()
    n, v, ld, dt = _logits_info(logits)
    dev = logits.device
    n_glob = tokens.numel()
    _need(tokens, "tokens", torch.int64, dev)
    _need(behav, "behav", torch.float64, dev, n_glob)
    _need(adv, "adv", torch.float64, dev, n_glob)
    if decoupled and not prox_from_lp:
        _need(prox, "prox", torch.float64, dev, n_glob)
    if versions is not None:
        _need(versions, "versions", torch.int32, dev, n_glob)
    if row_index is not None:
        _need(row_index, "row_index", torch.int32, dev, n)
    elif n_glob < n:
        raise ValueError("tokens shorter than the number of logits rows")
    if dlogits is None:
        dlogits = torch.empty_like(logits)
    if dlogits.dtype != logits.dtype or dlogits.shape != logits.shape or dlogits.stride(1) != 1:
        raise ValueError("dlogits must match logits in dtype/shape with unit column stride")
    ld_out = dlogits.stride(0) if n > 1 else v
    if stats is None:
        stats = torch.zeros(_lib.N_STATS, dtype=torch.float64, device=dev)
    _need(stats, "stats", torch.float64, dev, _lib.N_STATS)
    for name, t in (("lp_out", lp_out), ("entropy_out", entropy_out)):
        if t is not None:
            _need(t, name, torch.float64, dev, n_glob)
    p = PpoParams(float(clip_eps), float(behav_weight_cap), float(grad_scale), int(bool(decoupled)),
                  int(eta_mask), int(current_version), _lib.ALGO_CODES[algo], int(bool(prox_from_lp)))
    ws = workspace(dev)
    check(lib.areal_ppo_fwd_bwd(_ptr(logits), ld, _ptr(dlogits), ld_out, dt, n, v, _ptr(tokens),
                                _ptr(behav), _ptr(prox if decoupled and not prox_from_lp else None),
                                _ptr(adv),
                                _ptr(versions), _ptr(row_index), ctypes.byref(p), _ptr(lp_out),
                                _ptr(entropy_out), _ptr(stats), _ptr(ws), ws.numel(), _stream()),
          "areal_ppo_fwd_bwd")
    return dlogits, stats


# ---------------------------------------------------------------- K3
def advantages(rewards, traj_bounds, n_tokens: int, *, mode="reference", gamma=1.0, lam=1.0,
               values=None, norm="global", group_ids=None, n_groups=None, eps=0.0, out=None,
               returns_out=None, norm_stats=None):
    """Per-token advantages (K3).  ``mode='reference'`` + ``norm='global'`` is
    bit-identical to trainer.compute_advantages."""
    lib = _lib.load()
    dev = rewards.device
    n_traj = rewards.numel()
    _need(rewards, "rewards", torch.float64, dev)
    _need(traj_bounds, "traj_bounds", torch.int64, dev, n_traj + 1)
    if values is not None:
        _need(values, "values", torch.float64, dev, n_tokens)
    g = None
    if norm in ("group", "group_token", "group_sequence"):
        if group_ids is None:
            raise ValueError("group normalisation needs group_ids")
        g = _need(group_ids, "group_ids", torch.int32, dev, n_traj)
        if n_groups is None:
            n_groups = int(group_ids.max().item()) + 1 if n_traj else 0
    if out is None:
        out = torch.empty(n_tokens, dtype=torch.float64, device=dev)
    _need(out, "out", torch.float64, dev, n_tokens)
    p = AdvParams(float(gamma), float(lam), float(eps), ADV_MODES[mode], NORMS[norm])
    ws = workspace(dev)
    check(lib.areal_advantages(_ptr(rewards), _ptr(traj_bounds), n_traj, int(n_tokens),
                               _ptr(values), _ptr(g), int(n_groups or 0), ctypes.byref(p),
                               _ptr(out), _ptr(returns_out), _ptr(norm_stats), _ptr(ws),
                               ws.numel(), _stream()), "areal_advantages")
    return out


# ---------------------------------------------------------------- K4 + K5
@dataclass
class DevicePlan:
    """Device outputs of areal_plan_microbatches (+ the host inputs that sized them)."""
    group_of: torch.Tensor
    slot_of: torch.Tensor
    n_groups: torch.Tensor
    group_cu: torch.Tensor
    group_seq_cu: torch.Tensor
    packed_traj: torch.Tensor
    seq_cu: torch.Tensor
    status: torch.Tensor
    mb_offsets: np.ndarray
    mb_token_start: np.ndarray
    n_packed_tokens: int


def plan_microbatches(traj_bounds: torch.Tensor, item_traj: torch.Tensor, mb_offsets,
                      mb_token_start, capacity: int, min_groups: int) -> DevicePlan:
    """Dynamic micro-batch allocation for every minibatch at once (K4 + packing plan).

    ``item_traj`` (device int32, or a host int array: then it travels with the
    offsets in one pinned async copy) lists the non-empty trajectories of each
    minibatch back to back; ``mb_offsets`` (host, M+1) delimits them;
    ``mb_token_start`` (host, M) is each minibatch's offset in the packed stream.
    """
    lib = _lib.load()
    dev = traj_bounds.device
    _need(traj_bounds, "traj_bounds", torch.int64, dev)
    host_items = not isinstance(item_traj, torch.Tensor)
    if not host_items:
        _need(item_traj, "item_traj", torch.int32, dev)
    mb_offsets = np.asarray(mb_offsets, dtype=np.int32)
    mb_token_start = np.asarray(mb_token_start, dtype=np.int64)
    M = len(mb_offsets) - 1
    n_items = int(mb_offsets[-1]) if M > 0 else 0
    max_items = int(np.max(np.diff(mb_offsets))) if M > 0 else 0
    if max_items > _lib.MAX_ITEMS_PER_MINIBATCH:
        raise ValueError(f"{max_items} sequences in one minibatch exceeds "
                         f"{_lib.MAX_ITEMS_PER_MINIBATCH}")
    i32 = dict(dtype=torch.int32, device=dev)
    if host_items:  # all three host inputs in one pinned async copy
        item_traj, mb_off_d, mb_tok_d = _upload(
            [np.asarray(item_traj, dtype=np.int32), mb_offsets, mb_token_start], dev)
        if item_traj.numel() < n_items:
            raise ValueError(f"item_traj has {item_traj.numel()} entries, needs {n_items}")
    else:
        mb_off_d, mb_tok_d = _upload([mb_offsets, mb_token_start], dev)
    # two allocations sliced into the plan's outputs (every entry is written by K4,
    # status included: no memset)
    m1 = max(M, 1)
    b32 = torch.empty(4 * n_items + M + 2 * m1, **i32)
    b64 = torch.empty(2 * n_items + M + 1, dtype=torch.int64, device=dev)
    o = np.cumsum([0, n_items, n_items, n_items, n_items + M, m1, m1])
    plan = DevicePlan(
        group_of=b32[o[0]:o[1]], slot_of=b32[o[1]:o[2]], packed_traj=b32[o[2]:o[3]],
        group_seq_cu=b32[o[3]:o[4]], n_groups=b32[o[4]:o[5]], status=b32[o[5]:o[6]],
        group_cu=b64[:n_items + M], seq_cu=b64[n_items + M:],
        mb_offsets=mb_offsets, mb_token_start=mb_token_start, n_packed_tokens=0)
    if M == 0:  # nothing for K4 to write
        b32.zero_()
        b64.zero_()
    check(lib.areal_plan_microbatches(
        _ptr(traj_bounds), _ptr(item_traj), _ptr(mb_off_d), _ptr(mb_tok_d), M, n_items, max_items,
        int(capacity), int(min_groups), _ptr(plan.group_of), _ptr(plan.slot_of),
        _ptr(plan.n_groups), _ptr(plan.group_cu), _ptr(plan.group_seq_cu),
        _ptr(plan.packed_traj), _ptr(plan.seq_cu), _ptr(plan.status), _stream()),
        "areal_plan_microbatches")
    plan._keepalive = (item_traj, mb_off_d, mb_tok_d)  # host->device copies are async
    return plan


def fill_gather(traj_bounds, plan: DevicePlan, n_packed_tokens: int, with_seq_id=False):
    """Packed gather index (K5): gather[p] = global token index at packed position p."""
    lib = _lib.load()
    dev = traj_bounds.device
    gather = torch.empty(n_packed_tokens, dtype=torch.int32, device=dev)
    seq_id = torch.empty(n_packed_tokens, dtype=torch.int32, device=dev) if with_seq_id else None
    n_items = plan.packed_traj.numel()
    check(lib.areal_fill_gather(_ptr(traj_bounds), _ptr(plan.packed_traj), _ptr(plan.seq_cu),
                                n_items, int(n_packed_tokens), _ptr(gather), _ptr(seq_id),
                                _stream()), "areal_fill_gather")
    return gather, seq_id


# ---------------------------------------------------------------- K6
def adam_step(params, grads, exp_avgs, exp_avg_sqs, *, step: int, lr: float, beta1: float,
              beta2: float, eps: float, weight_decay: float, clip_norm: float,
              grad_scale: float = 1.0, exact_norm: bool | None = None, norm_out=None,
              grad_scale_divisor: torch.Tensor | None = None):
    """Fused global-norm clip + Adam over a list of tensors (K6), in place.

    Mirrors policy.apply_update (policy.py:225-258) applied to ``grad * grad_scale``
    (trainer.py:329-330 passes grad_scale = -1/n).  ``step`` is the optimizer step
    AFTER this update (the reference's ``opt.step += 1``).  Returns a device float64
    tensor [global_norm, n_nonfinite]; when n_nonfinite > 0 nothing was updated and
    the caller raises NonFiniteGradientError.  ``exact_norm`` (default: fp64 params)
    replays numpy's pairwise sums so the update is bit-identical to the reference.
    ``grad_scale_divisor`` (a 1-element float64 CUDA tensor, e.g. ``stats[1:2]`` of K2 after
    the all-reduce) makes the scale ``grad_scale / max(divisor, 1)`` on the device, so
    the loss -> optimizer hand-off needs no host synchronisation.
    """
    lib = _lib.load()
    n = len(params)
    if not (n == len(grads) == len(exp_avgs) == len(exp_avg_sqs)):
        raise ValueError("params, grads, exp_avgs, exp_avg_sqs must have the same length")
    if n > _lib.ADAM_MAX_TENSORS:
        raise ValueError(f"at most {_lib.ADAM_MAX_TENSORS} tensors per adam_step call")
    if n == 0:
        raise ValueError("adam_step needs at least one tensor")
    dev = params[0].device
    pdt = params[0].dtype
    gdt = grads[0].dtype
    if pdt not in (torch.float64, torch.float32):
        raise TypeError(f"params must be float64 or float32, got {pdt}")
    if (pdt == torch.float64) != (gdt == torch.float64) or gdt not in _lib.DTYPE_CODES:
        raise TypeError(f"grads of dtype {gdt} cannot update {pdt} params "
                        "(float64 with float64; float32/bfloat16/float16 with float32)")
    arr = (_lib.AdamTensor * n)()
    for k in range(n):
        p, g, m, v = params[k], grads[k], exp_avgs[k], exp_avg_sqs[k]
        _need(p, f"params[{k}]", pdt, dev)
        _need(g, f"grads[{k}]", gdt, dev)
        _need(m, f"exp_avgs[{k}]", pdt, dev)
        _need(v, f"exp_avg_sqs[{k}]", pdt, dev)
        if not (p.numel() == g.numel() == m.numel() == v.numel()):
            raise ValueError(f"tensor {k}: param/grad/moment sizes differ")
        arr[k] = _lib.AdamTensor(p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), p.numel())
    if exact_norm is None:
        exact_norm = pdt == torch.float64 and gdt == torch.float64
    # scalars exactly as the reference computes them in Python (policy.py:245-250)
    prm = _lib.AdamParams(float(lr), float(beta1), float(beta2), float(eps), float(weight_decay),
                          float(clip_norm), 1 - beta1, 1 - beta2, 1 - beta1 ** step,
                          1 - beta2 ** step, float(grad_scale), int(bool(exact_norm)),
                          _ptr(grad_scale_divisor))
    if grad_scale_divisor is not None:
        _need(grad_scale_divisor, "grad_scale_divisor", torch.float64, dev, 1)
    if norm_out is None:
        norm_out = torch.empty(2, dtype=torch.float64, device=dev)
    _need(norm_out, "norm_out", torch.float64, dev, 2)
    ws = workspace(dev)
    check(lib.areal_adam_step(arr, n, _lib.DTYPE_CODES[pdt], _lib.DTYPE_CODES[gdt],
                              ctypes.byref(prm), _ptr(norm_out), _ptr(ws), ws.numel(), _stream()),
          "areal_adam_step")
    return norm_out


# ---------------------------------------------------------------- K7
_SCRATCH: dict = {}


def _scratch(dev, nbytes):
    key = (dev.index, torch.cuda.current_stream(dev).cuda_stream)
    buf = _SCRATCH.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=dev)
        _SCRATCH[key] = buf
    return buf


def linear_logprob_fwd(hidden: torch.Tensor, weight: torch.Tensor, tokens: torch.Tensor,
                       bias: torch.Tensor | None = None, row_index: torch.Tensor | None = None,
                       lp_out=None, entropy_out=None, with_entropy: bool = False,
                       cta_group: int = 0):
    """Fused LM head + log-softmax-gather (K7, tcgen05): lp[idx] = log_softmax(h W^T + b)[tok].

    ``hidden`` [n, d] and ``weight`` [V, d] are bf16/fp16 (row-contiguous, d % 64 == 0),
    ``bias`` fp32 [V] or None.  Mirrors recompute_prox_logprobs / batch_token_log_probs
    (trainer.py:128-137, policy.py:133-163) with the output layer fused in: the [n, V]
    logits are never materialised.  Returns (lp, entropy-or-None), float64, indexed like K1.
    """
    lib = _lib.load()
    if hidden.dim() != 2 or weight.dim() != 2 or hidden.shape[1] != weight.shape[1]:
        raise ValueError("hidden [n, d] and weight [V, d] must share d")
    if hidden.dtype not in (torch.bfloat16, torch.float16) or weight.dtype != hidden.dtype:
        raise TypeError("hidden and weight must both be bfloat16 or float16")
    if hidden.stride(1) != 1 or weight.stride(1) != 1:
        raise ValueError("hidden / weight rows must be contiguous")
    dev = hidden.device
    n, d = hidden.shape
    V = weight.shape[0]
    if bias is not None:
        _need(bias, "bias", torch.float32, dev, V)
    _need(tokens, "tokens", torch.int64, dev)
    if row_index is not None:
        _need(row_index, "row_index", torch.int32, dev, n)
    n_idx = tokens.numel() if row_index is not None else n
    if lp_out is None:
        lp_out = torch.empty(n_idx, dtype=torch.float64, device=dev)
    if with_entropy and entropy_out is None:
        entropy_out = torch.empty(n_idx, dtype=torch.float64, device=dev)
    nbytes = int(lib.areal_linear_logprob_scratch_bytes(n, V))
    scratch = _scratch(dev, nbytes)
    ld_h = hidden.stride(0) if n > 1 else d
    ld_w = weight.stride(0) if V > 1 else d
    check(lib.areal_linear_logprob_fwd(_ptr(hidden), ld_h, _ptr(weight), ld_w, _ptr(bias),
                                       _lib.DTYPE_CODES[hidden.dtype], n, V, d, _ptr(tokens),
                                       _ptr(row_index), _ptr(lp_out), _ptr(entropy_out),
                                       _ptr(scratch), scratch.numel(), int(cta_group), _stream()),
          "areal_linear_logprob_fwd")
    return lp_out, entropy_out


# ---------------------------------------------------------------- LM-head GEMMs (tcgen05)
def _ld(t: torch.Tensor) -> int:
    """Row stride in elements; a single row's is free, so report it 16-byte rounded."""
    return t.stride(0) if t.shape[0] > 1 else (t.shape[1] + 7) // 8 * 8


def lm_head_gemm(op: str, A: torch.Tensor, B: torch.Tensor, C: torch.Tensor | None = None, *,
                 bias: torch.Tensor | None = None, accumulate: bool = False) -> torch.Tensor:
    """The LM head's GEMMs on tcgen05 (areal_lm_head_gemm, lm_head.cu):

    ``"logits"``  C[T, V] = A[T, d] @ B[V, d]^T (+ bias[V])   (16-bit out)
    ``"dhidden"`` C[T, d] = A[T, V] @ B[V, d]                 (16-bit out)
    ``"dweight"`` C[V, d] (+)= A[T, V]^T @ B[T, d]            (fp32 out, += if accumulate)

    trainer.py:163 (logits = features W^T + b) and 183-184 (grad_w = resid^T features);
    fp32 accumulation in Tensor Memory.  Rows must be unit-stride with 16-byte aligned
    row strides."""
    lib = _lib.load()
    if op not in _lib.LMH_OPS:
        raise ValueError(f"unknown op {op!r}")
    if A.dim() != 2 or B.dim() != 2 or A.dtype != B.dtype or A.dtype not in (torch.bfloat16, torch.float16):
        raise TypeError("A and B must be 2-D bfloat16 / float16 tensors of one dtype")
    if A.device != B.device or (A.numel() and A.stride(1) != 1) or (B.numel() and B.stride(1) != 1):
        raise ValueError("A and B must be row-major (unit column stride) on one device")
    dev = A.device
    if op == "logits":
        (M, K), (N, K2) = A.shape, B.shape
        out_dtype = A.dtype
    elif op == "dhidden":
        (M, K), (K2, N) = A.shape, B.shape
        out_dtype = A.dtype
    else:
        (K, M), (K2, N) = A.shape, B.shape
        out_dtype = torch.float32
    if K != K2:
        raise ValueError(f"{op}: inner dimensions differ ({K} vs {K2})")
    if C is None:  # rows padded to 16 bytes (the kernel's vector stores)
        C = (torch.zeros if accumulate else torch.empty)((M, (N + 7) // 8 * 8), dtype=out_dtype,
                                                         device=dev)[:, :N]
    if C.shape != (M, N) or C.dtype != out_dtype or (C.numel() and C.stride(1) != 1):
        raise ValueError(f"{op}: C must be a row-major {out_dtype} [{M}, {N}] tensor")
    if bias is not None:
        if op != "logits":
            raise ValueError("bias applies to the logits GEMM only")
        _need(bias, "bias", torch.float32, dev, N)
    check(lib.areal_lm_head_gemm(_lib.LMH_OPS[op], _ptr(A), _ld(A), _ptr(B), _ld(B), _ptr(C), _ld(C),
                                 M, N, K, _ptr(bias), int(bool(accumulate)),
                                 _lib.DTYPE_CODES[A.dtype], _stream()), f"areal_lm_head_gemm({op})")
    return C


def lm_head_backward(dlogits: torch.Tensor, hidden: torch.Tensor, weight: torch.Tensor,
                     grad_hidden: torch.Tensor | None = None, grad_weight: torch.Tensor | None = None,
                     grad_bias: torch.Tensor | None = None, accumulate: bool = False, with_bias: bool = True):
    """One launch for the chunk's backward through the head (areal_lm_head_backward):
    grad_hidden = dL @ W, grad_weight (+)= dL^T @ hidden, grad_bias (+)= dL.sum(0)
    (trainer.py:183-184), grouped on tcgen05 with grad_b fused into the DWEIGHT tiles."""
    lib = _lib.load()
    for t, nm in ((dlogits, "dlogits"), (hidden, "hidden"), (weight, "weight")):
        if t.dim() != 2 or (t.numel() and t.stride(1) != 1):
            raise ValueError(f"{nm} must be a row-major 2-D tensor")
    if not (dlogits.dtype == hidden.dtype == weight.dtype) or dlogits.dtype not in (torch.bfloat16, torch.float16):
        raise TypeError("dlogits, hidden and weight must share a 16-bit dtype")
    T, V = dlogits.shape
    d = hidden.shape[1]
    if hidden.shape[0] != T or weight.shape != (V, d):
        raise ValueError("shapes: dlogits [T, V], hidden [T, d], weight [V, d]")
    dev = dlogits.device
    if grad_hidden is None:
        grad_hidden = torch.empty((T, (d + 7) // 8 * 8), dtype=hidden.dtype, device=dev)[:, :d]
    if grad_weight is None:
        grad_weight = (torch.zeros if accumulate else torch.empty)((V, (d + 3) // 4 * 4), dtype=torch.float32,
                                                                   device=dev)[:, :d]
    if with_bias and grad_bias is None:
        grad_bias = (torch.zeros if accumulate else torch.empty)(V, dtype=torch.float32, device=dev)
    if grad_bias is not None:
        _need(grad_bias, "grad_bias", torch.float32, dev, V)
    if grad_hidden.shape != (T, d) or grad_weight.shape != (V, d) or grad_weight.dtype != torch.float32:
        raise ValueError("grad_hidden [T, d] (hidden dtype) and grad_weight [V, d] fp32")
    check(lib.areal_lm_head_backward(_ptr(dlogits), _ld(dlogits) if T else V, _ptr(hidden),
                                     _ld(hidden) if T else d, _ptr(weight), _ld(weight), T, V, d,
                                     _ptr(grad_hidden), _ld(grad_hidden) if T else d, _ptr(grad_weight),
                                     _ld(grad_weight), _ptr(grad_bias), int(bool(accumulate)),
                                     _lib.DTYPE_CODES[dlogits.dtype], _stream()), "areal_lm_head_backward")
    return grad_hidden, grad_weight, grad_bias


def colsum(x: torch.Tensor, out: torch.Tensor | None = None, accumulate: bool = False) -> torch.Tensor:
    """out[c] (+)= sum_r x[r, c] in fp32, deterministic (areal_colsum): grad_b of the head
    (trainer.py:184, resid.sum over tokens)."""
    lib = _lib.load()
    if x.dim() != 2 or x.dtype not in (torch.bfloat16, torch.float16) or (x.numel() and x.stride(1) != 1):
        raise TypeError("x must be a row-major 2-D bfloat16 / float16 tensor")
    rows, cols = x.shape
    dev = x.device
    if out is None:
        out = (torch.zeros if accumulate else torch.empty)(cols, dtype=torch.float32, device=dev)
    _need(out, "out", torch.float32, dev, cols)
    scratch = _scratch(dev, int(lib.areal_colsum_scratch_bytes(rows, cols)))
    check(lib.areal_colsum(_ptr(x), _ld(x) if rows else cols, rows, cols, _lib.DTYPE_CODES[x.dtype],
                           _ptr(out), int(bool(accumulate)), _ptr(scratch), scratch.numel(), _stream()),
          "areal_colsum")
    return out
