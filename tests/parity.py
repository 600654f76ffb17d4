"""Shared parity checks: the CUDA path against the float64 oracle (trainer.py:150-195
restated in oracle/ppo_oracle.py), element by element and counter by counter.

Tolerances (north star): lp / sums 1e-5 relative for every logits dtype (the kernels
compute in fp32 from the exact rounded inputs the oracle also sees); dlogits on 100% of
the elements: fp32 within 1e-5 |d| + 1e-7 |g|, 16-bit outputs within 2e-2 |d| with no
floor relative to g except on the token's own element g*(p_tok - 1), which cancels as
p_tok -> 1 (1e-6 |g|), plus one ulp of the output format's smallest numbers (fp16
subnormals; fp32/bf16 below 2^-126 are flushed).

Counters are exact.  A decoupled ratio exp(lp - prox) that lies within the kernels'
lp error of a clip boundary 1 +- eps may legitimately flip ``take``/``clipped`` for
that token; such tokens are identified from the oracle's own ratio, counted, and
their rows are the only ones excused from the element check.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

import oracle as O

LP_RTOL = 1e-5
DL_RTOL = {"f32": 1e-5, "bf16": 2e-2, "f16": 2e-2, "f64": 1e-12}
# floor relative to |g| on every element: fp32 takes the bar 1e-5 |d| + 1e-7 |g| (the
# fp32 exponent arguments of the tiniest probabilities carry ~1e-5 relative error);
# 16-bit outputs are checked purely relatively
ALL_FLOOR = {"f32": 1e-7, "bf16": 1e-30, "f16": 1e-30, "f64": 1e-30}
# the token's own element g (p_tok - 1) cancels in fp32 as p_tok -> 1
TOK_FLOOR = {"f32": 1e-7, "bf16": 1e-6, "f16": 1e-6, "f64": 1e-14}
# absolute: one ulp of the output format's smallest numbers (fp16 subnormals are 2^-24
# apart; fp32/bf16 kernels flush below 2^-126)
OUT_FLOOR = {"f32": 2.0 ** -126, "bf16": 2.0 ** -126, "f16": 2.0 ** -24, "f64": 1e-300}
# relative lp error of the fp32 kernels that can move a ratio across a clip boundary
BOUNDARY_RTOL = 1e-5


def threads() -> int:
    return max(1, min(16, os.cpu_count() or 1))


def boundary_tokens(ref: dict, clip_eps: float, rtol: float = BOUNDARY_RTOL) -> np.ndarray:
    """Valid tokens whose oracle ratio sits within ``rtol`` of 1 - eps or 1 + eps."""
    r = np.asarray(ref["ratio"], dtype=np.float64)
    with np.errstate(invalid="ignore"):
        near = (np.abs(r - (1 + clip_eps)) <= rtol * (1 + clip_eps)) | \
               (np.abs(r - (1 - clip_eps)) <= rtol * (1 - clip_eps))
    return near & ref["valid"]


def check_counters(st, rs, n_boundary: int = 0, what: str = ""):
    """GPU stats [8] vs oracle stats [8]: n_valid, n_excluded, n_masked, n_tokens exact;
    n_clipped exact up to the identified boundary tokens."""
    st = np.asarray(st)
    rs = np.asarray(rs)
    assert st[1] == rs[1], (what, "n_valid", st[1], rs[1])
    assert st[4] == rs[4], (what, "n_excluded", st[4], rs[4])
    assert st[5] == rs[5], (what, "n_masked", st[5], rs[5])
    assert st[7] == rs[7], (what, "n_tokens", st[7], rs[7])
    assert abs(st[2] - rs[2]) <= n_boundary, (what, "n_clipped", st[2], rs[2], n_boundary)


def check_sums(st, rs, abs_obj: float, abs_ratio: float, rtol: float = LP_RTOL, what: str = ""):
    """objective_sum / ratio_sum within rtol of the sum of the magnitudes of their terms."""
    assert abs(st[0] - rs[0]) <= rtol * max(abs_obj, 1.0), (what, "objective_sum", st[0], rs[0])
    assert abs(st[3] - rs[3]) <= rtol * max(abs_ratio, 1.0), (what, "ratio_sum", st[3], rs[3])


def check_lp(got, want, rtol: float = LP_RTOL, what: str = "lp"):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    fin = np.isfinite(want)
    assert np.array_equal(np.isfinite(got), fin), (what, "finiteness differs")
    err = np.abs(got[fin] - want[fin])
    bound = rtol * (1.0 + np.abs(want[fin]))
    assert np.all(err <= bound), (what, float(np.max(err / bound)))


def dlogits_bound(want, coef, tokens, dt: str):
    """Element-wise bound for one block of rows (see module doc)."""
    g = np.abs(np.asarray(coef, dtype=np.float64))[:, None]
    bound = DL_RTOL[dt] * np.abs(want) + ALL_FLOOR[dt] * g + OUT_FLOOR[dt]
    rows = np.arange(want.shape[0])
    bound[rows, tokens] += TOK_FLOOR[dt] * g[:, 0]
    return bound


def check_dlogits(got, want, coef, tokens, dt: str, skip_rows=None, what: str = "dlogits"):
    """100% of the elements of every row (rows with a non-finite reference or an identified
    boundary token excepted) within dlogits_bound.  Returns the worst err / bound."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    ok = np.isfinite(want).all(axis=1)
    if skip_rows is not None:
        ok &= ~np.asarray(skip_rows, dtype=bool)
    if not ok.any():
        return 0.0
    w, gg = want[ok], got[ok]
    bound = dlogits_bound(w, np.asarray(coef)[ok], np.asarray(tokens)[ok], dt)
    ratio = np.abs(gg - w) / bound
    worst = float(ratio.max())
    if worst > 1.0:
        r, c = np.unravel_index(int(np.argmax(ratio)), ratio.shape)
        raise AssertionError(f"{what}: worst err/bound {worst:.3g} at row {r} col {c}: "
                             f"got {gg[r, c]!r} want {w[r, c]!r} "
                             f"({int((ratio > 1).sum())} of {ratio.size} elements out)")
    return worst


def oracle_rows(get_rows, n_rows: int, per_token: dict, *, chunk: int = 256, dt: str = "f32",
                got_rows=None, clip_eps: float = 0.2, decoupled: bool = True,
                current_version: int = 0, eta_mask: int = -1, grad_scale: float = 1.0,
                n_threads: int | None = None):
    """The oracle over a [n_rows, V] block, in row chunks on a thread pool (the float64
    numpy ufuncs release the GIL), optionally checking the kernel's dlogits chunk by chunk.

    get_rows(lo, hi) -> float64 logits rows; got_rows(lo, hi) -> kernel dlogits rows (or
    None); per_token: tokens / behav / prox / adv / versions arrays for the block's rows.
    Returns dict(stats, lp, ratio, valid, coef, boundary, abs_obj, abs_ratio, worst)."""
    keys = ("tokens", "behav", "prox", "adv", "versions")

    def work(lo):
        hi = min(n_rows, lo + chunk)
        x = get_rows(lo, hi)
        pt = {k: (None if per_token.get(k) is None else per_token[k][lo:hi]) for k in keys}
        with np.errstate(invalid="ignore", over="ignore", divide="ignore"):
            ref = O.surrogate_terms(x, pt["tokens"], pt["behav"], pt["prox"], pt["adv"],
                                    clip_eps=clip_eps, decoupled=decoupled,
                                    versions=pt["versions"], current_version=current_version,
                                    eta_mask=eta_mask, grad_scale=grad_scale,
                                    want_dlogits=got_rows is not None)
        bnd = boundary_tokens(ref, clip_eps)
        worst = 0.0
        if got_rows is not None:
            worst = check_dlogits(got_rows(lo, hi), ref["dlogits"], ref["coef"], pt["tokens"], dt,
                                  skip_rows=bnd, what=f"dlogits rows {lo}..{hi}")
        return dict(stats=ref["stats"], lp=ref["lp"], ratio=ref["ratio"], valid=ref["valid"],
                    coef=ref["coef"], boundary=bnd, worst=worst,
                    abs_obj=float(np.abs(ref["obj"]).sum()),
                    abs_ratio=float(np.abs(np.where(ref["valid"], ref["ratio"], 0.0)).sum()))

    with ThreadPoolExecutor(n_threads or threads()) as ex:
        parts = list(ex.map(work, range(0, n_rows, chunk)))
    if not parts:
        z = np.zeros(0)
        return dict(stats=np.zeros(8), lp=z, ratio=z, valid=z.astype(bool), coef=z,
                    boundary=z.astype(bool), abs_obj=0.0, abs_ratio=0.0, worst=0.0)
    cat = lambda k: np.concatenate([p[k] for p in parts])
    return dict(stats=np.sum([p["stats"] for p in parts], axis=0), lp=cat("lp"),
                ratio=cat("ratio"), valid=cat("valid"), coef=cat("coef"),
                boundary=cat("boundary"), abs_obj=sum(p["abs_obj"] for p in parts),
                abs_ratio=sum(p["abs_ratio"] for p in parts),
                worst=max(p["worst"] for p in parts))


def oracle_logprobs(get_rows, tokens, n_rows: int, chunk: int = 512, n_threads=None):
    """token_logprobs (policy.py:159-163) over a large block, chunked and threaded."""
    def work(lo):
        hi = min(n_rows, lo + chunk)
        with np.errstate(invalid="ignore", over="ignore"):
            return O.token_logprobs(get_rows(lo, hi), tokens[lo:hi])
    with ThreadPoolExecutor(n_threads or threads()) as ex:
        parts = list(ex.map(work, range(0, n_rows, chunk)))
    return np.concatenate(parts) if parts else np.zeros(0)
