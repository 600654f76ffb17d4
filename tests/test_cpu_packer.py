"""Native rollout packer (csrc/packer.c) vs build_train_batch's flattening
(trainer.py:83-111) — CPU only: tokens / behaviour log-probs / cu_seqlens /
per-token versions / rewards must be identical, errors must match."""
from types import SimpleNamespace

import numpy as np
import pytest

from paper_2505_24298_b200.build import build_packer


@pytest.fixture(scope="module")
def P():
    build_packer()
    from paper_2505_24298_b200 import _packer
    return _packer


def _trajs(rng, n, with_versions=True, empty_every=5):
    out = []
    for k in range(n):
        m = 0 if (empty_every and k % empty_every == 3) else int(rng.integers(1, 60))
        t = SimpleNamespace(trajectory_id=k, prompt=SimpleNamespace(id=k // 4),
                            tokens=[int(x) for x in rng.integers(0, 151936, size=m)],
                            behavior_logprobs=[float(x) for x in rng.normal(-3, 1, size=m)],
                            reward=SimpleNamespace(reward=float(rng.choice([5.0, -5.0]))))
        if with_versions:
            t.versions = [int(x) for x in np.sort(rng.integers(90, 100, size=m))]
        out.append(t)
    return out


def _fill(P, trajs):
    T, n = P.count(trajs)
    tok = np.empty(T, np.int64)
    beh = np.empty(T, np.float64)
    ver = np.empty(T, np.int32)
    bnd = np.empty(n + 1, np.int64)
    rew = np.empty(n, np.float64)
    hv = P.fill(trajs, tok.ctypes.data, beh.ctypes.data, ver.ctypes.data, bnd.ctypes.data,
                rew.ctypes.data, T)
    return tok, beh, ver if hv else None, bnd, rew


def test_packer_matches_python_flattening(P):
    rng = np.random.default_rng(0)
    trajs = _trajs(rng, 200)
    tok, beh, ver, bnd, rew = _fill(P, trajs)
    # build_train_batch's flattening (trainer.py:91-101), restated
    r_tok, r_beh, r_ver, r_bnd = [], [], [], [0]
    for t in trajs:
        r_tok.extend(t.tokens)
        r_beh.extend(t.behavior_logprobs)
        r_ver.extend(t.versions)
        r_bnd.append(len(r_tok))
    assert np.array_equal(tok, np.array(r_tok, dtype=np.int64))
    assert np.array_equal(beh, np.array(r_beh, dtype=np.float64))  # bit-exact
    assert np.array_equal(ver, np.array(r_ver, dtype=np.int32))
    assert np.array_equal(bnd, np.array(r_bnd, dtype=np.int64))
    assert np.array_equal(rew, np.array([t.reward.reward for t in trajs]))


def test_packer_versions_optional_and_empty(P):
    rng = np.random.default_rng(1)
    trajs = _trajs(rng, 20, with_versions=False)
    tok, beh, ver, bnd, rew = _fill(P, trajs)
    assert ver is None and bnd[-1] == len(tok)
    assert P.count([]) == (0, 0)


def test_packer_errors_match_reference(P):
    rng = np.random.default_rng(2)
    trajs = _trajs(rng, 6)
    trajs[2].reward = None
    with pytest.raises(ValueError, match="trajectory 2 is unrewarded"):  # trainer.py:93-94
        _fill(P, trajs)
    trajs = _trajs(rng, 6, empty_every=0)
    trajs[1].behavior_logprobs = trajs[1].behavior_logprobs[:-1]
    with pytest.raises(ValueError, match="behavior_logprobs length"):
        _fill(P, trajs)
    trajs = _trajs(rng, 3)
    T, n = P.count(trajs)
    buf, beh, bnd, rew = np.empty(T, np.int64), np.empty(T), np.empty(n + 1, np.int64), np.empty(n)
    with pytest.raises(ValueError, match="capacity"):
        P.fill(trajs, buf.ctypes.data, beh.ctypes.data, 0, bnd.ctypes.data, rew.ctypes.data, T - 1)
