"""Rollout-side recording at emission: EmissionRecorder vs the
reference's RolloutWorker.step (rollout.py:140-165), which appends the token, its
behaviour log-prob under the generating params and that params' version."""
import os
import sys

import numpy as np
import pytest
import torch

import oracle as O
from paper_2505_24298_b200 import kernels as K
from paper_2505_24298_b200.hotpath import EmissionRecorder

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _decode(rec, n_slots, steps, V, dtype, seed, head=None):
    """Ragged decode loop: a random subset of slots emits each step, the version moves
    every few steps (update_weights at a token boundary).  Returns the host record."""
    rng = np.random.default_rng(seed)
    want = {s: ([], [], []) for s in range(n_slots)}
    version = 3
    for step in range(steps):
        if step % 4 == 3:
            version += 1
        live = np.sort(rng.choice(n_slots, size=rng.integers(1, n_slots + 1), replace=False))
        B = len(live)
        tok = rng.integers(0, V, size=B)
        if head is None:
            x = (torch.randn(B, V, generator=torch.Generator().manual_seed(seed * 1000 + step))
                 * 2).to(dtype)
            lp = O.token_logprobs(x.double().numpy(), tok)
            rec.step(torch.as_tensor(live, dtype=torch.int32).cuda(), torch.as_tensor(tok).cuda(),
                     version, logits=x.cuda())
        else:
            W, b = head
            h = (torch.randn(B, W.shape[1], generator=torch.Generator().manual_seed(step)) * 0.5
                 ).to(W.dtype)
            x = h.double() @ W.double().cpu().t() + b.double().cpu()
            lp = O.token_logprobs(x.numpy(), tok)
            rec.step(torch.as_tensor(live, dtype=torch.int32).cuda(), torch.as_tensor(tok).cuda(),
                     version, hidden=h.cuda(), weight=W, bias=b)
        for i, s in enumerate(live):
            want[s][0].append(tok[i])
            want[s][1].append(lp[i])
            want[s][2].append(version)
    return want


@pytest.mark.parametrize("dtype,V", [(torch.float32, 32000), (torch.bfloat16, 151936),
                                     (torch.float64, 1000)])
def test_recorder_matches_per_token_record(dtype, V):
    rec = EmissionRecorder(n_slots=24, max_len=40, device="cuda")
    want = _decode(rec, 24, 30, V, dtype, seed=V % 97)
    tol = 1e-12 if dtype == torch.float64 else 1e-5
    for s, (tok, lp, ver) in want.items():
        got_tok, got_lp, got_ver = rec.trajectory(s)
        assert got_tok.tolist() == [int(t) for t in tok]
        assert got_ver.tolist() == ver
        assert np.allclose(got_lp, lp, rtol=tol, atol=tol)
    assert rec.launches == 2 * 30


def test_recorder_fused_head_k7():
    V, d = 4096, 256
    g = torch.Generator().manual_seed(5)
    W = (torch.randn(V, d, generator=g) * 0.05).to(torch.bfloat16).cuda()
    b = (torch.randn(V, generator=g) * 0.1).float().cuda()
    rec = EmissionRecorder(n_slots=300, max_len=8, device="cuda")
    want = _decode(rec, 300, 6, V, None, seed=2, head=(W, b))
    for s, (tok, lp, ver) in want.items():
        got_tok, got_lp, got_ver = rec.trajectory(s)
        assert got_tok.tolist() == [int(t) for t in tok] and got_ver.tolist() == ver
        assert np.allclose(got_lp, lp, rtol=1e-5, atol=1e-5)


def test_recorder_overflow_and_bad_slot_are_reported():
    V = 64
    rec = EmissionRecorder(n_slots=2, max_len=2, device="cuda")
    x = torch.randn(2, V, device="cuda")
    for _ in range(2):
        rec.step(torch.tensor([0, 1], dtype=torch.int32, device="cuda"),
                 torch.tensor([1, 2], device="cuda"), 0, logits=x)
    rec.check()
    rec.step(torch.tensor([1], dtype=torch.int32, device="cuda"), torch.tensor([3], device="cuda"),
             0, logits=x[:1])
    with pytest.raises(K._lib.ArealError, match="exceeds capacity"):
        rec.check()
    assert int(rec.lengths[1]) == 2  # the refused token is not recorded
    rec2 = EmissionRecorder(n_slots=2, max_len=2, device="cuda")
    rec2.step(torch.tensor([5], dtype=torch.int32, device="cuda"), torch.tensor([3], device="cuda"),
              0, logits=x[:1])
    with pytest.raises(K._lib.ArealError, match="bad shape"):
        rec2.check()
    rec.release(0)
    assert int(rec.lengths[0]) == 0


@pytest.fixture
def ref_rollout(monkeypatch):
    if not os.path.isdir(os.path.join(REF, "asyncrl")):
        pytest.skip("reference not installed in baseline/_ref")
    monkeypatch.syspath_prepend(REF)
    for name in [m for m in sys.modules if m == "asyncrl" or m.startswith("asyncrl.")]:
        monkeypatch.delitem(sys.modules, name)
    import asyncrl.policy as P
    import asyncrl.rollout as R
    import asyncrl.tasks as TK
    return P, R, TK


def test_recorder_reproduces_reference_rollout_worker(ref_rollout):
    """Drive the reference's RolloutWorker (interleaved sequences, update_weights between
    steps), then replay each emission on the GPU — logits of the same features under the
    params in effect (float64), the worker's sampled token and version — through the
    recorder: tokens and versions exact, behaviour log-probs within 1e-12."""
    P, R, TK = ref_rollout
    feat = P.ContextFeaturizer(P.PolicyConfig())
    rng = np.random.default_rng(0)

    def params(v):
        return P.VersionedParams(v, rng.normal(0, 0.3, (feat.config.vocab_size, feat.feature_dim)),
                                 rng.normal(0, 0.3, feat.config.vocab_size))

    snaps = [params(0)]
    worker = R.RolloutWorker(snaps[0], feat, seed=11)
    prompts = [TK.make_prompt(100 + i, TK.TASK_KINDS[i % 2]) for i in range(6)]
    handles = [worker.start(R.GenerateRequest(p, max_new_tokens=12, trajectory_id=i))
               for i, p in enumerate(prompts)]
    live = dict(enumerate(handles))
    emitted = []  # (slot, prefix, token, version) in emission order, one decode step per round
    trajs = {}
    while live:
        step = []
        for slot, h in list(live.items()):
            seq = worker._active[h]
            prefix = list(seq.trajectory.tokens)
            done = worker.step(h)
            t = seq.trajectory
            step.append((slot, prefix, t.tokens[-1], t.versions[-1]))
            if done:
                trajs[slot] = worker.finish(h)
                del live[slot]
        emitted.append(step)
        if len(emitted) % 3 == 0:
            snaps.append(params(len(snaps)))
            worker.update_weights(snaps[-1])

    rec = EmissionRecorder(n_slots=len(prompts), max_len=16, device="cuda")
    for step in emitted:
        versions = {v for _, _, _, v in step}
        assert len(versions) == 1  # one weight version per decode step
        v = versions.pop()
        pr = snaps[v]
        x = np.stack([feat.features(prompts[s], pre) @ pr.weights.T + pr.bias
                      for s, pre, _, _ in step])
        rec.step(torch.tensor([s for s, _, _, _ in step], dtype=torch.int32, device="cuda"),
                 torch.tensor([t for _, _, t, _ in step], device="cuda"), v,
                 logits=torch.as_tensor(x).cuda())
    for slot, t in trajs.items():
        tok, lp, ver = rec.trajectory(slot)
        assert tok.tolist() == list(t.tokens)
        assert ver.tolist() == list(t.versions)
        assert np.allclose(lp, t.behavior_logprobs, rtol=1e-12, atol=1e-12)
