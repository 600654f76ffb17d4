"""K6 fused clip + Adam (areal_adam_step) vs the reference's apply_update.

Golden vectors: tests/golden/adam.npz (the real reference's grad.scale_(-1/n) +
apply_update, trainer.py:329-331 / policy.py:215-258, 3 chained steps).  The fp64
EXACT mode must be bit-identical; the fp32 FAST mode (LM-scale master weights,
bf16/fp32 grads) is checked against a float64 torch restatement."""
import numpy as np
import pytest
import torch

from conftest import load_cases

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2505_24298_b200 import kernels as K

DEV = "cuda"


def _run_case(c, sign=1.0):
    W = torch.as_tensor(c["W0"], device=DEV).clone()
    b = torch.as_tensor(c["b0"], device=DEV).clone()
    mw, vw, mb, vb = (torch.zeros_like(W), torch.zeros_like(W), torch.zeros_like(b),
                      torch.zeros_like(b))
    norms = []
    for k in range(int(c["steps"])):
        gw = torch.as_tensor(c[f"gw{k}"], device=DEV) * sign
        gb = torch.as_tensor(c[f"gb{k}"], device=DEV) * sign
        nrm = K.adam_step([W, b], [gw, gb], [mw, mb], [vw, vb], step=k + 1, lr=float(c["lr"]),
                          beta1=0.9, beta2=0.95, eps=1e-5, weight_decay=float(c["wd"]),
                          clip_norm=float(c["clip"]), grad_scale=-sign / int(c[f"n{k}"]))
        norms.append(nrm.cpu().numpy())
    return W, b, mw, vw, mb, vb, norms


def test_adam_exact_bit_identical_to_reference():
    for c in load_cases("adam.npz"):
        W, b, mw, vw, mb, vb, norms = _run_case(c)
        for k, nrm in enumerate(norms):
            assert nrm[0] == float(c[f"norm{k}"]) and nrm[1] == 0
        for got, key in ((W, "W"), (b, "b"), (mw, "mw"), (vw, "vw"), (mb, "mb"), (vb, "vb")):
            assert np.array_equal(got.cpu().numpy(), c[key]), key


def test_adam_exact_negated_gradient_same_result():
    # the trainer feeds -grad with grad_scale = +1/n: sign flips are exact
    c = load_cases("adam.npz")[2]
    W, b, *_ = _run_case(c, sign=-1.0)
    assert np.array_equal(W.cpu().numpy(), c["W"]) and np.array_equal(b.cpu().numpy(), c["b"])


def test_adam_nonfinite_leaves_state_untouched():
    W = torch.randn(50, 7, dtype=torch.float64, device=DEV)
    b = torch.randn(50, dtype=torch.float64, device=DEV)
    gw = torch.randn_like(W)
    gb = torch.randn_like(b)
    gw[3, 4] = float("nan")
    gb[7] = float("inf")
    mw, vw, mb, vb = (torch.rand_like(W), torch.rand_like(W), torch.rand_like(b), torch.rand_like(b))
    before = [t.clone() for t in (W, b, mw, vw, mb, vb)]
    nrm = K.adam_step([W, b], [gw, gb], [mw, mb], [vw, vb], step=3, lr=1e-2, beta1=0.9,
                      beta2=0.95, eps=1e-5, weight_decay=0.05, clip_norm=1.0)
    assert int(nrm[1].item()) == 2
    for x, y in zip((W, b, mw, vw, mb, vb), before):
        assert torch.equal(x, y)


def _torch_adam(ps, gs, ms, vs, step, lr, b1, b2, eps, wd, clip, scale):
    gs = [g.double() * scale for g in gs]
    norm = torch.sqrt(sum((g * g).sum() for g in gs))
    if clip > 0 and norm > clip:
        gs = [g * (clip / norm) for g in gs]
    out = []
    for p, g, m, v in zip(ps, gs, ms, vs):
        p, m, v = p.double(), m.double(), v.double()
        m = b1 * m + (1 - b1) * g
        v = b2 * v + (1 - b2) * g * g
        p = p - lr * ((m / (1 - b1 ** step)) / (torch.sqrt(v / (1 - b2 ** step)) + eps) + wd * p)
        out.append((p, m, v))
    return out, float(norm)


@pytest.mark.parametrize("gdt", [torch.float32, torch.bfloat16, torch.float16])
@pytest.mark.parametrize("mag", [1e-3, 10.0])
def test_adam_fast_fp32_master_multi_tensor(gdt, mag):
    g = torch.Generator(device=DEV).manual_seed(0)
    shapes = [(1536, 1536), (151936 // 64, 96), (1536,), (7,), (3, 5, 11)]
    ps = [torch.randn(s, device=DEV, generator=g) * 0.02 for s in shapes]
    gs = [(torch.randn(s, device=DEV, generator=g) * mag).to(gdt) for s in shapes]
    ms = [torch.randn(s, device=DEV, generator=g) * 1e-3 for s in shapes]
    vs = [torch.rand(s, device=DEV, generator=g) * 1e-4 for s in shapes]
    ref, ref_norm = _torch_adam(ps, gs, ms, vs, 5, 1e-4, 0.9, 0.95, 1e-8, 0.1, 1.0, 0.5)
    nrm = K.adam_step(ps, gs, ms, vs, step=5, lr=1e-4, beta1=0.9, beta2=0.95, eps=1e-8,
                      weight_decay=0.1, clip_norm=1.0, grad_scale=0.5)
    assert abs(float(nrm[0]) - ref_norm) <= 1e-9 * ref_norm and int(nrm[1]) == 0
    for (p, m, v), P, M, Vv in zip(ref, ps, ms, vs):
        torch.testing.assert_close(P.double(), p, rtol=1e-6, atol=1e-9)
        torch.testing.assert_close(M.double(), m, rtol=1e-6, atol=1e-12)
        torch.testing.assert_close(Vv.double(), v, rtol=1e-6, atol=1e-14)


def test_adam_fast_deterministic():
    g = torch.Generator(device=DEV).manual_seed(1)
    p0 = torch.randn(1 << 22, device=DEV, generator=g)
    gr = torch.randn(1 << 22, device=DEV, generator=g)
    outs = []
    for _ in range(2):
        p, m, v = p0.clone(), torch.zeros_like(p0), torch.zeros_like(p0)
        n = K.adam_step([p], [gr], [m], [v], step=1, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8,
                        weight_decay=0.0, clip_norm=1.0)
        outs.append((p, float(n[0])))
    assert torch.equal(outs[0][0], outs[1][0]) and outs[0][1] == outs[1][1]


def test_adam_rejects_bad_arguments():
    p = torch.zeros(4, dtype=torch.float64, device=DEV)
    with pytest.raises(TypeError):
        K.adam_step([p], [p.float()], [p], [p], step=1, lr=1, beta1=0.9, beta2=0.9, eps=1,
                    weight_decay=0, clip_norm=1)
    with pytest.raises(ValueError):
        K.adam_step([p], [p[:2]], [p], [p], step=1, lr=1, beta1=0.9, beta2=0.9, eps=1,
                    weight_decay=0, clip_norm=1)


def test_adam_device_divisor_bit_identical():
    """grad_scale = -1 with the divisor n on the device (K2's all-reduced n_valid) gives
    the same bits as the host-computed -1.0/n (trainer.py:330), with no host sync."""
    for c in load_cases("adam.npz")[:3]:
        W = torch.as_tensor(c["W0"], device=DEV).clone()
        b = torch.as_tensor(c["b0"], device=DEV).clone()
        mw, vw, mb, vb = (torch.zeros_like(W), torch.zeros_like(W), torch.zeros_like(b),
                          torch.zeros_like(b))
        for k in range(int(c["steps"])):
            n_dev = torch.tensor([float(int(c[f"n{k}"]))], dtype=torch.float64, device=DEV)
            K.adam_step([W, b], [torch.as_tensor(c[f"gw{k}"], device=DEV),
                                 torch.as_tensor(c[f"gb{k}"], device=DEV)], [mw, mb], [vw, vb],
                        step=k + 1, lr=float(c["lr"]), beta1=0.9, beta2=0.95, eps=1e-5,
                        weight_decay=float(c["wd"]), clip_norm=float(c["clip"]),
                        grad_scale=-1.0, grad_scale_divisor=n_dev)
        assert np.array_equal(W.cpu().numpy(), c["W"]) and np.array_equal(b.cpu().numpy(), c["b"])
    # divisor 0 -> max(n, 1) = 1 (trainer.py:329)
    p = torch.ones(5, device=DEV)
    K.adam_step([p], [torch.ones(5, device=DEV)], [torch.zeros(5, device=DEV)],
                [torch.zeros(5, device=DEV)], step=1, lr=0.1, beta1=0.9, beta2=0.95, eps=1e-8,
                weight_decay=0.0, clip_norm=0.0, grad_scale=1.0,
                grad_scale_divisor=torch.zeros(1, dtype=torch.float64, device=DEV))
    torch.testing.assert_close(p, torch.full((5,), 0.9, device=DEV), rtol=1e-6, atol=1e-6)
