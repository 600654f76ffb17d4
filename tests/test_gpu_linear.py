"""K7 fused LM-head + log-softmax-gather (areal_linear_logprob_fwd, tcgen05) vs the
float64 oracle: recompute_prox_logprobs with the model's output layer
(logits = features @ W.T + b, policy.py:133-163; trainer.py:128-137), computed from
the same 16-bit values in float64.  The fused kernel accumulates in fp32 on the
tensor cores and never rounds logits to 16 bits, so the tolerance is fp32-level."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2505_24298_b200 import kernels as K

DEV = "cuda"
ATOL = 2e-4


def _case(n, V, d, dtype=torch.bfloat16, bias=True, seed=0, scale=1.0):
    g = torch.Generator(device=DEV).manual_seed(seed)
    h = (torch.randn(n, d, device=DEV, generator=g) * scale).to(dtype)
    w = (torch.randn(V, d, device=DEV, generator=g) / d ** 0.5 * 4).to(dtype)
    b = torch.randn(V, device=DEV, generator=g) if bias else None
    tok = torch.randint(0, V, (n,), device=DEV, generator=g)
    return h, w, b, tok


def _ref(h, w, b, tok, entropy=True):
    x = h.double() @ w.double().t()
    if b is not None:
        x = x + b.double()
    lse = torch.logsumexp(x, dim=1)
    lp = x.gather(1, tok[:, None])[:, 0] - lse
    ent = None
    if entropy:
        p = torch.softmax(x, dim=1)
        ent = -(p * torch.log_softmax(x, dim=1)).sum(1)
    return lp, ent


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("n,V,d", [(1, 1000, 64), (100, 4096, 128), (300, 32000, 256),
                                   (129, 2049, 64), (257, 151936, 1536), (64, 152064, 512),
                                   (1000, 2000, 64)])
def test_linear_logprob_matches_float64(n, V, d, cg):
    h, w, b, tok = _case(n, V, d)
    lp, ent = K.linear_logprob_fwd(h, w, tok, bias=b, with_entropy=True, cta_group=cg)
    rlp, rent = _ref(h, w, b, tok)
    torch.testing.assert_close(lp, rlp, rtol=0, atol=ATOL)
    torch.testing.assert_close(ent, rent, rtol=1e-5, atol=ATOL)


def test_linear_logprob_numpy_oracle_small():
    # the CPU oracle (linear_logits + token_logprobs) on the same bf16 values
    h, w, b, tok = _case(37, 517, 64, seed=3)
    lp, ent = K.linear_logprob_fwd(h, w, tok, bias=b, with_entropy=True)
    x = O.linear_logits(h.double().cpu().numpy(), w.double().cpu().numpy(), b.double().cpu().numpy())
    np.testing.assert_allclose(lp.cpu().numpy(), O.token_logprobs(x, tok.cpu().numpy()), atol=ATOL)
    np.testing.assert_allclose(ent.cpu().numpy(), O.token_entropy(x), atol=ATOL)


@pytest.mark.parametrize("cg", [1, 2])
def test_linear_logprob_fp16_no_bias_row_index(cg):
    h, w, _, tok_rows = _case(200, 5000, 192, dtype=torch.float16, bias=False, seed=5)
    # rows map to a permuted global token order
    perm = torch.randperm(200, device=DEV).to(torch.int32)
    tokens = torch.empty(200, dtype=torch.int64, device=DEV)
    tokens[perm.long()] = tok_rows
    lp, _ = K.linear_logprob_fwd(h, w, tokens, row_index=perm, cta_group=cg)
    rlp, _ = _ref(h, w, None, tok_rows, entropy=False)
    torch.testing.assert_close(lp[perm.long()], rlp, rtol=0, atol=ATOL)


def test_linear_logprob_matches_materialised_path():
    # fused K7 == cuBLAS logits (fp32 out) + K1 on the same inputs
    h, w, b, tok = _case(512, 32000, 512, seed=7)
    lp, _ = K.linear_logprob_fwd(h, w, tok, bias=b)
    logits = torch.addmm(b, h.float(), w.float().t())
    lp1, _ = K.logprob_fwd(logits, tok, with_entropy=False)
    torch.testing.assert_close(lp, lp1, rtol=0, atol=ATOL)


def test_linear_logprob_rejects_bad_shapes():
    h = torch.zeros(4, 100, dtype=torch.bfloat16, device=DEV)
    w = torch.zeros(10, 100, dtype=torch.bfloat16, device=DEV)
    t = torch.zeros(4, dtype=torch.int64, device=DEV)
    with pytest.raises(RuntimeError):
        K.linear_logprob_fwd(h, w, t)  # d % 64 != 0
    with pytest.raises(TypeError):
        K.linear_logprob_fwd(h.float(), w.float(), t)


@pytest.mark.parametrize("chunk", [64, 1000])
def test_linear_ppo_fwd_bwd_matches_float64_autograd(chunk):
    """Loss + backward through the LM head in token chunks (hotpath.linear_ppo_fwd_bwd)
    vs float64 autograd of the restated objective (trainer.py:150-184) on the same
    16-bit inputs: gradients wrt hidden, W and b, and the statistics."""
    from paper_2505_24298_b200.hotpath import linear_ppo_fwd_bwd
    T, V, d = 300, 5000, 128
    h, w, b, tok = _case(T, V, d, seed=11)
    g = torch.Generator(device=DEV).manual_seed(12)
    x64 = h.double() @ w.double().t() + b.double()
    lp = torch.log_softmax(x64, 1).gather(1, tok[:, None])[:, 0]
    # ratios stay well inside (1-eps, 1+eps): the bf16 rounding of the head's logits
    # (any bf16 LM head does it) must not flip a token across the clip boundary
    prox = lp + 0.01 * torch.randn(T, dtype=torch.float64, device=DEV, generator=g)
    behav = prox + 0.2 * torch.randn(T, dtype=torch.float64, device=DEV, generator=g)
    adv = torch.randn(T, dtype=torch.float64, device=DEV, generator=g)
    dh, dw, db, st = linear_ppo_fwd_bwd(h, w, tok, behav, prox, adv, bias=b, chunk_tokens=chunk)
    # float64 autograd of -sum(objective), objective as trainer.py:165-176
    H = h.double().requires_grad_(True)
    W = w.double().requires_grad_(True)
    B = b.double().requires_grad_(True)
    lpa = torch.log_softmax(H @ W.t() + B, 1).gather(1, tok[:, None])[:, 0]
    scale = torch.exp(prox - behav)
    ratio = torch.exp(lpa - prox)
    obj = scale * torch.minimum(ratio * adv, torch.clamp(ratio, 0.8, 1.2) * adv)
    (-obj.sum()).backward()
    # (1) tight: the float64 chain rule through the head's own bf16 logits (the library's
    # logits GEMM, tested on its own above), i.e. the restated _surrogate_terms on
    # exactly what K2 sees
    lg16 = K.lm_head_gemm("logits", h, w, bias=b)
    ref = O.surrogate_terms(lg16.double().cpu().numpy(), tok.cpu().numpy(), behav.cpu().numpy(),
                            prox.cpu().numpy(), adv.cpu().numpy())
    dl = torch.as_tensor(ref["dlogits"], device=DEV)
    for got, r in ((dh, dl @ w.double()), (dw, dl.t() @ h.double()), (db, dl.sum(0))):
        err = (got.double() - r).abs().max() / r.abs().max()
        assert float(err) < 2e-2, float(err)
    # (2) loose: float64 autograd with unrounded logits.  bf16 logits of magnitude ~16
    # carry 0.06 absolute rounding (6% on individual probabilities): inherent in a bf16
    # head, so this only guards signs and scales
    for got, r in ((dh.double(), H.grad), (dw.double(), W.grad), (db.double(), B.grad)):
        err = (got - r).abs().max() / r.abs().max()
        assert float(err) < 1e-1, float(err)
    s = st.cpu().numpy()
    assert s[7] == T and s[1] == T and s[2] == 0
    o = float(obj.detach().sum())
    assert abs(s[0] - o) <= 2e-2 * max(1.0, abs(o))


@pytest.mark.parametrize("cg", [1, 2])
def test_linear_logprob_edge_shapes(cg):
    # tiny vocab (< one 256-column tile), one row, empty batch, out-of-range token
    for n, V, d in ((1, 7, 64), (3, 255, 64), (5, 257, 128)):
        h, w, b, tok = _case(n, V, d, seed=n)
        lp, ent = K.linear_logprob_fwd(h, w, tok, bias=b, with_entropy=True, cta_group=cg)
        rlp, rent = _ref(h, w, b, tok)
        torch.testing.assert_close(lp, rlp, rtol=0, atol=ATOL)
        torch.testing.assert_close(ent, rent, rtol=1e-5, atol=ATOL)
    h, w, b, tok = _case(4, 300, 64, seed=9)
    tok[1] = 300  # out of range: lp = NaN (K1's documented behaviour), others unaffected
    lp, _ = K.linear_logprob_fwd(h, w, tok, bias=b, cta_group=cg)
    assert torch.isnan(lp[1]) and torch.isfinite(lp[[0, 2, 3]]).all()
    empty = torch.empty(0, 64, dtype=torch.bfloat16, device=DEV)
    lp0, _ = K.linear_logprob_fwd(empty, w, torch.empty(0, dtype=torch.int64, device=DEV))
    assert lp0.numel() == 0


def test_linear_logprob_deterministic():
    h, w, b, tok = _case(700, 40000, 256, seed=21)
    a1, e1 = K.linear_logprob_fwd(h, w, tok, bias=b, with_entropy=True)
    a2, e2 = K.linear_logprob_fwd(h, w, tok, bias=b, with_entropy=True)
    assert torch.equal(a1, a2) and torch.equal(e1, e2)


def test_linear_ppo_fwd_bwd_row_index_and_prox_from_lp():
    """row_index (packed rows -> global tokens) and prox_from_lp (first minibatch):
    chunked backward through the head == the unchunked call; prox written via lp_out."""
    from paper_2505_24298_b200.hotpath import linear_ppo_fwd_bwd
    T, V, d = 257, 3000, 64
    h, w, b, tok_rows = _case(T, V, d, seed=31)
    g = torch.Generator(device=DEV).manual_seed(32)
    perm = torch.randperm(T, device=DEV, generator=g).to(torch.int32)
    tokens = torch.empty(T, dtype=torch.int64, device=DEV)
    tokens[perm.long()] = tok_rows
    behav = torch.full((T,), -8.0, dtype=torch.float64, device=DEV)
    adv = torch.randn(T, dtype=torch.float64, device=DEV, generator=g)
    outs = []
    for chunk in (50, T):
        lp = torch.zeros(T, dtype=torch.float64, device=DEV)
        dh, dw, db, st = linear_ppo_fwd_bwd(h, w, tokens, behav, None, adv, bias=b,
                                            row_index=perm, chunk_tokens=chunk,
                                            prox_from_lp=True, lp_out=lp)
        outs.append((dh.float(), dw, db, st, lp))
    for a, c in zip(outs[0], outs[1]):
        torch.testing.assert_close(a, c, rtol=1e-4, atol=1e-5)
    # prox == the float64 log-softmax of the head's own bf16 logits (what K2 reads)
    lg16 = K.lm_head_gemm("logits", h, w, bias=b).double()
    rlp = torch.log_softmax(lg16, 1).gather(1, tok_rows[:, None])[:, 0]
    torch.testing.assert_close(outs[0][4][perm.long()], rlp, rtol=0, atol=1e-4)
    s = outs[0][3].cpu().numpy()
    assert s[1] == T and abs(s[3] - T) < 1e-9  # every ratio exactly 1


@pytest.mark.parametrize("seed", range(16))
def test_linear_logprob_fuzz(seed):
    """Seeded random shapes for K7: rows, vocab (tails vs the 256-column tiles and the
    2048-column blocks), d in multiples of 64, bias on/off, entropy on/off, both CTA
    groups, fp16/bf16 — against the float64 head + log-softmax."""
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(1, 700))
    V = int(rng.integers(1, 20000))
    d = int(64 * rng.integers(1, 9))
    dtype = torch.bfloat16 if seed % 2 == 0 else torch.float16
    h, w, b, tok = _case(n, V, d, dtype=dtype, bias=bool(seed % 3), seed=seed)
    ent_on = bool(seed % 4 < 2)
    lp, ent = K.linear_logprob_fwd(h, w, tok, bias=b, with_entropy=ent_on, cta_group=1 + seed % 2)
    rlp, rent = _ref(h, w, b, tok, entropy=ent_on)
    torch.testing.assert_close(lp, rlp, rtol=0, atol=ATOL)
    if ent_on:
        torch.testing.assert_close(ent, rent, rtol=1e-5, atol=ATOL)


def _gemm_operands(op, M, N, K, dtype, seed, pad=0):
    """A, B (row-major, rows padded by `pad` elements) for areal_lm_head_gemm and the
    float64 reference C."""
    g = torch.Generator(device=DEV).manual_seed(seed)

    def mat(r, c):  # row stride: c rounded up to 8 elements (16 bytes) + pad
        full = torch.randn(r, (c + 7) // 8 * 8 + pad, device=DEV, generator=g).to(dtype)
        return full[:, :c]
    if op == "logits":
        A, B = mat(M, K), mat(N, K)
        ref = A.double() @ B.double().t()
    elif op == "dhidden":
        A, B = mat(M, K), mat(K, N)
        ref = A.double() @ B.double()
    else:
        A, B = mat(K, M), mat(K, N)
        ref = A.double().t() @ B.double()
    absref = {"logits": lambda: A.double().abs() @ B.double().abs().t(),
              "dhidden": lambda: A.double().abs() @ B.double().abs(),
              "dweight": lambda: A.double().abs().t() @ B.double().abs()}[op]()
    return A, B, ref, absref


@pytest.mark.parametrize("op", ["logits", "dhidden", "dweight"])
@pytest.mark.parametrize("M,N,Kd", [(256, 256, 64), (300, 1000, 128), (1, 7, 64), (517, 333, 200),
                                    (1024, 1536, 4096), (77, 4096, 1000),
                                    # odd N-tile counts: the second CTA pair of a 2x2 cluster
                                    # computes a tile past N (zero B, clipped store)
                                    (300, 700, 128), (640, 1200, 96)])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_lm_head_gemm_matches_float64(op, M, N, Kd, dtype):
    """Each tcgen05 GEMM of the head (K-major / MN-major operands, tails of every tile
    dimension, padded row strides) against float64 matmul of the same 16-bit values:
    fp32 accumulation error <= 2^-20 x K of the absolute products, plus the output
    rounding (16-bit outputs: half an ulp)."""
    A, B, ref, absref = _gemm_operands(op, M, N, Kd, dtype, seed=M + N + Kd, pad=8)
    bias = torch.randn(N, device=DEV) if op == "logits" else None
    C = K.lm_head_gemm(op, A, B, bias=bias)
    if bias is not None:
        ref = ref + bias.double()
        absref = absref + bias.double().abs()
    ulp = 2.0 ** -8 if dtype == torch.bfloat16 else 2.0 ** -11
    out_round = ulp * ref.abs() if op != "dweight" else 0.0
    bound = 2.0 ** -20 * Kd * absref + out_round + 1e-30
    err = (C.double() - ref).abs()
    assert bool((err <= bound).all()), float((err / bound).max())


def test_lm_head_gemm_accumulate_and_strides():
    """DWEIGHT accumulates into an existing fp32 C (row stride > N); LOGITS writes into a
    row-strided 16-bit buffer and leaves the padding untouched."""
    A, B, ref, _ = _gemm_operands("dweight", 300, 200, 129, torch.bfloat16, seed=5)
    Cbig = torch.ones(300, 208, dtype=torch.float32, device=DEV)
    C = Cbig[:, :200]
    K.lm_head_gemm("dweight", A, B, C, accumulate=True)
    torch.testing.assert_close(C.double(), ref + 1.0, rtol=1e-5, atol=1e-4)
    assert bool((Cbig[:, 200:] == 1).all())
    K.lm_head_gemm("dweight", A, B, C, accumulate=False)
    torch.testing.assert_close(C.double(), ref, rtol=1e-5, atol=1e-4)
    A, B, ref, _ = _gemm_operands("logits", 70, 1000, 64, torch.bfloat16, seed=6)
    big = torch.full((70, 1008), 7.0, dtype=torch.bfloat16, device=DEV)
    K.lm_head_gemm("logits", A, B, big[:, :1000])
    torch.testing.assert_close(big[:, :1000].double(), ref, rtol=1e-2, atol=1e-2)
    assert bool((big[:, 1000:] == 7).all())


def test_lm_head_gemm_rejects_bad_inputs():
    a = torch.randn(64, 64, device=DEV).to(torch.bfloat16)
    with pytest.raises(ValueError):
        K.lm_head_gemm("logits", a, a[:, :32])  # inner dims differ
    with pytest.raises(TypeError):
        K.lm_head_gemm("logits", a.float(), a.float())
    with pytest.raises(ValueError):
        K.lm_head_gemm("dhidden", a, a, bias=torch.zeros(64, device=DEV))
    odd = torch.randn(64, 70, device=DEV).to(torch.bfloat16)[:, :65]  # row stride 140 B
    with pytest.raises(K._lib.ArealError, match="misaligned"):
        K.lm_head_gemm("logits", odd, odd)


@pytest.mark.parametrize("rows,cols", [(1, 7), (3000, 5000), (4100, 151936), (0, 9)])
def test_colsum_matches_float64(rows, cols):
    g = torch.Generator(device=DEV).manual_seed(rows + cols)
    x = torch.randn(rows, cols, device=DEV, generator=g).to(torch.bfloat16)
    ref = x.double().sum(0)
    got = K.colsum(x)
    assert torch.allclose(got.double(), ref, rtol=1e-5, atol=1e-5 * max(rows, 1) ** 0.5)
    got2 = K.colsum(x, out=torch.ones(cols, device=DEV), accumulate=True)
    assert torch.allclose(got2.double(), ref + 1, rtol=1e-5, atol=1e-5 * max(rows, 1) ** 0.5)
    assert torch.equal(K.colsum(x), got)  # deterministic


@pytest.mark.parametrize("T,V,d", [(1, 7, 64), (300, 1000, 128), (517, 2049, 192), (2000, 5000, 256)])
@pytest.mark.parametrize("accumulate", [False, True])
def test_lm_head_backward_grouped(T, V, d, accumulate):
    """areal_lm_head_backward (one grouped launch: DHIDDEN + DWEIGHT, grad_b summed from
    the shared-memory dL tiles) == the float64 products of the same 16-bit values."""
    g = torch.Generator(device=DEV).manual_seed(T + V + d)
    ldv = (V + 7) // 8 * 8  # 16-byte row stride, as the hot path allocates the chunk buffer
    dl = (torch.randn(T, ldv, device=DEV, generator=g) * 0.1).to(torch.bfloat16)[:, :V]
    h = torch.randn(T, d, device=DEV, generator=g).to(torch.bfloat16)
    w = (torch.randn(V, d, device=DEV, generator=g) / d ** 0.5).to(torch.bfloat16)
    gw0 = torch.randn(V, d, device=DEV, generator=g) if accumulate else None
    gb0 = torch.randn(V, device=DEV, generator=g) if accumulate else None
    gw = gw0.clone() if accumulate else None
    gb = gb0.clone() if accumulate else None
    dh, gw, gb = K.lm_head_backward(dl, h, w, grad_weight=gw, grad_bias=gb, accumulate=accumulate)
    rdh = dl.double() @ w.double()
    rgw = dl.double().t() @ h.double() + (gw0.double() if accumulate else 0)
    rgb = dl.double().sum(0) + (gb0.double() if accumulate else 0)
    bound_h = 2.0 ** -20 * V * (dl.double().abs() @ w.double().abs()) + 2.0 ** -8 * rdh.abs() + 1e-30
    assert bool(((dh.double() - rdh).abs() <= bound_h).all())
    bound_w = 2.0 ** -20 * T * (dl.double().abs().t() @ h.double().abs()) + 1e-6 * rgw.abs() + 1e-30
    assert bool(((gw.double() - rgw).abs() <= bound_w).all())
    bound_b = 2.0 ** -20 * T * dl.double().abs().sum(0) + 1e-6 * rgb.abs() + 1e-30
    assert bool(((gb.double() - rgb).abs() <= bound_b).all())
    dh2, gw2, gb2 = K.lm_head_backward(dl, h, w, grad_weight=gw0.clone() if accumulate else None,
                                       grad_bias=gb0.clone() if accumulate else None,
                                       accumulate=accumulate)
    assert torch.equal(dh, dh2) and torch.equal(gw, gw2) and torch.equal(gb, gb2)  # deterministic
