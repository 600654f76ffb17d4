"""Randomised K1/K2 parity sweep (seeded, deterministic): vocab sizes across every
kernel path (row_warp / row_ring / cluster ring / TMEM), all logits dtypes, both
objectives, masks, row_index permutations, in-place backward, entropy on/off, and
injected NaN / +-inf / extreme logits — each case against the float64 oracle
(trainer.py:150-195 restated) at the tolerances of tests/parity.py: lp 1e-5 for every
dtype, dlogits on 100% of the elements, counters exact except identified clip-boundary
tokens."""
import numpy as np
import pytest
import torch

import oracle as O
import parity as PY

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2505_24298_b200 import kernels as K

DT = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}
VOCABS = [7, 100, 4097, 8192, 32000, 50257, 65536, 128256, 151936, 152064, 200003, 262144,
          151937, 16381, 98305]  # + unaligned TMEM / ring rows and a chunk-boundary case


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    dt = ["f32", "bf16", "f16"][(seed + seed // len(VOCABS)) % 3]  # every (V, dtype) pair
    V = int(VOCABS[seed % len(VOCABS)])
    if dt == "f32" and V > 160000:
        V = 65536
    T = int(rng.integers(1, 40))
    scale = float(rng.choice([0.5, 2.0, 6.0]))
    x = rng.normal(0, scale, size=(T, V))
    special = rng.integers(0, 4)
    if special == 1 and T > 2:
        x[0, rng.integers(0, V)] = np.inf       # +inf logit: lse = inf -> token excluded
    elif special == 2 and T > 2:
        x[1, rng.integers(0, V)] = np.nan       # NaN row
    elif special == 3:
        x[-1, : V // 3] -= 60.0                 # strongly skewed row (fixed-shift paths)
    logits = torch.as_tensor(x).to(DT[dt])
    x64 = logits.double().numpy()
    tokens = rng.integers(0, V, size=T)
    with np.errstate(invalid="ignore", over="ignore"):
        lp = O.token_logprobs(x64, tokens)
    lp = np.where(np.isfinite(lp), lp, -5.0)
    prox = lp + rng.normal(0, 0.1, size=T)
    behav = prox + rng.normal(0, 0.3, size=T)
    adv = rng.normal(0, 1, size=T)
    versions = rng.integers(90, 101, size=T).astype(np.int32)
    return dict(dt=dt, V=V, T=T, logits=logits, x64=x64, tokens=tokens, prox=prox, behav=behav,
                adv=adv, versions=versions, decoupled=bool(seed % 2 == 0),
                eta=int(rng.choice([-1, 3])), ent=bool(seed % 4 < 2), inplace=bool(seed % 5 == 0),
                permute=bool(seed % 3 == 1), special=int(special))


@pytest.mark.parametrize("seed", range(90))
def test_k1_k2_fuzz(seed):
    c = _case(seed)
    T, dt = c["T"], c["dt"]
    cu = lambda a, d=None: torch.as_tensor(a).to(d).cuda() if d else torch.as_tensor(a).cuda()
    # rows of the logits matrix map to global tokens through a permutation
    perm = np.random.default_rng(seed).permutation(T) if c["permute"] else np.arange(T)
    rows = c["logits"][perm]           # logits row r holds global token perm[r]
    ri = cu(perm.astype(np.int32)) if c["permute"] else None
    with np.errstate(invalid="ignore", over="ignore", divide="ignore"):
        ref = O.surrogate_terms(c["x64"], c["tokens"], c["behav"], c["prox"], c["adv"],
                                decoupled=c["decoupled"], versions=c["versions"],
                                current_version=100, eta_mask=c["eta"])
        ref_lp = O.token_logprobs(c["x64"], c["tokens"])
    lg = rows.cuda()
    lp = torch.zeros(T, dtype=torch.float64, device="cuda")
    ent = torch.zeros(T, dtype=torch.float64, device="cuda") if c["ent"] else None
    K.logprob_fwd(lg, cu(c["tokens"]), row_index=ri, lp_out=lp, entropy_out=ent,
                  with_entropy=c["ent"])
    got_lp = lp.cpu().numpy()
    # K1 computes in fp32 from the exact rounded inputs the oracle sees: 1e-5 for every dtype
    PY.check_lp(got_lp, ref_lp, what=f"K1 lp seed {seed}")
    if c["ent"]:
        with np.errstate(invalid="ignore", over="ignore"):
            ref_ent = O.token_entropy(c["x64"])
        fe = np.isfinite(ref_ent) & np.isfinite(ref_lp)  # the oracle's 0 log 0 := 0 also
        # turns rows with a NaN / +inf logit into H = 0; the kernels give NaN there
        err = np.abs(ent.cpu().numpy()[fe] - ref_ent[fe])
        assert np.all(err <= 1e-4 * (1.0 + np.abs(ref_ent[fe]))), float(err.max())
    dl = lg if c["inplace"] else None
    dl, st = K.ppo_fwd_bwd(lg, cu(c["tokens"]), cu(c["behav"]), cu(c["prox"]), cu(c["adv"]),
                           decoupled=c["decoupled"], versions=cu(c["versions"]),
                           current_version=100, eta_mask=c["eta"], row_index=ri, dlogits=dl)
    s = st.cpu().numpy()
    # counters exact; n_clipped may differ only by the identified clip-boundary tokens
    bnd = PY.boundary_tokens(ref, 0.2)
    PY.check_counters(s, ref["stats"], int(bnd.sum()), what=f"seed {seed}")
    # dlogits: 100% of the elements of every row (boundary rows excepted)
    got = dl.double().cpu().numpy()
    PY.check_dlogits(got, ref["dlogits"][perm], ref["coef"][perm], c["tokens"][perm], dt,
                     skip_rows=bnd[perm], what=f"K2 dlogits seed {seed} ({dt}, V={c['V']})")
