"""Small invocation of every kernel (K1-K8), for compute-sanitizer runs:
    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2505_24298_b200 import kernels as K

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
for V, dt, algo in ((151936, torch.bfloat16, "auto"), (32000, torch.float32, "auto"),
                    (1000, torch.bfloat16, "warp"), (152064, torch.bfloat16, "ring")):
    T = 300
    x = torch.randn(T, V, device=dev, generator=g).to(dt)
    tok = torch.randint(0, V, (T,), device=dev, generator=g)
    lp, ent = K.logprob_fwd(x, tok, algo=algo)
    beh = lp + 0.1
    adv = torch.randn(T, dtype=torch.float64, device=dev, generator=g)
    K.ppo_fwd_bwd(x, tok, beh, lp, adv, algo=algo, dlogits=x)
rng = np.random.default_rng(0)
lengths = rng.integers(1, 200, size=50)
bounds = torch.as_tensor(np.concatenate([[0], np.cumsum(lengths)]), device=dev)
T = int(bounds[-1])
rew = torch.randn(50, dtype=torch.float64, device=dev, generator=g)
K.advantages(rew, bounds, T)
K.advantages(rew, bounds, T, mode="gae", gamma=0.99, lam=0.95, norm="group",
             group_ids=torch.arange(50, dtype=torch.int32, device=dev) // 5)
items = torch.arange(50, dtype=torch.int32, device=dev)
plan = K.plan_microbatches(bounds, items, [0, 25, 50], [0, int(lengths[:25].sum())], 400, 2)
torch.cuda.synchronize()
K.fill_gather(bounds, plan, T)
ps = [torch.randn(1000, device=dev), torch.randn(7, device=dev)]
K.adam_step(ps, [p.clone() for p in ps], [torch.zeros_like(p) for p in ps],
            [torch.zeros_like(p) for p in ps], step=1, lr=1e-3, beta1=0.9, beta2=0.95,
            eps=1e-8, weight_decay=0.1, clip_norm=1.0)
pd = [torch.randn(100, 3, dtype=torch.float64, device=dev)]
K.adam_step(pd, [p.clone() for p in pd], [torch.zeros_like(p) for p in pd],
            [torch.zeros_like(p) for p in pd], step=1, lr=1e-3, beta1=0.9, beta2=0.95,
            eps=1e-8, weight_decay=0.1, clip_norm=1.0)
for cg in (1, 2):
    h = torch.randn(300, 256, device=dev, generator=g).to(torch.bfloat16)
    w = torch.randn(5000, 256, device=dev, generator=g).to(torch.bfloat16)
    tok = torch.randint(0, 5000, (300,), device=dev, generator=g)
    K.linear_logprob_fwd(h, w, tok, bias=torch.randn(5000, device=dev), with_entropy=True, cta_group=cg)
# LM-head GEMMs (K8): CTA-pair LOGITS, 2x2-cluster multicast DHIDDEN / DWEIGHT (+= through
# TMA reduce-add) and the grouped backward with the fused column sum
T, V, d = 600, 3000, 192
h = torch.randn(T, d, device=dev, generator=g).to(torch.bfloat16)
w = (torch.randn(V, d, device=dev, generator=g) / d ** 0.5).to(torch.bfloat16)
ldv = (V + 7) // 8 * 8
lg = torch.empty(T, ldv, device=dev, dtype=torch.bfloat16)[:, :V]
K.lm_head_gemm("logits", h, w, lg, bias=torch.randn(V, device=dev, generator=g))
dh = K.lm_head_gemm("dhidden", lg, w)
gw = K.lm_head_gemm("dweight", lg, h)
K.lm_head_gemm("dweight", lg, h, gw, accumulate=True)
K.lm_head_backward(lg, h, w, grad_weight=torch.zeros(V, d, device=dev),
                   grad_bias=torch.zeros(V, device=dev), accumulate=True)
K.colsum(lg)
torch.cuda.synchronize()
print("sanitize smoke ok")
