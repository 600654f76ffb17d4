"""Host packing throughput: native packer (csrc/packer.c) vs the Python flattening of
build_train_batch (trainer.py:91-111) at the cfg2 batch shape (512 rollouts, lengths
U[128, 8192]).  CPU only.  python tools/pack_bench.py"""
import json, os, sys, time
from types import SimpleNamespace
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2505_24298_b200.build import build_packer

build_packer()
from paper_2505_24298_b200 import _packer as P  # noqa: E402

rng = np.random.default_rng(0)
lengths = rng.integers(128, 8193, size=512)
trajs = [SimpleNamespace(trajectory_id=k, prompt=SimpleNamespace(id=k // 4),
                         tokens=rng.integers(0, 151936, size=m).tolist(),
                         behavior_logprobs=rng.normal(-2, 1, size=m).tolist(),
                         versions=[100] * m, reward=SimpleNamespace(reward=5.0))
         for k, m in enumerate(lengths)]
T = int(lengths.sum())

t0 = time.perf_counter()
tok, beh, ver, bnd = [], [], [], [0]
for t in trajs:
    tok.extend(t.tokens); beh.extend(t.behavior_logprobs); ver.extend(t.versions); bnd.append(len(tok))
a = (np.array(tok, np.int64), np.array(beh), np.array(ver, np.int32), np.array(bnd, np.int64))
py = time.perf_counter() - t0

bufs = (np.empty(T, np.int64), np.empty(T), np.empty(T, np.int32), np.empty(513, np.int64), np.empty(512))
t0 = time.perf_counter()
P.count(trajs)
P.fill(trajs, *(b.ctypes.data for b in bufs), T)
nat = time.perf_counter() - t0
assert np.array_equal(bufs[0], a[0]) and np.array_equal(bufs[1], a[1])
print(json.dumps(dict(tokens=T, python_s=py, native_s=nat, speedup=py / nat,
                      native_tokens_per_s=T / nat)))
