"""CPU-only tests: the C-ABI library builds, loads and exports every declared symbol;
host-side logic (minibatch split, DP sharding, config validation) matches the
reference semantics; the data-parallel statistics exchange works across 2 ranks
(gloo, world_size 2)."""
import os
import re
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from conftest import ROOT
import oracle as O


def test_library_exports_every_header_symbol():
    from paper_2505_24298_b200.build import build
    from paper_2505_24298_b200 import _lib
    build()
    lib = _lib.load()
    with open(os.path.join(ROOT, "include", "areal_b200.h")) as f:
        decls = set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(areal_\w+)\(", f.read(), re.M))
    assert decls == set(_lib.EXPORTED_SYMBOLS), decls ^ set(_lib.EXPORTED_SYMBOLS)
    for name in decls:
        assert hasattr(lib, name), name
    assert lib.areal_abi_version() == _lib.ABI_VERSION
    assert lib.areal_workspace_bytes() == _lib.WORKSPACE_BYTES
    assert _lib.status_string(_lib.ERR_LEN_EXCEEDS_CAPACITY) == "sequence length exceeds capacity"


def test_library_validates_without_gpu():
    """Argument checks run on the host before any launch (no GPU needed)."""
    import ctypes
    from paper_2505_24298_b200 import _lib
    lib = _lib.load()
    p = _lib.PpoParams(1.5, 0.0, 1.0, 1, -1, 0, 0)
    rc = lib.areal_ppo_fwd_bwd(None, 16, None, 16, 0, 4, 16, None, None, None, None, None, None,
                               ctypes.byref(p), None, None, None, None, 0, None)
    assert rc == _lib.ERR_BAD_CLIP_EPS
    p.clip_eps = 0.2
    rc = lib.areal_ppo_fwd_bwd(None, 16, None, 16, 9, 4, 16, None, None, None, None, None, None,
                               ctypes.byref(p), None, None, None, None, 0, None)
    assert rc == _lib.ERR_BAD_DTYPE
    rc = lib.areal_plan_microbatches(None, None, None, None, 1, 1, 1, 10, 0, *([None] * 9))
    assert rc == _lib.ERR_MIN_GROUPS
    # zero rows is a no-op
    assert lib.areal_logprob_fwd(None, 16, 0, 0, 16, None, None, None, None, 0, None, 0, None) == 0
    # decoupled without prox is only legal with prox_from_lp (then the kernel would run)
    p2 = _lib.PpoParams(0.2, 0.0, 1.0, 1, -1, 0, 0, 0)
    rc = lib.areal_ppo_fwd_bwd(ctypes.c_void_p(16), 16, ctypes.c_void_p(16), 16, 0, 4, 16,
                               ctypes.c_void_p(16), ctypes.c_void_p(16), None, ctypes.c_void_p(16),
                               None, None, ctypes.byref(p2), None, None, ctypes.c_void_p(16),
                               None, 0, None)
    assert rc == _lib.ERR_INVALID_ARGUMENT
    # K6: dtype / tensor-count validation
    t = (_lib.AdamTensor * 1)()
    ap = _lib.AdamParams(1e-3, 0.9, 0.95, 1e-8, 0.0, 1.0, 0.1, 0.05, 0.1, 0.05, 1.0, 1, None)
    ws = ctypes.create_string_buffer(_lib.WORKSPACE_BYTES)
    assert lib.areal_adam_step(t, 1, 0, 0, ctypes.byref(ap), None, ws, _lib.WORKSPACE_BYTES,
                               None) == _lib.ERR_UNSUPPORTED  # exact norm needs fp64
    assert lib.areal_adam_step(t, 33, 3, 3, ctypes.byref(ap), None, ws, _lib.WORKSPACE_BYTES,
                               None) == _lib.ERR_INVALID_ARGUMENT
    # K7: shape / alignment / dtype validation
    assert lib.areal_linear_logprob_fwd(ctypes.c_void_p(256), 100, ctypes.c_void_p(256), 100,
                                        None, 1, 4, 1000, 100, ctypes.c_void_p(256), None,
                                        ctypes.c_void_p(256), None, None, 0, 0, None) \
        == _lib.ERR_UNSUPPORTED  # dim % 64 != 0
    assert lib.areal_linear_logprob_fwd(ctypes.c_void_p(256), 128, ctypes.c_void_p(256), 128,
                                        None, 0, 4, 1000, 128, ctypes.c_void_p(256), None,
                                        ctypes.c_void_p(256), None, None, 0, 0, None) \
        == _lib.ERR_BAD_DTYPE  # fp32 operands
    assert lib.areal_linear_logprob_scratch_bytes(1000, 151936) == 1000 * 149 * 2 * 16


def test_tuning_api_validates_and_restores():
    """Kernel-selection overrides go through areal_set_tuning (nothing is read from the
    environment); bad knobs / values are rejected; the scoped helper restores defaults."""
    from paper_2505_24298_b200 import _lib, kernels as K
    with open(os.path.join(ROOT, "include", "areal_b200.h")) as f:
        hdr = f.read()
    for name, code in _lib.TUNE_KNOBS.items():
        assert re.search(rf"AREAL_TUNE_{name.upper()}\s*=\s*{code},", hdr), name
    for src in ("ppo_kernels.cu", "linear_lp.cu", "ppo_ring.cuh", "ppo_tmem.cuh", "capi.cu"):
        with open(os.path.join(ROOT, "paper_2505_24298_b200", "csrc", src)) as f:
            assert "getenv" not in f.read(), src
    with pytest.raises(ValueError):
        K.set_tuning("no_such_knob", 1)
    with pytest.raises(_lib.ArealError):
        K.set_tuning("k2_cluster_size", 3)
    with pytest.raises(_lib.ArealError):
        K.set_tuning("k7_group", 0)
    assert _lib.load().areal_set_tuning(99, 0) == _lib.ERR_INVALID_ARGUMENT
    with K.tuning(k2_tmem=0, k7_nt=4):
        assert K.set_tuning("k2_tmem", 0) == 0
        assert K.set_tuning("k7_nt", 4) == 4
    assert K.set_tuning("k2_tmem", -1) == -1 and K.set_tuning("k7_nt", -1) == -1


def test_minibatch_items_matches_reference_split():
    from paper_2505_24298_b200.trainer import minibatch_items
    rng = np.random.default_rng(3)
    for _ in range(200):
        n = int(rng.integers(0, 40))
        lengths = rng.integers(0, 5, size=n)
        bounds = np.concatenate([[0], np.cumsum(lengths)])
        k = int(rng.integers(1, 7))
        ref = [mb["traj_ids"] for mb in O.train_step_plan(bounds, k, 1000, 1)]
        assert minibatch_items(bounds, k) == ref


def test_lpt_assign_balanced_and_deterministic():
    from paper_2505_24298_b200.hotpath import lpt_assign
    sizes = [32000, 31000, 9000, 8000, 7000, 100, 32768, 5]
    a = lpt_assign(sizes, 3)
    assert a == lpt_assign(sizes, 3)
    loads = [sum(s for s, r in zip(sizes, a) if r == k) for k in range(3)]
    assert max(loads) - min(loads) <= max(sizes)
    assert lpt_assign(sizes, 1) == [0] * len(sizes)


def test_configs_validate_like_reference():
    from paper_2505_24298_b200.hotpath import HotPathConfig
    from paper_2505_24298_b200.trainer import BatchError, TrainerConfig
    for bad in (dict(clip_eps=0.0), dict(clip_eps=1.0), dict(minibatches=0),
                dict(objective="x")):
        with pytest.raises(BatchError):
            TrainerConfig(**bad)
        with pytest.raises(BatchError):
            HotPathConfig(**bad)
    assert issubclass(BatchError, ValueError)


def _oracle_plan_layout(bounds, k, cap, kmin):
    """Oracle plan in the C-ABI layout (group_cu, n_groups, mb_offsets) + gathers."""
    plan = O.train_step_plan(bounds, k, cap, kmin)
    mb_offsets = np.concatenate([[0], np.cumsum([len(mb["traj_ids"]) for mb in plan])])
    group_cu = np.zeros(int(mb_offsets[-1]) + len(plan), dtype=np.int64)
    n_groups = []
    t = 0
    gathers = []
    for m, mb in enumerate(plan):
        base = int(mb_offsets[m]) + m
        n_groups.append(len(mb["groups"]))
        for g, idx in enumerate(mb["gather"]):
            group_cu[base + g] = t
            t += len(idx)
            gathers.append(idx)
        group_cu[base + len(mb["groups"])] = t
    return plan, group_cu, np.array(n_groups), mb_offsets, np.concatenate(gathers)


def _dp_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_24298_b200.hotpath import shard_micro_batches
        rng = np.random.default_rng(0)
        lengths = rng.integers(1, 40, size=24)
        bounds = np.concatenate([[0], np.cumsum(lengths)])
        T, V = int(bounds[-1]), 50
        x = rng.normal(0, 2, size=(T, V))
        tok = rng.integers(0, V, size=T)
        prox = O.token_logprobs(x, tok) + rng.normal(0, 0.05, size=T)
        behav = prox + rng.normal(0, 0.2, size=T)
        adv = O.compute_advantages_ref(rng.choice([5.0, -5.0], size=24), bounds)
        plan, group_cu, n_groups, mb_offsets, packed = _oracle_plan_layout(bounds, 2, 80, world)
        micro, mine = shard_micro_batches(group_cu, n_groups, mb_offsets, world, rank)
        out = []
        for m in range(len(plan)):
            st = torch.zeros(8, dtype=torch.float64)
            for g, lo, hi in mine[m]:
                idx = packed[lo:hi]
                st += torch.from_numpy(O.surrogate_terms(x[idx], tok[idx], behav[idx], prox[idx],
                                                         adv[idx], want_dlogits=False)["stats"])
            dist.all_reduce(st)  # the hot path's one collective
            full = O.surrogate_terms(np.concatenate([x[i] for i in plan[m]["gather"]]),
                                     np.concatenate([tok[i] for i in plan[m]["gather"]]),
                                     np.concatenate([behav[i] for i in plan[m]["gather"]]),
                                     np.concatenate([prox[i] for i in plan[m]["gather"]]),
                                     np.concatenate([adv[i] for i in plan[m]["gather"]]),
                                     want_dlogits=False)["stats"]
            out.append((st.numpy(), full, len(mine[m]), int(n_groups[m])))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_data_parallel_stats_allreduce_gloo_world2():
    world = 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for m in range(len(res[0])):
        a, full, mine0, ng = res[0][m]
        b, _, mine1, _ = res[1][m]
        assert np.array_equal(a, b)                     # every rank sees the same sums
        assert mine0 + mine1 == ng and mine0 >= 1 and mine1 >= 1  # k_min = world: both busy
        assert np.allclose(a, full, rtol=1e-12, atol=1e-12)
        assert a[1] == full[1] and a[7] == full[7]


def test_rank_upload_ranges_cover_exactly_the_rank_tokens():
    """DP e2e uploads only the per-token arrays of the trajectories in a rank's
    micro-batches (hotpath.own_token_ranges): over all ranks the ranges tile the
    non-empty trajectories exactly once, and each rank's ranges hold exactly the tokens
    its micro-batches pack.  The [M, world] load is identical on every rank."""
    from types import SimpleNamespace
    from paper_2505_24298_b200.hotpath import (DecoupledPPOStep, load_summary,
                                               shard_micro_batches)
    rng = np.random.default_rng(5)
    lengths = rng.integers(0, 90, size=60)
    bounds = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    for world in (1, 2, 3, 8):
        plan, group_cu, n_groups, mb_offsets, packed = _oracle_plan_layout(bounds, 3, 200, world)
        # group_seq_cu / packed_traj in the C-ABI layout
        gsc = np.zeros_like(group_cu, dtype=np.int32)
        ptraj, s = [], 0
        for m, mb in enumerate(plan):
            base = int(mb_offsets[m]) + m
            for g, grp in enumerate(mb["groups"]):
                gsc[base + g] = s
                ptraj.extend(mb["traj_ids"][j] for j in grp)
                s += len(grp)
            gsc[base + len(mb["groups"])] = s
        seen = np.zeros(int(bounds[-1]), dtype=np.int64)
        loads = []
        for rank in range(world):
            micro, mine, load = shard_micro_batches(group_cu, n_groups, mb_offsets, world, rank,
                                                    with_load=True)
            loads.append(load)
            sp = SimpleNamespace(mine=mine, host_seq=(gsc, np.array(ptraj, dtype=np.int32)),
                                 device_plan=SimpleNamespace(mb_offsets=mb_offsets))
            ro = SimpleNamespace(traj_bounds_host=bounds)
            ranges = DecoupledPPOStep.own_token_ranges(None, ro, sp)
            assert all(a[1] < b[0]  # sorted, disjoint and coalesced
                       for a, b in zip(ranges, ranges[1:]))
            mine_tokens = np.sort(np.concatenate([packed[lo:hi] for grp in mine
                                                  for _, lo, hi in grp] or [np.zeros(0, int)]))
            got = np.concatenate([np.arange(lo, hi) for lo, hi in ranges] or [np.zeros(0, int)])
            assert np.array_equal(np.sort(got), mine_tokens)
            seen[got] += 1
            assert int(load[:, rank].sum()) == len(mine_tokens)
        assert np.all(seen == 1)
        assert all(np.array_equal(loads[0], x) for x in loads)
        summ = load_summary(loads[0])
        assert sum(summ["rank_tokens"]) == int(bounds[-1])
        assert 0 < summ["efficiency_bound"] <= 1.0 and summ["max_over_mean"] >= 1.0
