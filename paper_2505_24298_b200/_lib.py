"""ctypes binding of libareal_b200.so (the C-ABI in include/areal_b200.h).

There is no fallback: if the library is missing or a call fails, an exception
is raised.  ``import torch`` happens first so the library's dynamic
``libcudart.so.12`` dependency binds to the runtime torch already loaded.
"""
from __future__ import annotations

import ctypes
import os

import torch  # noqa: F401  (load torch's CUDA runtime before the library)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libareal_b200.so")

ABI_VERSION = 1
N_STATS = 8
WORKSPACE_BYTES = 1 << 20
MAX_ITEMS_PER_MINIBATCH = 8192

# status codes (areal_status_t)
OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_BAD_DTYPE = 2
ERR_BAD_SHAPE = 3
ERR_MISALIGNED = 4
ERR_LEN_NONPOSITIVE = 5
ERR_LEN_EXCEEDS_CAPACITY = 6
ERR_MIN_GROUPS = 7
ERR_WORKSPACE = 8
ERR_CUDA = 9
ERR_UNSUPPORTED = 10
ERR_BAD_CLIP_EPS = 11

DTYPE_CODES = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2, torch.float64: 3}
ALGO_CODES = {"auto": 0, "warp": 1, "ring": 2}

c_i32, c_i64, c_f64, c_sz, c_vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_double,
                                   ctypes.c_size_t, ctypes.c_void_p)


class PpoParams(ctypes.Structure):
    """areal_ppo_params_t"""
    _fields_ = [("clip_eps", c_f64), ("behav_weight_cap", c_f64), ("grad_scale", c_f64),
                ("decoupled", c_i32), ("eta_mask", c_i32), ("current_version", c_i32),
                ("algo", c_i32), ("prox_from_lp", c_i32)]


class AdvParams(ctypes.Structure):
    """areal_adv_params_t"""
    _fields_ = [("gamma", c_f64), ("lam", c_f64), ("eps", c_f64), ("mode", c_i32),
                ("norm", c_i32)]


class AdamTensor(ctypes.Structure):
    """areal_adam_tensor_t"""
    _fields_ = [("param", c_vp), ("grad", c_vp), ("exp_avg", c_vp), ("exp_avg_sq", c_vp),
                ("numel", c_i64)]


class AdamParams(ctypes.Structure):
    """areal_adam_params_t"""
    _fields_ = [("lr", c_f64), ("beta1", c_f64), ("beta2", c_f64), ("eps", c_f64),
                ("weight_decay", c_f64), ("clip_norm", c_f64), ("one_minus_beta1", c_f64),
                ("one_minus_beta2", c_f64), ("bias_correction1", c_f64),
                ("bias_correction2", c_f64), ("grad_scale", c_f64), ("exact_norm", c_i32),
                ("grad_scale_divisor", c_vp)]


ADAM_MAX_TENSORS = 32

# areal_tune_t (kernel-selection overrides; -1 = the shipped rule)
TUNE_KNOBS = {"k2_cluster_size": 0, "k2_tmem": 1, "k2_tmem_stream": 2, "k2_tmem_unaligned": 3,
              "k1_ring_unaligned": 4, "k2_small_rowcta_kb": 5, "rowcta": 6, "k7_nt": 7,
              "k7_group": 8, "k1_cluster_size": 9, "lmh_group_m": 10}
TUNE_DEFAULT = -1

LMH_OPS = {"logits": 0, "dhidden": 1, "dweight": 2}  # areal_lmh_op_t

_SIGS = {
    "areal_abi_version": ([], c_i32),
    "areal_status_string": ([ctypes.c_int], ctypes.c_char_p),
    "areal_workspace_bytes": ([], c_sz),
    "areal_set_tuning": ([ctypes.c_int, c_i64], ctypes.c_int),
    "areal_get_tuning": ([ctypes.c_int, ctypes.POINTER(c_i64)], ctypes.c_int),
    "areal_logprob_fwd": ([c_vp, c_i64, ctypes.c_int, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp,
                           ctypes.c_int, c_vp, c_sz, c_vp], ctypes.c_int),
    "areal_ppo_fwd_bwd": ([c_vp, c_i64, c_vp, c_i64, ctypes.c_int, c_i64, c_i64, c_vp, c_vp,
                           c_vp, c_vp, c_vp, c_vp, ctypes.POINTER(PpoParams), c_vp, c_vp, c_vp,
                           c_vp, c_sz, c_vp], ctypes.c_int),
    "areal_advantages": ([c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_i32,
                          ctypes.POINTER(AdvParams), c_vp, c_vp, c_vp, c_vp, c_sz, c_vp],
                         ctypes.c_int),
    "areal_plan_microbatches": ([c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i64, c_i32,
                                 c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
                                ctypes.c_int),
    "areal_fill_gather": ([c_vp, c_vp, c_vp, c_i32, c_i64, c_vp, c_vp, c_vp], ctypes.c_int),
    "areal_linear_logprob_scratch_bytes": ([c_i64, c_i64], c_sz),
    "areal_linear_logprob_fwd": ([c_vp, c_i64, c_vp, c_i64, c_vp, ctypes.c_int, c_i64, c_i64, c_i64,
                                  c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, ctypes.c_int, c_vp],
                                 ctypes.c_int),
    "areal_lm_head_gemm": ([ctypes.c_int, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64,
                            c_vp, ctypes.c_int, ctypes.c_int, c_vp], ctypes.c_int),
    "areal_lm_head_backward": ([c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64,
                                c_vp, c_i64, c_vp, ctypes.c_int, ctypes.c_int, c_vp], ctypes.c_int),
    "areal_colsum_scratch_bytes": ([c_i64, c_i64], c_sz),
    "areal_colsum": ([c_vp, c_i64, c_i64, c_i64, ctypes.c_int, c_vp, ctypes.c_int, c_vp, c_sz, c_vp],
                     ctypes.c_int),
    "areal_emission_append": ([c_vp, c_vp, c_i64, c_vp, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp,
                               c_vp, c_vp], ctypes.c_int),
    "areal_adam_step": ([ctypes.POINTER(AdamTensor), c_i32, ctypes.c_int, ctypes.c_int,
                         ctypes.POINTER(AdamParams), c_vp, c_vp, c_sz, c_vp], ctypes.c_int),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_LIB = None


class ArealError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {status_string(status)} (status {status})")


def use_library(path: str) -> None:
    """Select a non-default build (tools/variants.py tuning builds) before the first
    load(); the product path always loads the in-tree libareal_b200.so."""
    global LIB_PATH
    if _LIB is not None:
        raise RuntimeError("library already loaded from " + LIB_PATH)
    LIB_PATH = os.path.abspath(path)


def load() -> ctypes.CDLL:
    """Load (once) and type the library; raises ImportError if it is not built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2505_24298_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.areal_abi_version() != ABI_VERSION:
        raise ImportError(f"ABI mismatch: library {lib.areal_abi_version()} != {ABI_VERSION}")
    _LIB = lib
    return lib


def status_string(status: int) -> str:
    return load().areal_status_string(int(status)).decode()


def check(status: int, where: str) -> None:
    if status != OK:
        raise ArealError(status, where)
