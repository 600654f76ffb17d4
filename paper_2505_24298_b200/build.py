"""Build libareal_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch build).

    python -m paper_2505_24298_b200.build [--verbose]

The shared library links the CUDA runtime dynamically (``-cudart shared``) so
that, inside a process that already imported torch, it binds to the same
``libcudart.so.12`` instance (and therefore the same current device / streams).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB_NAME = "libareal_b200.so"
LIB_PATH = os.path.join(HERE, LIB_NAME)
SOURCES = ["ppo_kernels.cu", "advantages.cu", "microbatch.cu", "adam.cu", "linear_lp.cu", "lm_head.cu", "emission.cu", "capi.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libareal_b200.so")


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if not f.endswith(".c")]
    deps.append(os.path.join(ROOT, "include", "areal_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps)


PACKER_SRC = os.path.join(CSRC, "packer.c")


def packer_path() -> str:
    import sysconfig
    return os.path.join(HERE, "_packer" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_packer(force: bool = False) -> str:
    """gcc -> the CPython extension _packer (host-side rollout packing, no CUDA)."""
    import sysconfig
    out = packer_path()
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(PACKER_SRC):
        return out
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        raise RuntimeError("gcc not found; needed for the native rollout packer")
    cmd = [cc, "-O3", "-shared", "-fPIC", "-Wall", "-Wno-unused-label",
           "-I", sysconfig.get_paths()["include"], PACKER_SRC, "-o", out + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"gcc failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    os.replace(out + ".tmp", out)
    return out


def build(verbose: bool = False, force: bool = False, extra_flags=(), out: str | None = None) -> str:
    """Compile every translation unit in parallel (one nvcc per source), then link."""
    from concurrent.futures import ThreadPoolExecutor
    import tempfile
    build_packer(force=force)
    out = out or LIB_PATH
    if out == LIB_PATH and not force and not _stale():
        return LIB_PATH
    nvcc = nvcc_path()
    common = [*ARCH, "-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr",
              "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), *extra_flags]
    if verbose:
        common += ["-Xptxas", "-v"]
    tmpdir = tempfile.mkdtemp(prefix="areal_build_")

    def compile_one(src):
        obj = os.path.join(tmpdir, os.path.splitext(src)[0] + ".o")
        cmd = [nvcc, *common, "-c", os.path.join(CSRC, src), "-o", obj]
        return cmd, subprocess.run(cmd, capture_output=True, text=True), obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    logs = []
    for cmd, res, _ in results:
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
        logs.append(res.stdout + res.stderr)
    tmp = out + ".tmp"
    link = [nvcc, *ARCH, "-shared", "-cudart", "shared", "-Xlinker", "-rpath,/usr/local/cuda/lib64",
            *[obj for _, _, obj in results], "-o", tmp]
    res = subprocess.run(link, capture_output=True, text=True)
    shutil.rmtree(tmpdir, ignore_errors=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({res.returncode}):\n{' '.join(link)}\n{res.stdout}\n{res.stderr}")
    if verbose:
        sys.stderr.write("".join(logs))
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force=True))
