"""Build libhbgpu.so (sm_100a) in-tree with nvcc.

The shared library is the product: it carries the fused stage kernel, the
halo / force / norm kernels, the C ABI of include/hbgpu.h and the per-rank
iteration engine.  No torch headers are involved: the ABI is plain C.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
LIB_PATH = os.path.join(PKG_DIR, "libhbgpu.so")

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-Xcompiler", "-fPIC",
              "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _nccl_include():
    for base in sys.path:
        cand = os.path.join(base, "nvidia", "nccl", "include")
        if os.path.exists(os.path.join(cand, "nccl.h")):
            return cand
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include"
    raise RuntimeError("nccl.h not found (venv nvidia/nccl/include or /usr/include)")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build():
    if not os.path.exists(LIB_PATH):
        return True
    stamp = os.path.getmtime(LIB_PATH)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(REPO_DIR, "include", "hbgpu.h")]
    return any(os.path.getmtime(p) > stamp for p in deps)


def build(force=False, verbose=False):
    """Compile every .cu under csrc/ into paper_1304_7654_b200/libhbgpu.so."""
    if not force and not needs_build():
        return LIB_PATH
    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = os.path.join(PKG_DIR, "build")
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(REPO_DIR, "include"), "-I", CSRC, "-I", _nccl_include()]
    # HBGPU_NVCC_EXTRA: extra flags for measurement builds (e.g. -D overrides)
    extra = os.environ.get("HBGPU_NVCC_EXTRA", "").split()

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc, *ARCH_FLAGS, *NVCC_FLAGS, *extra, *inc, "-c", src, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
        return obj, res.stdout + res.stderr

    # one nvcc per source, side by side (the template-heavy files take a minute each)
    with ThreadPoolExecutor(max_workers=min(len(sources()), os.cpu_count() or 1)) as pool:
        done = list(pool.map(compile_one, sources()))
    objs = [o for o, _ in done]
    logs = [l for _, l in done]
    tmp = LIB_PATH + ".tmp"
    cmd = [nvcc, *ARCH_FLAGS, "-shared", "-o", tmp, *objs, "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stderr}")
    os.replace(tmp, LIB_PATH)
    with open(os.path.join(objdir, "ptxas.log"), "w") as fh:
        fh.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return LIB_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
