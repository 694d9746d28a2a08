"""The C ABI surface of libhbgpu.so, checked without a GPU.

* every function include/hbgpu.h declares is exported by the library and
  bound by paper_1304_7654_b200.native (and nothing else is bound);
* the ctypes / numpy mirrors of the ABI structs have the library's own
  sizes and offsets;
* the product path refuses to run without a CUDA device (no CPU fallback).
"""

import ctypes
import os
import re

import pytest

from paper_1304_7654_b200 import native
from paper_1304_7654_b200.exceptions import NativeUnavailable

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(REPO, "include", h) for h in ("hbgpu.h", "hbns.h")]


def declared_functions():
    names = []
    for header in HEADERS:
        text = open(header).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\**\s*(hb(?:gpu|ns)_[a-z_0-9]+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_header_functions_are_all_bound():
    decl = declared_functions()
    assert len(decl) >= 20
    assert sorted(native.SIGNATURES) == decl


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(native.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing


def test_abi_struct_layout_matches_library():
    assert native.abi_layout_native() == native.abi_layout_python()
    assert native.load().hbgpu_abi_version() == native.ABI_VERSION


def test_launch_counter_starts_at_zero_without_gpu_work():
    assert native.launch_count() >= 0


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(NativeUnavailable):
        native.require_cuda()
    from paper_1304_7654_b200 import RunSpec, run_case, tc_tiny
    with pytest.raises(NativeUnavailable):
        run_case(RunSpec(case=tc_tiny(), ranks=1, iterations=1))


def test_sm100a_cubin_present():
    """The library carries sm_100a SASS (cuobjdump lists the stage kernels)."""
    import shutil
    import subprocess
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-lelf", native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", native.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass          # tensor TMA loads in the stage kernel
    assert "UTMASTG" in sass          # tensor TMA stores (update stages, pass B)
    assert "SYNCS" in sass            # mbarrier pipeline
    assert "pair_tma_kernel" in sass and "band_kernel" in sass   # paired-stage schedule
    # no fused multiply-adds in the reference-rounded arithmetic: the only
    # DFMAs are the residual-norm partials (P per row of the first stage)
    assert sass.count("DMUL") > sass.count("DFMA")
