"""ctypes binding of libhbgpu.so (include/hbgpu.h).

The library is the only compute path: if it is missing, or no CUDA device is
visible, every entry point raises NativeUnavailable -- there is no CPU
fallback.  Structures here mirror the C header byte for byte (checked by
tests/test_native_abi.py against the compiled library's own sizes).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .exceptions import NativeUnavailable

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# HBGPU_LIB selects another build of the library (A/B measurements)
LIB_PATH = os.environ.get("HBGPU_LIB") or os.path.join(PKG_DIR, "libhbgpu.so")

NPDE = 4
MAX_TEMPLATED_P = 17
MAX_P = 127
MAX_PAIR_P = 9                # paired-stage kernel (HBGPU_MAX_PAIR_P)
ROW_LEAD = 7
STRIP = 64
TILE_WARPS = 8                # consumer warps per stage tile
TILE_COLS = {4: 64, 1: 256}   # tile_pdes -> interior columns per strip
ABI_VERSION = 2
# status keys (include/hbgpu.h): (gstage << STATUS_LIN_BITS) | lin, HAZARD_BIT for |v| >= 2^1022
STATUS_LIN_BITS = 40
HAZARD_BIT = 1 << 39
REDUCE_SUM_F64, REDUCE_MIN_U64 = 0, 1
TMAP_SETS = 10                 # tensor-map sets per block (hbgpu_encode_tensor_maps)

c_i32, c_i64, c_f64, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p

# ---- device table dtypes (C structs stored in device arrays) ---------------

BLOCK_DTYPE = np.dtype([
    ("base", "<i8"), ("ps", "<i8"), ("rs", "<i8"), ("ni", "<i4"), ("nj", "<i4"), ("pitch", "<i4"),
    ("gid", "<i4"), ("tiles_i", "<i4"), ("tiles_j", "<i4"), ("tile_begin", "<i4"),
    ("ntiles", "<i4"), ("sxy_pitch", "<i4"), ("pad0", "<i4"), ("nu_h2", "<f8"),
    ("adv_2h", "<f8"), ("h", "<f8"),
    ("sxy_off", "<i8"), ("face_off", "<i8", (4,))], align=True)

FACE_TARGET_DTYPE = np.dtype([("off", "<i8"), ("ps", "<i8")], align=True)

HALO_DIR_DTYPE = np.dtype([
    ("src_off", "<i8"), ("src_es", "<i8"), ("src_vs", "<i8"),
    ("dst_off", "<i8"), ("dst_es", "<i8"), ("dst_vs", "<i8"),
    ("length", "<i4"), ("src_kind", "<i4"), ("dst_kind", "<i4"), ("flags", "<i4")], align=True)
HALO_SECTOR_DST = 1

BAND_SEG_DTYPE = np.dtype([
    ("block", "<i4"), ("dir", "<i4"), ("j", "<i4"), ("i", "<i4"), ("len", "<i4"), ("pad", "<i4")])

OUT_RECORD_DTYPE = np.dtype([
    ("block", "<i4"), ("plane", "<i4"), ("kind", "<i4"), ("pad", "<i4"),
    ("dst", "<i8"), ("xy", "<i8")], align=True)
RECORD_RESTART, RECORD_FLOWTEC = 0, 1

FORCE_SEG_DTYPE = np.dtype([
    ("start", "<i8"), ("stride", "<i8"), ("ps", "<i8"), ("length", "<i4"),
    ("body", "<i4"), ("h", "<f8")], align=True)


class PeerMsg(ctypes.Structure):
    _fields_ = [("peer", c_i32), ("pad", c_i32), ("offset", c_i64), ("count", c_i64)]


class StageArgs(ctypes.Structure):
    _fields_ = [
        ("in_", c_vp), ("q0", c_vp), ("out", c_vp), ("band", c_vp), ("sendbuf", c_vp),
        ("blocks", c_vp), ("tile_block", c_vp), ("sxy", c_vp), ("faces", c_vp),
        ("norm_part", c_vp), ("status", c_vp), ("iter", c_vp), ("dmat", c_vp), ("tmaps", c_vp),
        ("nblocks", c_i32), ("total_tiles", c_i32), ("planes", c_i32), ("stage", c_i32),
        ("tile_rows", c_i32), ("in_slot", c_i32), ("interleaved", c_i32), ("tile_pdes", c_i32),
        ("out_slot", c_i32), ("pair", c_i32), ("coef", c_f64), ("coef2", c_f64),
        ("band_segs", c_vp), ("nband_segs", c_i32), ("band_max_len", c_i32),
        ("edge_q0", c_vp),
        ("tile_order", c_vp), ("tile_lo", c_i32), ("tile_hi", c_i32),
        ("D", c_f64 * (MAX_TEMPLATED_P * MAX_TEMPLATED_P)),
        ("ap", c_f64 * (MAX_P * NPDE))]


class EngineDesc(ctypes.Structure):
    _fields_ = [
        ("slot", c_vp * 3), ("sendbuf", c_vp), ("recvbuf", c_vp),
        ("blocks", c_vp), ("tile_block", c_vp), ("sxy", c_vp), ("faces", c_vp), ("dmat", c_vp),
        ("norm_part", c_vp), ("sumsq", c_vp), ("status", c_vp), ("iter", c_vp),
        ("prime_dirs", c_vp), ("nprime", c_i32), ("prime_max_len", c_i32),
        ("unpack_dirs", c_vp), ("nunpack", c_i32), ("unpack_max_len", c_i32),
        ("post_dirs", c_vp), ("npost", c_i32), ("post_max_len", c_i32),
        ("band_segs", c_vp), ("nband_segs", c_i32), ("band_max_len", c_i32),
        ("fused", c_i32), ("small", c_i32), ("edge_q0", c_vp),
        ("tile_order", c_vp), ("nbound_tiles", c_i32), ("prime_remote", c_i32), ("post_remote", c_i32),
        ("small_max_cells", c_i32),
        ("segs", c_vp), ("nsegs", c_i32),
        ("force_hist", c_vp),
        ("sends", ctypes.POINTER(PeerMsg)), ("nsends", c_i32),
        ("recvs", ctypes.POINTER(PeerMsg)), ("nrecvs", c_i32),
        ("comm", c_vp), ("tmaps", c_vp),
        ("nblocks", c_i32), ("total_tiles", c_i32), ("planes", c_i32), ("nbody", c_i32),
        ("tile_rows", c_i32), ("max_iters", c_i32), ("interleaved", c_i32), ("tile_pdes", c_i32),
        ("coef", c_f64 * 4),
        ("D", c_f64 * (MAX_TEMPLATED_P * MAX_TEMPLATED_P)),
        ("ap", c_f64 * (MAX_P * NPDE))]


# name -> (restype, argtypes); the full exported surface of include/hbgpu.h
SIGNATURES = {
    "hbgpu_residual": (c_i32, [c_vp, c_vp, c_vp, c_f64, c_f64, c_vp] + [c_i64] * 8 + [c_vp]),
    "hbgpu_update": (c_i32, [c_vp, c_vp, c_vp, c_f64, c_i32] + [c_i64] * 8 + [c_vp, c_vp]),
    "hbgpu_first_nonfinite": (c_i32, [c_vp] + [c_i64] * 4 + [c_vp, c_vp]),
    "hbgpu_stage": (c_i32, [ctypes.POINTER(StageArgs), c_vp]),
    "hbgpu_band": (c_i32, [ctypes.POINTER(StageArgs), c_vp]),
    "hbgpu_stage_prepare": (c_i32, [c_i32]),
    "hbgpu_stage_first_forwards": (c_i32, [c_i32]),
    "hbgpu_encode_tensor_maps": (c_i32, [c_vp * 3, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_i64]),
    "hbgpu_halo": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp]),
    "hbgpu_hazard_scan": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_vp, c_vp]),
    "hbgpu_norm_fold": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp]),
    "hbgpu_forces": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_i32, c_vp]),
    "hbgpu_ordered_fold": (c_i32, [c_vp, c_i32, c_i64, c_vp, c_vp]),
    "hbgpu_pack_records": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "hbgpu_engine_create": (c_i32, [ctypes.POINTER(EngineDesc), ctypes.POINTER(c_vp)]),
    "hbgpu_engine_prime": (c_i32, [c_vp, c_vp]),
    "hbgpu_engine_iterate": (c_i32, [c_vp, c_i32, c_i32, c_vp]),
    "hbgpu_engine_launches_per_iteration": (c_i32, [c_vp]),
    "hbgpu_engine_iterations_done": (c_i32, [c_vp]),
    "hbgpu_engine_rewind": (c_i32, [c_vp, c_vp]),
    "hbgpu_engine_step": (c_i32, [c_vp, c_i32, c_vp]),
    "hbgpu_engine_unpack": (c_i32, [c_vp, c_i32, c_vp]),
    "hbgpu_engine_step_split": (c_i32, [c_vp, c_i32, c_i32, c_vp]),
    "hbgpu_engine_destroy": (c_i32, [c_vp]),
    "hbgpu_comm_unique_id": (c_i32, [ctypes.c_char_p]),
    "hbgpu_comm_init": (c_i32, [ctypes.c_char_p, c_i32, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "hbgpu_comm_allgather": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "hbgpu_comm_destroy": (c_i32, [c_vp]),
    "hbgpu_comm_allreduce": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp]),
    "hbgpu_comm_async_error": (c_i32, [c_vp]),
    "hbgpu_comm_exchange": (c_i32, [c_vp, c_vp, ctypes.POINTER(PeerMsg), c_i32, c_vp, ctypes.POINTER(PeerMsg),
                                    c_i32, c_vp]),
    "hbgpu_comm_abort": (c_i32, [c_vp]),
    "hbgpu_norm_totals": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_vp]),
    "hbns_boundaries": (c_i32, [c_vp, c_i32, c_vp]),
    "hbns_stage": (c_i32, [c_vp, c_i32, c_i32, c_f64, c_i32, c_i32, c_vp]),
    "hbns_forces": (c_i32, [c_vp, c_i32, c_vp]),
    "hbns_wall_fold": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "hbgpu_abi_version": (c_i32, []),
    "hbgpu_last_error": (ctypes.c_char_p, []),
    "hbgpu_launch_count": (ctypes.c_uint64, []),
    "hbgpu_abi_layout": (c_i32, [ctypes.POINTER(c_i64), c_i32]),
}

_lib = None


def load(path=LIB_PATH):
    """Load libhbgpu.so and bind its C ABI (no GPU needed to load)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.hbgpu_abi_version() != ABI_VERSION:
        raise NativeUnavailable(f"libhbgpu ABI {lib.hbgpu_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


def abi_layout_python():
    """The same numbers hbgpu_abi_layout reports, from the Python mirrors."""
    return [BLOCK_DTYPE.itemsize, FACE_TARGET_DTYPE.itemsize, HALO_DIR_DTYPE.itemsize,
            FORCE_SEG_DTYPE.itemsize, ctypes.sizeof(PeerMsg), ctypes.sizeof(StageArgs),
            ctypes.sizeof(EngineDesc), EngineDesc.coef.offset, StageArgs.coef.offset,
            OUT_RECORD_DTYPE.itemsize]


def abi_layout_native():
    out = (c_i64 * 16)()
    k = load().hbgpu_abi_layout(out, 16)
    return list(out[:k])


def check(rc, what):
    if rc != 0:
        msg = load().hbgpu_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed (status {rc}): {msg}")


def require_cuda():
    """The product path runs on a CUDA device or not at all."""
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible: the HB solver has no CPU path")
    return load()


def launch_count():
    return int(load().hbgpu_launch_count())
