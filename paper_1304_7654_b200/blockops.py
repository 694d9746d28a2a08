"""Kernel-level drop-ins for the reference's solver-core block API.

Mirrors hbcore.BlockState / HarmonicField / residual_into / residual /
update_stage / exchange_halos / compute_forces (reference hbcore.py:115-382,
exchange.py:382-402) on CUDA tensors in the reference's dense layout
(planes, npde, nj+2, ni+2), calling libhbgpu's C ABI:

  residual_into  -> hbgpu_residual      (hbcore._residual_kernel, hbcore.py:184-221)
  update_stage   -> hbgpu_update        (hbcore._update_kernel, hbcore.py:224-245)
                    + hbgpu_first_nonfinite for the DivergenceError location
  exchange_halos -> hbgpu_halo          (exchange.py:295-316, all cuts local)
  compute_forces -> hbgpu_forces        (hbcore.py:359-382)

Sub-range bounds are the reference's array coordinates.  Results are bitwise
the reference's.  The fused production path is solver.run_case; these exist
so code written against the reference's block API can move to the GPU
piecewise, and so each kernel can be checked in isolation.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import hbop, native
from .exceptions import DivergenceError
from .solver import ForceCoefficients

NO_BAD = (1 << 64) - 1


def _vp(t):
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class BlockState:
    """One block's arrays on the device (views into its HarmonicField's pools)."""

    def __init__(self, spec, planes, npde=4, q=None, q0=None, device=None):
        import torch
        native.require_cuda()
        self.spec, self.planes, self.npde = spec, planes, npde
        shape = (planes, npde, spec.nj + 2, spec.ni + 2)
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.q = q if q is not None else torch.zeros(shape, dtype=torch.float64, device=dev)
        self.q0 = q0 if q0 is not None else torch.zeros(shape, dtype=torch.float64, device=dev)
        self.resid = torch.zeros((planes, npde, spec.nj, spec.ni), dtype=torch.float64, device=dev)
        self.forcing = torch.from_numpy(hbop.forcing_values(spec, planes, npde)).to(dev)
        self.first_bad = torch.full((1,), -1, dtype=torch.int64, device=dev)

    def interior(self):
        return self.q[:, :, 1:self.spec.nj + 1, 1:self.spec.ni + 1]


class HarmonicField:
    """The rank-local field: every block's q in one pool (halo moves address
    all blocks through one base pointer)."""

    def __init__(self, planes, npde, blocks, pool, offsets):
        self.planes, self.npde, self.blocks = planes, npde, blocks
        self.pool, self.offsets = pool, offsets

    @classmethod
    def allocate(cls, specs, planes, npde=4):
        import torch
        native.require_cuda()
        specs = sorted(specs, key=lambda s: s.id)
        sizes = [planes * npde * (s.nj + 2) * (s.ni + 2) for s in specs]
        pool = torch.zeros(sum(sizes), dtype=torch.float64, device="cuda")
        blocks, offsets, off = {}, {}, 0
        for s, n in zip(specs, sizes):
            q = pool[off:off + n].view(planes, npde, s.nj + 2, s.ni + 2)
            blocks[s.id] = BlockState(s, planes, npde, q=q)
            offsets[s.id] = off
            off += n
        return cls(planes, npde, blocks, pool, offsets)


def residual_into(block, deriv, n_lo, n_hi, j_lo, j_hi):
    """block.resid[n_lo:n_hi, :, j_lo-1:j_hi-1] <- R(block.q) (hbcore.py:248-258)."""
    import torch
    h = block.spec.h
    nu_h2, adv_2h = hbop.stencil_coefficients(h)
    dmat = torch.from_numpy(np.array(deriv.matrix, dtype=np.float64)).to(block.q.device)
    P, npde, nj2, ni2 = block.q.shape
    native.check(native.load().hbgpu_residual(_vp(block.q), _vp(dmat), _vp(block.forcing), nu_h2, adv_2h,
                                              _vp(block.resid), P, npde, nj2, ni2, n_lo, n_hi, j_lo, j_hi,
                                              _stream()), "hbgpu_residual")


def residual(block, deriv):
    """Full-interior residual of one block, returned as a host array."""
    residual_into(block, deriv, 0, block.planes, 1, block.spec.nj + 1)
    return block.resid.cpu().numpy()


def update_stage(block, alpha_dtau, n_lo, n_hi, j_lo, j_hi, snapshot=False):
    """q <- q0 - alpha*dtau*R over a sub-range; DivergenceError on non-finite
    values with the reference's location rule (hbcore.py:267-284)."""
    P, npde, nj2, ni2 = block.q.shape
    lib = native.load()
    block.first_bad.fill_(-1)
    bad_ptr = _vp(block.first_bad)
    native.check(lib.hbgpu_update(_vp(block.q), _vp(block.q0), _vp(block.resid), alpha_dtau,
                                  int(bool(snapshot)), P, npde, nj2, ni2, n_lo, n_hi, j_lo, j_hi,
                                  bad_ptr, _stream()), "hbgpu_update")
    if int(block.first_bad.item()) != -1:
        _raise_divergence(block)


def _raise_divergence(block):
    P, npde, nj2, ni2 = block.q.shape
    block.first_bad.fill_(-1)
    native.check(native.load().hbgpu_first_nonfinite(_vp(block.q), P, npde, nj2, ni2,
                                                     _vp(block.first_bad), _stream()),
                 "hbgpu_first_nonfinite")
    lin = int(block.first_bad.cpu().numpy().view(np.uint64)[0])
    ni, nj = ni2 - 2, nj2 - 2
    i, j = lin % ni, (lin // ni) % nj
    npl = lin // (ni * nj)
    raise DivergenceError(block.spec.id, i + 1, j + 1, npl % npde, npl // npde)


def _face_cell(spec, face, k, halo):
    if face == "south":
        return (0 if halo else 1), k
    if face == "north":
        return (spec.nj + 1 if halo else spec.nj), k
    if face == "west":
        return k, (0 if halo else 1)
    return k, (spec.ni + 1 if halo else spec.ni)


def _dense_run(field, gid, face, first, reversed_, halo):
    b = field.blocks[gid]
    s = b.spec
    j, i = _face_cell(s, face, first, halo)
    nj2, ni2 = s.nj + 2, s.ni + 2
    step = 1 if face in ("south", "north") else ni2
    return field.offsets[gid] + j * ni2 + i, (-step if reversed_ else step), nj2 * ni2


def exchange_halos(field, plan):
    """One halo exchange of an all-local plan: every cut halo cell <- its paired
    interior cell (exchange.py:382-402)."""
    rows = []
    for d in plan.directions():
        if not d.local:
            raise NotImplementedError("remote cuts run through solver.run_case (NCCL engine)")
        s_off, s_es, s_vs = _dense_run(field, d.src_block, d.src_face, d.src_index(0),
                                       d.src_reversed, False)
        t_off, t_es, t_vs = _dense_run(field, d.dst_block, d.dst_face, d.dst_index(0),
                                       d.dst_reversed, True)
        rows.append((s_off, s_es, s_vs, t_off, t_es, t_vs, d.length, 0, 0, 0))
    if not rows:
        return
    import torch
    arr = np.array(rows, dtype=native.HALO_DIR_DTYPE)
    dirs = torch.from_numpy(arr.view(np.uint8).copy()).to(field.pool.device)
    native.check(native.load().hbgpu_halo(_vp(field.pool), None, None, _vp(dirs), len(rows),
                                          int(arr["length"].max()), field.planes, _stream()),
                 "hbgpu_halo")


def compute_forces(field, topology):
    """Rank-local force partials of the owned body faces (hbcore.py:359-382)."""
    import torch
    segs = []
    for gid in sorted(field.blocks):
        s = field.blocks[gid].spec
        for face, body in s.body_faces:
            off, step, ps = _dense_run(field, gid, face, 1, False, False)
            segs.append((off, step, ps, s.face_extent(face), body, s.h))
    P, nbody = field.planes, topology.nbody
    if nbody == 0:
        return ForceCoefficients.zeros(P, 0)
    dev = field.pool.device
    arr = np.array(segs, dtype=native.FORCE_SEG_DTYPE) if segs else np.zeros(1, native.FORCE_SEG_DTYPE)
    t_segs = torch.from_numpy(arr.view(np.uint8).copy()).to(dev)
    hist = torch.zeros(3 * P * nbody, dtype=torch.float64, device=dev)
    it = torch.zeros(1, dtype=torch.int32, device=dev)
    native.check(native.load().hbgpu_forces(_vp(field.pool), _vp(t_segs), len(segs), P, nbody, _vp(hist),
                                            _vp(it), 1, _stream()), "hbgpu_forces")
    return ForceCoefficients.from_stack(hist.cpu().numpy().reshape(3, P, nbody))
