"""Kernel-level drop-ins for the reference's solver-core block API.

Mirrors hbcore.BlockState / HarmonicField / residual_into / residual /
update_stage / exchange_halos / compute_forces (reference hbcore.py:115-382,
exchange.py:382-402) on CUDA tensors in the reference's dense layout
(planes, npde, nj+2, ni+2), calling libhbgpu's C ABI:

  residual_into  -> hbgpu_residual      (hbcore._residual_kernel, hbcore.py:184-221)
  update_stage   -> hbgpu_update        (hbcore._update_kernel, hbcore.py:224-245)
                    + hbgpu_first_nonfinite for the DivergenceError location
  exchange_halos -> hbgpu_halo          (exchange.py:295-316: local copies, remote
                                         pack / unpack around a HaloContext transfer)
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


class HaloContext:
    """A rank's side of block-level halo exchange with remote cuts: its rank
    in the plan's partition and a transport for the per-peer payloads (the
    reference passes its RankContext, exchange.py:382-402 /
    runtime.py:196-309).

    comm: an NCCL communicator from solver.make_comm -> one grouped
    ncclSend/ncclRecv per peer on the current stream (hbgpu_comm_exchange);
    hub: a LoopbackHub shared by the ranks' threads of one process (device
    copies between their buffers)."""

    def __init__(self, rank, comm=None, hub=None):
        if (comm is None) == (hub is None):
            raise ValueError("HaloContext needs exactly one of comm or hub")
        self.rank, self.comm, self.hub = rank, comm, hub

    def transfer(self, sendbuf, sends, recvbuf, recvs):
        if self.comm is not None:
            snd = (native.PeerMsg * max(1, len(sends)))(*[native.PeerMsg(p, 0, o, c) for p, o, c in sends])
            rcv = (native.PeerMsg * max(1, len(recvs)))(*[native.PeerMsg(p, 0, o, c) for p, o, c in recvs])
            native.check(native.load().hbgpu_comm_exchange(self.comm, _vp(sendbuf), snd, len(sends), _vp(recvbuf),
                                                           rcv, len(recvs), _stream()), "hbgpu_comm_exchange")
        else:
            self.hub.transfer(self.rank, sendbuf, sends, recvbuf, recvs)


class LoopbackHub:
    """In-process transport of HaloContext for ranks run as threads of one
    process on one GPU: each rank posts its send buffer and segments, all
    ranks meet, every rank copies its receive segments from the peers'
    send buffers, all ranks meet again (so no buffer is reused early)."""

    def __init__(self, nranks):
        import threading
        self.posted = {}
        self.barrier = threading.Barrier(nranks)

    def transfer(self, rank, sendbuf, sends, recvbuf, recvs):
        import torch
        torch.cuda.current_stream().synchronize()
        self.posted[rank] = (sendbuf, {p: (o, c) for p, o, c in sends})
        self.barrier.wait()
        for peer, off, cnt in recvs:
            buf, segs = self.posted[peer]
            soff, scnt = segs[rank]
            if scnt != cnt:
                from .exceptions import ProtocolError
                raise ProtocolError(f"rank {peer} -> {rank}: {scnt} != {cnt} doubles")
            recvbuf[off:off + cnt].copy_(buf[soff:soff + cnt])
        torch.cuda.current_stream().synchronize()
        self.barrier.wait()


def _segments(dirs, peer_of, datasize):
    """Element-major payload offsets per direction, grouped by peer ascending
    (plan order inside), and the (peer, offset, count) messages."""
    order = sorted(range(len(dirs)), key=lambda k: (peer_of(dirs[k]), k))
    offs, msgs, pos = {}, [], 0
    for k in order:
        d = dirs[k]
        offs[k] = pos
        n = d.length * datasize
        if msgs and msgs[-1][0] == peer_of(d):
            msgs[-1][2] += n
        else:
            msgs.append([peer_of(d), pos, n])
        pos += n
    return offs, [tuple(m) for m in msgs], pos


def exchange_halos(field, plan, ctx=None):
    """One halo exchange (exchange.py:382-402): every cut halo cell of the
    field's blocks <- its paired interior cell, bitwise.  Cuts between two
    of this rank's blocks are copied on the device; with `ctx` (HaloContext)
    the remote ones are packed element-major (exchange.py:248-252), moved
    one aggregated payload per peer, and unpacked (exchange.py:254-258)."""
    import torch
    from .cutplan import rank_routes
    from .exceptions import ProtocolError
    rank = ctx.rank if ctx is not None else None
    if rank is None:
        dirs = list(plan.directions())
        if any(not d.local for d in dirs):
            raise ProtocolError("the plan has remote cuts: pass a HaloContext (rank + transport)")
        local, sends, recvs = dirs, (), ()
    else:
        routes = rank_routes(plan, rank)
        local, sends, recvs = routes.local, routes.sends, routes.recvs
    ds = plan.datasize
    dev = field.pool.device
    send_off, send_msgs, nsend = _segments(sends, lambda d: d.recv_rank, ds)
    recv_off, recv_msgs, nrecv = _segments(recvs, lambda d: d.sender_rank, ds)
    sendbuf = torch.zeros(max(1, nsend), dtype=torch.float64, device=dev)
    recvbuf = torch.zeros(max(1, nrecv), dtype=torch.float64, device=dev)

    def run(rows):
        if not rows:
            return
        arr = np.array(rows, dtype=native.HALO_DIR_DTYPE)
        t = torch.from_numpy(arr.view(np.uint8).copy()).to(dev)
        native.check(native.load().hbgpu_halo(_vp(field.pool), _vp(sendbuf), _vp(recvbuf), _vp(t), len(rows),
                                              int(arr["length"].max()), field.planes, _stream()), "hbgpu_halo")

    rows = []
    for d in local:
        s_off, s_es, s_vs = _dense_run(field, d.src_block, d.src_face, d.src_index(0), d.src_reversed, False)
        t_off, t_es, t_vs = _dense_run(field, d.dst_block, d.dst_face, d.dst_index(0), d.dst_reversed, True)
        rows.append((s_off, s_es, s_vs, t_off, t_es, t_vs, d.length, 0, 0, 0))
    for k, d in enumerate(sends):   # pack: element e of the direction at send_off + e * datasize
        s_off, s_es, s_vs = _dense_run(field, d.src_block, d.src_face, d.src_index(0), d.src_reversed, False)
        rows.append((s_off, s_es, s_vs, send_off[k], ds, 1, d.length, 0, 1, 0))
    run(rows)
    if ctx is not None and (send_msgs or recv_msgs):
        ctx.transfer(sendbuf, send_msgs, recvbuf, recv_msgs)
        rows = []
        for k, d in enumerate(recvs):
            t_off, t_es, t_vs = _dense_run(field, d.dst_block, d.dst_face, d.dst_index(0), d.dst_reversed, True)
            rows.append((recv_off[k], ds, 1, t_off, t_es, t_vs, d.length, 2, 0, 0))
        run(rows)


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
