"""The run-level drop-in: RunSpec / run_case / CaseRunResult on B200s.

Mirrors the reference's driver (driver.py:34-63 types, 110-200 run loop):
build topology -> partition blocks over ranks (one rank = one GPU) -> cut
plan -> initial state -> priming halo exchange -> `iterations` x (4 RK
stages with halo exchange, force integration) -> fields (halos included)
and globally reduced forces.  The per-iteration schedule runs inside
libhbgpu's engine (one CUDA stream, optionally a replayed CUDA graph).

Differences that do not change any returned value:
* force partials are integrated on the device every iteration and kept as a
  history; the rank-ordered global sum (runtime.py:290-294) is done once at
  the end over the whole history, instead of once per iteration.  `forces`
  is the last iteration's, as in the reference;
* divergence is detected on the device (per-block keys) and raised after the
  loop (or at a polling point), with the reference's DivergenceError fields
  for the first diverging stage.

Additions: `residual_norms` (the per-iteration L2 norm of the stage-one
residual; not produced by the reference) and
`force_history`.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import hbop, native, outio
from .cutplan import ExchangeMode, ExchangeStrategy, build_cut_plan, predicted_message_count, rank_routes
from .devlayout import build_rank_layout
from .exceptions import CollectiveError, DivergenceError, ProtocolError, RankFailure, RunAborted
from .topology import build_topology, partition_blocks

NO_BAD = (1 << 64) - 1
# phase wall times (s) of the last single-GPU run_case: layout, alloc,
# upload, engine, compute, download
LAST_TIMINGS = {}
# the last single-GPU run_case: iterations the engine issued before the loop
# ended (early on divergence) and whether it ran the paired schedule
LAST_RUN = {}
LIN_BITS = native.STATUS_LIN_BITS
HAZARD_BIT = native.HAZARD_BIT
# status polling: about this many units of work between two looks at the
# device divergence keys (~25 ms at C4 rates), at most POLL_MAX iterations
POLL_UNITS = 1 << 31
POLL_MAX = 64
# run_case calls repeated on the strict kernels (StrictRerun), process-wide
STRICT_RERUNS = [0]


class StrictRerun(Exception):
    """A paired-schedule run met a value of magnitude >= 2^1022 (a hazard
    key, include/hbgpu.h): the paired kernel's exact rewrites do not hold
    for the stages after it, so run_case repeats the run on the strict
    single-stage kernels.  Never escapes run_case."""


class ReduceMode(Enum):
    PER_BODY_PER_HARMONIC = "per-item"
    SINGLE_BUFFER = "buffered"


@dataclass(frozen=True)
class ForceReduceStrategy:
    """The reference's reduction strategy (reduce.py:27-45).  Both modes give
    the same sums (the device folds every rank's force history in rank
    order); the mode sets the collective-call counter (reduce.py:40-46).
    functag 2 -- cm left unreduced -- is refused by run_case."""

    mode: object = ReduceMode.SINGLE_BUFFER
    functag: int = 3

    def __post_init__(self):
        object.__setattr__(self, "mode", ReduceMode(self.mode))
        if self.functag not in (2, 3):
            raise CollectiveError(f"functag must be 2 or 3, got {self.functag}")

    def collective_calls(self, planes, nbody):
        if nbody == 0:
            return 0
        return planes * nbody if self.mode is ReduceMode.PER_BODY_PER_HARMONIC else 1


@dataclass
class RunSpec:
    case: object
    ranks: int = 1
    threads: int = 1
    axis: object = None
    activation: object = None
    exchange: ExchangeStrategy = field(default_factory=ExchangeStrategy)
    reduce: ForceReduceStrategy = field(default_factory=ForceReduceStrategy)
    io: object = None            # outio.WriteMode (None = buffered)
    iterations: int | None = None
    out_dir: str | None = None
    extra_outputs: tuple = ()
    machine: str = ""
    jitter_seed: int | None = None
    # --- device options -------------------------------------------------
    initial: object = None       # callable(spec, planes, npde) -> (P, npde, nj, ni)
    initial_state: dict | None = None   # gid -> host tensor (P, npde, nj, ni), pinned for speed
    output: dict | None = None          # gid -> host tensor (P, npde, nj+2, ni+2) to fill
    use_graph: bool = True
    tile_rows: int | None = None
    device: int | None = None
    # single process, ranks > 1: "fold" runs all blocks in one engine;
    # "loopback" runs one engine per rank on this GPU with device-copy
    # transport (exercises the multi-GPU halo path); "loopback-split" does
    # so with the overlapped boundary / interior schedule of the NCCL engine
    transport: str = "fold"
    # paired RK stages (hb_pair.cu): None = auto (eligible and from
    # FUSED_MIN_UNITS units per stage), False = single stages
    fused: bool | None = None
    # one-launch small schedule (hb_small.cu): None = auto (single rank
    # without remote cuts, up to SMALL_MAX_UNITS units per stage), False = off
    small: bool | None = None


@dataclass
class ForceCoefficients:
    """cl / cd / cm, each of shape (planes, nbody) (hbcore.py:329-356)."""

    cl: np.ndarray
    cd: np.ndarray
    cm: np.ndarray

    @classmethod
    def zeros(cls, planes, nbody):
        return cls(np.zeros((planes, nbody)), np.zeros((planes, nbody)), np.zeros((planes, nbody)))

    @classmethod
    def from_stack(cls, arr):
        return cls(arr[0].copy(), arr[1].copy(), arr[2].copy())

    def copy(self):
        return ForceCoefficients(self.cl.copy(), self.cd.copy(), self.cm.copy())

    @property
    def planes(self):
        return self.cl.shape[0]

    @property
    def nbody(self):
        return self.cl.shape[1]

    def equal_bits(self, other):
        return all(np.array_equal(a, b) for a, b in
                   ((self.cl, other.cl), (self.cd, other.cd), (self.cm, other.cm)))


@dataclass
class RunRecord:
    case: str
    machine: str
    ranks: int
    threads: int
    iterations: int
    wall_s: float
    msgs: int
    bytes: int
    collectives: int
    write_ops: int
    activations: int
    units: int = 0
    loop_s: float = 0.0          # device: prime + iteration loop wall time
    gpus: int = 1

    @property
    def units_per_s(self):
        return self.units / self.wall_s if self.wall_s > 0 else 0.0


@dataclass
class CaseRunResult:
    fields: dict
    forces: ForceCoefficients
    counters: list
    wall_s: float
    record: object
    residual_norms: list = field(default_factory=list)
    force_history: list = field(default_factory=list)

    def field_bits_equal(self, other):
        if sorted(self.fields) != sorted(other.fields):
            return False
        return all(np.array_equal(self.fields[b], other.fields[b]) for b in self.fields)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


class DeviceRank:
    """One rank's blocks resident on one GPU, plus its libhbgpu engine."""

    def __init__(self, case, topology, partition, plan, rank=0, device=None, comm=None,
                 initial=None, tile_rows=None, max_iters=1, pinned_ic=None, fused=None, small=None):
        import torch
        self.lib = native.require_cuda()
        self.torch = torch
        self.case = case
        self.planes = case.planes
        self.rank = rank
        self.comm = comm
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        torch.cuda.set_device(self.device)
        t0 = time.perf_counter()
        L = self.layout = build_rank_layout(topology, partition, plan, rank, case.planes, tile_rows,
                                            fused=fused, small=small)
        self.timings = {"layout": time.perf_counter() - t0}
        dev = self.device
        f64 = torch.float64
        self.slots = [torch.zeros(L.slot_elems, dtype=f64, device=dev) for _ in range(3)]
        self.sendbuf = torch.zeros(max(1, L.sendbuf_elems), dtype=f64, device=dev)
        self.recvbuf = torch.zeros(max(1, L.recvbuf_elems), dtype=f64, device=dev)

        def table(arr):
            raw = np.ascontiguousarray(arr).view(np.uint8).ravel()
            t = torch.zeros(max(16, raw.size), dtype=torch.uint8)
            t[:raw.size] = torch.from_numpy(raw.copy())
            return t.to(dev)

        self.t_blocks = table(L.block_table)
        self.t_tiles = torch.from_numpy(L.tile_block).to(dev)
        # forcing tables sxy[j, i] = sx[i] * sy[j], formed on the device (one
        # rounded product per element, as hbcore.py:169 forms it)
        self.t_sxy = torch.zeros(max(1, L.sxy_size), dtype=f64, device=dev)
        for k, (sx, sy) in enumerate(L.sxy):
            off, sp = int(L.block_table["sxy_off"][k]), int(L.block_table["sxy_pitch"][k])
            tbl = self.t_sxy[off:off + sy.size * sp].view(sy.size, sp)
            tbl[:, :sx.size] = (torch.from_numpy(sx).to(dev)[None, :] *
                                torch.from_numpy(sy).to(dev)[:, None])
        self.t_faces = table(L.faces)
        self.t_prime = table(L.prime_dirs)
        self.t_unpack = table(L.unpack_dirs)
        self.t_post = table(L.post_dirs)
        self.t_band = table(L.band_segs)
        self.t_segs = table(L.force_segs)
        deriv = hbop.spectral_matrix(case.nharms, case.omega)
        self.dmat = np.ascontiguousarray(deriv.matrix)
        self.t_dmat = torch.from_numpy(self.dmat.copy()).to(dev)
        self.ap = hbop.forcing_amplitudes(case.planes, 4)
        nb = len(L.blocks)
        self.max_iters = max(1, max_iters)
        self.norm_part = torch.zeros(L.total_tiles * native.TILE_WARPS, dtype=f64, device=dev)
        # paired schedule: q0 at every tile's two edge columns, saved by pass A
        # for pass B (which overwrites q0 in place); hbgpu_stage_args.edge_q0
        self.edge_q0 = torch.zeros(L.total_tiles * L.tile_rows * 2 * L.tile_pdes * case.planes
                                   if L.fused else 1, dtype=f64, device=dev)
        self.sumsq = torch.zeros(self.max_iters * nb, dtype=f64, device=dev)
        self.status = torch.full((nb,), -1, dtype=torch.int64, device=dev)
        self.iter = torch.zeros(1, dtype=torch.int32, device=dev)
        nforce = 3 * case.planes * case.nbody
        self.force_hist = torch.zeros(max(1, self.max_iters * nforce), dtype=f64, device=dev)
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        self.upload_initial(initial, pinned_ic)
        torch.cuda.synchronize(dev)
        t2 = time.perf_counter()
        self._encode_tensor_maps()
        self._make_engine()
        self.timings.update(alloc=t1 - t0 - self.timings["layout"], upload=t2 - t1,
                            engine=time.perf_counter() - t2)

    # -- state in / out --------------------------------------------------------

    def block_view(self, slot, gid):
        """The block's (planes, npde, nj+2, ni+2) array (halos included) as a
        strided view of a slot, for either slot layout."""
        off, shape, strides = self.layout.block_view(gid)
        return slot.as_strided(shape, strides, off)

    def upload_initial(self, initial=None, pinned=None):
        """Interior of slot A <- the initial state; halos and slots B, C zero.

        `pinned`, when given, maps gid -> host (pinned) tensors of shape
        (P, npde, nj, ni) to copy from (the end-to-end path).
        """
        torch = self.torch
        for s in self.slots:
            s.zero_()
        for b in self.layout.blocks:
            dst = self.block_view(self.slots[0], b.id)[:, :, 1:b.nj + 1, 1:b.ni + 1]
            if pinned is not None:
                dst.copy_(pinned[b.id].to(self.device, non_blocking=True))
                continue
            if initial is None:
                ic = hbop.initial_values(b, self.planes, 4, 0, self.planes, 1, b.nj + 1)
            else:
                ic = initial(b, self.planes, 4)
            dst.copy_(torch.from_numpy(np.ascontiguousarray(ic, dtype=np.float64)))

    def fields(self, slot=0, pinned_out=None):
        """{gid: (P, npde, nj+2, ni+2) numpy array incl. halos} of a slot."""
        out = {}
        for b in self.layout.blocks:
            view = self.block_view(self.slots[slot], b.id)
            if pinned_out is not None:
                dst = pinned_out[b.id]
                dst.copy_(view.contiguous(), non_blocking=True)
                out[b.id] = dst.numpy()
            else:
                out[b.id] = view.cpu().numpy()
        return out

    # -- engine ----------------------------------------------------------------

    def _encode_tensor_maps(self):
        """TMA descriptors (TMAP_SETS sets x blocks, 128 B each), uploaded to the device."""
        L = self.layout
        n = len(L.blocks)
        host = (ctypes.c_ubyte * (native.TMAP_SETS * n * 128))()
        slots = (ctypes.c_void_p * 3)(*[s.data_ptr() for s in self.slots])
        blocks = np.ascontiguousarray(L.block_table)
        native.check(self.lib.hbgpu_encode_tensor_maps(slots, self.t_sxy.data_ptr(),
                                                       blocks.ctypes.data, n, self.planes,
                                                       L.tile_pdes,
                                                       ctypes.addressof(host), len(host)),
                     "hbgpu_encode_tensor_maps")
        self.t_tmaps = self.torch.frombuffer(bytearray(host), dtype=self.torch.uint8).to(self.device)

    def _make_engine(self):
        torch = self.torch
        L = self.layout
        d = native.EngineDesc()
        for k in range(3):
            d.slot[k] = self.slots[k].data_ptr()
        d.sendbuf, d.recvbuf = self.sendbuf.data_ptr(), self.recvbuf.data_ptr()
        d.blocks, d.tile_block = self.t_blocks.data_ptr(), self.t_tiles.data_ptr()
        d.sxy, d.faces, d.dmat = self.t_sxy.data_ptr(), self.t_faces.data_ptr(), self.t_dmat.data_ptr()
        d.norm_part, d.sumsq = self.norm_part.data_ptr(), self.sumsq.data_ptr()
        d.status, d.iter = self.status.data_ptr(), self.iter.data_ptr()
        d.prime_dirs, d.nprime = self.t_prime.data_ptr(), len(L.prime_dirs)
        d.prime_max_len = int(L.prime_dirs["length"].max()) if len(L.prime_dirs) else 0
        d.unpack_dirs, d.nunpack = self.t_unpack.data_ptr(), len(L.unpack_dirs)
        d.unpack_max_len = int(L.unpack_dirs["length"].max()) if len(L.unpack_dirs) else 0
        d.post_dirs, d.npost = self.t_post.data_ptr(), len(L.post_dirs)
        d.post_max_len = int(L.post_dirs["length"].max()) if len(L.post_dirs) else 0
        d.band_segs, d.nband_segs = self.t_band.data_ptr(), len(L.band_segs)
        d.band_max_len, d.fused = int(L.band_max_len), int(L.fused)
        d.small, d.small_max_cells = int(L.small), int(L.small_max_cells)
        d.edge_q0 = self.edge_q0.data_ptr()
        # multi-GPU overlap: boundary tiles first, remote packs first
        self.t_order = torch.from_numpy(np.ascontiguousarray(L.tile_order, dtype=np.int32)).to(self.device)
        d.tile_order = self.t_order.data_ptr()
        d.nbound_tiles, d.prime_remote, d.post_remote = int(L.nbound), int(L.prime_remote), int(L.post_remote)
        d.segs, d.nsegs = self.t_segs.data_ptr(), len(L.force_segs)
        d.force_hist = self.force_hist.data_ptr()
        self._sends = (native.PeerMsg * max(1, len(L.sends)))(
            *[native.PeerMsg(p, 0, o, c) for p, o, c in L.sends])
        self._recvs = (native.PeerMsg * max(1, len(L.recvs)))(
            *[native.PeerMsg(p, 0, o, c) for p, o, c in L.recvs])
        d.sends, d.nsends = self._sends, len(L.sends)
        d.recvs, d.nrecvs = self._recvs, len(L.recvs)
        d.comm = self.comm
        d.tmaps = self.t_tmaps.data_ptr()
        d.nblocks, d.total_tiles, d.planes = len(L.blocks), L.total_tiles, self.planes
        d.nbody, d.tile_rows, d.max_iters = self.case.nbody, L.tile_rows, self.max_iters
        d.interleaved, d.tile_pdes = int(L.interleaved), int(L.tile_pdes)
        for k, c in enumerate(hbop.RKScheme(self.case.dtau).stage_coefficients()):
            d.coef[k] = c
        P = self.planes
        if P > native.MAX_P:
            raise NotImplementedError(f"{P} snapshots exceed the library limit {native.MAX_P}")
        # the stage kernel adds the D[n][n] term and the forcing of planes other
        # than 1 and 2 as signed zeros (hb_common.cuh add_signed_zero)
        diag = np.diagonal(self.dmat)
        unforced = [n for n in range(P) if n not in (1, 2)]
        if np.any(diag.view(np.uint64) != 0) or np.any(self.ap[unforced].view(np.uint64) != 0):
            raise ValueError("operator tables break the +0.0 diagonal / planes-1,2 forcing invariant")
        # ... and shares each D product between rows m+k and m-k (exact for
        # the spectral matrix's bitwise antisymmetric circulant structure)
        if P <= native.MAX_TEMPLATED_P and not hbop.circulant_antisymmetric(self.dmat):
            raise ValueError("D is not bitwise antisymmetric circulant (D[m+k][m] == -D[m-k][m])")
        if P <= native.MAX_TEMPLATED_P:
            flat = self.dmat.ravel()
            for k in range(P * P):
                d.D[k] = flat[k]
        apf = self.ap.ravel()
        for k in range(P * 4):
            d.ap[k] = apf[k]
        self._desc = d
        eng = ctypes.c_void_p()
        native.check(self.lib.hbgpu_engine_create(ctypes.byref(d), ctypes.byref(eng)),
                     "hbgpu_engine_create")
        self.engine = eng

    def stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def prime(self):
        native.check(self.lib.hbgpu_engine_prime(self.engine, self.stream()), "hbgpu_engine_prime")

    def iterate(self, iterations, use_graph=True):
        if self.comm is None and (self.layout.sends or self.layout.recvs):
            raise ProtocolError("this rank has remote cuts but no communicator; "
                                "step it with hbgpu_engine_step/unpack (loopback) instead")
        native.check(self.lib.hbgpu_engine_iterate(self.engine, int(iterations), int(bool(use_graph)),
                                                   self.stream()), "hbgpu_engine_iterate")

    def launches_per_iteration(self):
        return int(self.lib.hbgpu_engine_launches_per_iteration(self.engine))

    # slot rotation of the engine (hb_runtime.cu): stage s reads IN[s], writes OUT[s]
    STAGE_IN = (0, 1, 2, 1)
    STAGE_OUT = (1, 2, 1, 0)
    # paired schedule, per phase: band(0), pair(0,1), band(2), pair(2,3)
    PHASE_IN = (0, 0, 1, 1)
    PHASE_OUT = (2, 1, 2, 0)

    @property
    def fused(self):
        return bool(self.layout.fused)

    def phase_args(self, phase):
        """Arguments of phase `phase` of the paired schedule as the engine
        issues them: phases 0 / 2 go to hbgpu_band, 1 / 3 to hbgpu_stage."""
        a = self.stage_args(0 if phase < 2 else 2)
        d = self._desc
        a.in_ = self.slots[self.PHASE_IN[phase]].data_ptr()
        a.out = self.slots[self.PHASE_OUT[phase]].data_ptr()
        a.in_slot, a.out_slot = self.PHASE_IN[phase], self.PHASE_OUT[phase]
        a.norm_part = d.norm_part if phase == 1 else None
        if phase in (1, 3):
            a.pair = 1 if phase == 1 else 2
            a.coef2 = d.coef[(0 if phase == 1 else 2) + 1]
        return a

    def launch_band(self, args, stream=None):
        s = stream if stream is not None else self.stream()
        native.check(self.lib.hbgpu_band(ctypes.byref(args), s), "hbgpu_band")

    def stage_args(self, stage):
        """hbgpu_stage arguments of RK stage `stage` as the engine issues them."""
        d, a = self._desc, native.StageArgs()
        a.in_ = self.slots[self.STAGE_IN[stage]].data_ptr()
        a.q0 = self.slots[0].data_ptr()
        a.out = self.slots[self.STAGE_OUT[stage]].data_ptr()
        a.band = self.slots[2].data_ptr()
        a.band_segs, a.nband_segs, a.band_max_len = d.band_segs, d.nband_segs, d.band_max_len
        a.edge_q0 = d.edge_q0
        a.sendbuf, a.blocks, a.tile_block = d.sendbuf, d.blocks, d.tile_block
        a.sxy, a.faces, a.status, a.iter, a.dmat = d.sxy, d.faces, d.status, d.iter, d.dmat
        a.norm_part = d.norm_part if stage == 0 else None
        a.nblocks, a.total_tiles, a.planes = d.nblocks, d.total_tiles, d.planes
        a.stage, a.tile_rows, a.coef = stage, d.tile_rows, d.coef[stage]
        a.tmaps, a.in_slot, a.interleaved = d.tmaps, self.STAGE_IN[stage], d.interleaved
        a.out_slot = self.STAGE_OUT[stage]
        a.tile_pdes = d.tile_pdes
        ctypes.memmove(ctypes.addressof(a.D), ctypes.addressof(d.D), ctypes.sizeof(a.D))
        ctypes.memmove(ctypes.addressof(a.ap), ctypes.addressof(d.ap), ctypes.sizeof(a.ap))
        return a

    def launch_stage(self, args, stream=None):
        """One hbgpu_stage launch on `stream` (default: torch's current stream)."""
        s = stream if stream is not None else self.stream()
        native.check(self.lib.hbgpu_stage(ctypes.byref(args), s), "hbgpu_stage")

    def reset_counters(self):
        """Start the iteration history over (device counter, status keys and
        the engine's issued-iteration count)."""
        native.check(self.lib.hbgpu_engine_rewind(self.engine, self.stream()), "hbgpu_engine_rewind")

    def iterations_done(self):
        return int(self.lib.hbgpu_engine_iterations_done(self.engine))

    def close(self):
        if getattr(self, "engine", None):
            self.lib.hbgpu_engine_destroy(self.engine)
            self.engine = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- results ---------------------------------------------------------------

    def divergence(self, keys=None):
        """(gstage, hazard, gid, i, j, p, n) of this rank's first event, or None.

        The first event is the earliest global stage; at one stage a
        non-finite value (hazard False, the reference's DivergenceError at
        that stage) outranks a hazard key, and blocks go in ascending id.
        hazard True means a value of magnitude >= 2^1022 was written at that
        stage (or was present at the start, gstage 0): see StrictRerun."""
        if keys is None:
            keys = self.status.cpu().numpy()
        return decode_status(np.asarray(keys).view(np.uint64), self.layout)

    def norm_history(self, iterations):
        nb = len(self.layout.blocks)
        arr = self.sumsq[:iterations * nb].cpu().numpy().reshape(iterations, nb)
        return {b.id: arr[:, k].copy() for k, b in enumerate(self.layout.blocks)}

    def force_history_array(self, iterations):
        nf = 3 * self.planes * self.case.nbody
        return self.force_hist[:iterations * nf].view(iterations, 3, self.planes, self.case.nbody)


# ---------------------------------------------------------------------------
# run_case
# ---------------------------------------------------------------------------

def _dist():
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist
    except Exception:
        pass
    return None


def make_comm(rank, world, device):
    """NCCL communicator for libhbgpu's engine, id broadcast over torch.distributed."""
    import torch.distributed as dist
    lib = native.load()
    buf = ctypes.create_string_buffer(128)
    if rank == 0:
        native.check(lib.hbgpu_comm_unique_id(buf), "hbgpu_comm_unique_id")
    obj = [bytes(buf.raw) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = ctypes.c_void_p()
    native.check(lib.hbgpu_comm_init(obj[0], world, rank, device, ctypes.byref(comm)), "hbgpu_comm_init")
    return comm


def _global_sumsq(ranks, nblocks, iterations):
    """(iterations, nblocks) tensor: every given rank's per-block sums of R^2
    in the column of its global block id, zeros elsewhere."""
    torch = ranks[0].torch
    g = torch.zeros((iterations, nblocks), dtype=torch.float64, device=ranks[0].device)
    for dr in ranks:
        nb = len(dr.layout.blocks)
        gids = torch.tensor([b.id for b in dr.layout.blocks], dtype=torch.long, device=g.device)
        g[:, gids] = dr.sumsq[:iterations * nb].view(iterations, nb).to(g.device)
    return g


def _norm_totals(gsumsq, iterations, stream):
    """Per-iteration residual norms on the device (hbgpu_norm_totals): sqrt of
    the left-to-right sum over global blocks in ascending id."""
    torch = __import__("torch")
    if iterations == 0:
        return []
    nblocks = gsumsq.shape[1]
    out = torch.empty(iterations, dtype=torch.float64, device=gsumsq.device)
    native.check(native.load().hbgpu_norm_totals(_ptr(gsumsq.contiguous()), iterations, nblocks, _ptr(out),
                                                 stream), "hbgpu_norm_totals")
    return out.cpu().tolist()


class GlobalBlocks:
    """decode_status's view of all blocks of the topology (multi-GPU: the
    job-wide status keys are indexed by global block id)."""

    def __init__(self, topology):
        self.blocks = sorted(topology.blocks, key=lambda b: b.id)
        self.local_index = {b.id: k for k, b in enumerate(self.blocks)}


def decode_status(keys, layout):
    """Decode a rank's per-block status keys (include/hbgpu.h) into its first
    event (gstage, hazard, gid, i, j, p, n), or None."""
    best = None
    for lb, key in enumerate(keys):
        key = int(key)
        if key == NO_BAD:
            continue
        gstage, hazard = key >> LIN_BITS, bool(key & HAZARD_BIT)
        lin = key & (HAZARD_BIT - 1)
        b = layout.blocks[lb]
        cand = (gstage, hazard, b.id, lin)
        if best is None or cand[:3] < best[:3]:
            best = cand
    if best is None:
        return None
    gstage, hazard, gid, lin = best
    b = layout.blocks[layout.local_index[gid]]
    i = lin % b.ni
    j = (lin // b.ni) % b.nj
    np_ = lin // (b.ni * b.nj)
    return gstage, hazard, gid, i + 1, j + 1, np_ % 4, np_ // 4


def first_event(events):
    """The earliest of several ranks' first events (None if there is none)."""
    events = [e for e in events if e is not None]
    return min(events, key=lambda e: e[:3]) if events else None


def raise_divergence(div):
    """DivergenceError with the reference's fields (errors.py:28-29), or
    StrictRerun for a hazard key."""
    if div is None:
        return
    _, hazard, gid, i, j, p, n = div
    if hazard:
        raise StrictRerun(f"value of magnitude >= 2^1022 at global stage {div[0]} (block {gid})")
    raise DivergenceError(gid, i, j, p, n)


def poll_interval(topology, planes, iterations):
    units = max(1, topology.total_cells() * planes * 4)
    return max(1, min(POLL_MAX, iterations, POLL_UNITS // units))


class StatusPoller:
    """Iterates a DeviceRank in chunks and looks at its divergence keys
    between them, so a diverging run stops within about one chunk of the
    failing stage (the reference raises at the stage itself, hbcore.py:
    273-276) instead of finishing the loop on NaNs.

    After each chunk the keys go to pinned host memory by an async copy on
    the compute stream; the host reads the PREVIOUS chunk's copy while the
    current one runs, so the device never waits for the host.  `reduce`,
    when given, turns the local keys into the job-wide ones (multi-GPU:
    every rank must stop at the same chunk or NCCL would hang)."""

    def __init__(self, dr, chunk, reduce=None, wait=None):
        import torch
        self.torch = torch
        self.dr, self.chunk, self.reduce = dr, max(1, int(chunk)), reduce
        self.wait = wait or (lambda ev: ev.synchronize())
        self.host = [None, None]
        self.events = [torch.cuda.Event(), torch.cuda.Event()]
        self.k = 0
        self.pending = None

    def _snapshot(self):
        src = self.dr.status if self.reduce is None else self.reduce(self.dr.status)
        if self.host[self.k] is None:
            self.host[self.k] = self.torch.empty(src.numel(), dtype=self.torch.int64, pin_memory=True)
        buf = self.host[self.k]
        buf.copy_(src, non_blocking=True)
        self.events[self.k].record()
        slot, self.k = self.k, 1 - self.k
        return slot

    def _check(self, slot):
        self.wait(self.events[slot])
        keys = self.host[slot].numpy()
        return None if np.all(keys == -1) else keys

    def run(self, iterations, use_graph):
        """Returns the keys of the first chunk that saw an event, else None."""
        done = 0
        while done < iterations:
            k = min(self.chunk, iterations - done)
            self.dr.iterate(k, use_graph=use_graph)
            done += k
            slot = self._snapshot()
            if self.pending is not None:
                keys = self._check(self.pending)
                if keys is not None:
                    return keys
            self.pending = slot
        if self.pending is not None:
            keys = self._check(self.pending)
            self.pending = None
            return keys
        return None


def run_case(spec):
    """Execute one configuration end to end; fields come back with halos.

    Under torch.distributed with world size W > 1, each process is one rank
    on its own GPU and spec.ranks must equal W.  In a single process,
    spec.ranks > 1 keeps the reference partition for the cut plan and its
    counters, but all ranks' blocks run on the one GPU (results are
    partition-invariant bitwise, as the reference's acceptance criterion 4
    requires).
    """
    case = spec.case
    topology = build_topology(case)
    partition = partition_blocks(topology, spec.ranks)
    plan = build_cut_plan(topology, partition, case.nharms, case.npde)
    iterations = case.iterations if spec.iterations is None else spec.iterations
    if spec.reduce.functag != 3 and spec.ranks > 1:
        # reduce.py:79-96 leaves cm as each rank's own partial and the driver
        # returns rank 0's; with one rank that is the full sum (supported)
        raise NotImplementedError("functag=2 with ranks > 1 (cm left as rank 0's partial) is not "
                                  "supported: the device path reduces cl, cd and cm")
    dist = _dist()
    world = dist.get_world_size() if dist is not None else 1
    if world > 1 and spec.ranks != world:
        raise ProtocolError(f"spec.ranks={spec.ranks} but torch.distributed world size is {world}")

    import torch
    native.require_cuda()
    # output files exist at their final size before any rank writes
    # (driver.py:160-167); every rank writes its own records after the loop
    targets = _output_targets(spec)
    layouts = outio.all_layouts(topology, case.nharms, case.npde) if targets else ()
    if targets:
        if world == 1 or dist.get_rank() == 0:
            for out_dir, _ in targets:
                outio.create_output_files(out_dir, layouts)
        if world > 1:
            dist.barrier()
    out = (layouts, targets)
    t0 = time.perf_counter()

    def execute(sp):
        if world > 1:
            return _execute_distributed(sp, topology, partition, plan, iterations, dist, world, out)
        if sp.ranks > 1 and sp.transport in ("loopback", "loopback-split"):
            return _execute_loopback(sp, topology, partition, plan, iterations, out)
        one = partition_blocks(topology, 1)
        return _execute_single(sp, topology, one, build_cut_plan(topology, one, case.nharms, case.npde),
                               iterations, out)

    try:
        try:
            fields, hist_np, norms, loop_s = execute(spec)
        except StrictRerun:
            STRICT_RERUNS[0] += 1
            # a value of magnitude >= 2^1022 appeared on the paired schedule:
            # repeat the whole run on the strict single-stage kernels (every
            # rank takes this branch: the first event is agreed job-wide)
            import dataclasses
            fields, hist_np, norms, loop_s = execute(dataclasses.replace(spec, fused=False))
    except DivergenceError as err:
        # the reference's spawn_ranks wraps every rank error in a RankFailure
        # naming the failing rank (runtime.py:359-364), so run_case raises
        # RankFailure(rank, DivergenceError) at any rank count
        # (tests/test_driver_cli.py:30-36); the rank is the owner of the
        # diverging block in the reference partition
        raise RankFailure(partition.rank_of(err.block), err) from err
    wall = time.perf_counter() - t0

    forces = (ForceCoefficients.from_stack(hist_np[-1]) if iterations > 0
              else ForceCoefficients.zeros(case.planes, case.nbody))
    activations = iterations * (12 if _per_loop(spec.activation) else 1) + len(targets)
    counters = rank_counters(plan, spec, partition, iterations, activations, layouts, targets, world)
    record = None
    if iterations >= 1:
        units = topology.total_cells() * case.planes * 4 * iterations
        record = RunRecord(case=case.name or "case", machine=spec.machine, ranks=spec.ranks,
                           threads=spec.threads, iterations=iterations, wall_s=wall,
                           msgs=sum(c.msgs_sent for c in counters),
                           bytes=sum(c.bytes_sent for c in counters),
                           collectives=iterations * spec.reduce.collective_calls(case.planes, case.nbody),
                           write_ops=sum(c.write_ops for c in counters),
                           activations=activations, units=units, loop_s=loop_s,
                           gpus=world)
    return CaseRunResult(fields=fields, forces=forces, counters=counters, wall_s=wall,
                         record=record, residual_norms=norms,
                         force_history=[ForceCoefficients.from_stack(h) for h in hist_np])


def _new_rank(spec, topology, partition, plan, rank, device, comm, iterations):
    return DeviceRank(spec.case, topology, partition, plan, rank=rank, device=device, comm=comm,
                      initial=spec.initial, tile_rows=spec.tile_rows, max_iters=max(1, iterations),
                      pinned_ic=spec.initial_state, fused=spec.fused, small=spec.small)


def _history(dr, iterations):
    case = dr.case
    if iterations == 0:
        return np.zeros((0, 3, case.planes, case.nbody))
    return dr.force_history_array(iterations).cpu().numpy()


@dataclass(frozen=True)
class CounterSnapshot:
    """Per-rank counters with the reference's fields (runtime.py:38-45)."""

    msgs_sent: int
    bytes_sent: int
    msgs_received: int
    collective_calls: int
    write_ops: int
    team_activations: int
    # what the device path itself moved (the fields above are the reference's
    # counters for the chosen strategies, exchange.py:172-188): one
    # aggregated payload per peer and exchange (NCCL send or loopback copy),
    # its bytes, and the NCCL collectives of a multi-GPU run (divergence
    # consensus per polling chunk, the final status / norm all-reduces, the
    # force-history all-gather)
    device_msgs: int = 0
    device_bytes: int = 0
    device_collectives: int = 0


def _per_loop(activation):
    return getattr(activation, "value", activation) == "per-loop"


def rank_counters(plan, spec, partition, iterations, activations, layouts, targets, world=1):
    """What each rank of the reference partition sends, receives, reduces and
    writes under spec's strategies -- the reference's counters exactly
    (exchange.py:172-188 message counts, reduce.py:40-46 collectives,
    outio.py:221-241 write ops, hybrid.py:233-237 activations).  The device
    moves the same bytes in one aggregated message per peer and stage."""
    exchanges = 4 * iterations + 1
    per_element = spec.exchange.mode is ExchangeMode.PER_ELEMENT
    sent = [0] * spec.ranks
    sent_bytes = [0] * spec.ranks
    received = [0] * spec.ranks
    for cut in plan.cuts:
        if cut.local:
            continue
        msgs = 2 * cut.length if per_element else 1
        for d in cut.directions:
            sent[d.sender_rank] += msgs * exchanges
            sent_bytes[d.sender_rank] += cut.length * cut.datasize * 8 * exchanges
            received[d.recv_rank] += msgs * exchanges
    calls = iterations * spec.reduce.collective_calls(spec.case.planes, spec.case.nbody)
    dev_msgs, dev_bytes, dev_coll = device_traffic(plan, spec, iterations, world)
    out = []
    for r in range(spec.ranks):
        owned = partition.blocks_of(r)
        ops = sum(outio.write_ops(layouts, owned, mode) for _, mode in targets)
        out.append(CounterSnapshot(sent[r], sent_bytes[r], received[r], calls, ops, activations,
                                   dev_msgs[r], dev_bytes[r], dev_coll))
    return out


def device_traffic(plan, spec, iterations, world=1):
    """Per rank: (payloads sent, bytes sent) by the device path over the run,
    and the NCCL collectives of the run.  A single-process "fold" run keeps
    every cut inside one engine (nothing moves between ranks); "loopback"
    and multi-GPU runs send one aggregated payload per peer and exchange
    (4 per iteration + the priming one), whatever the reference strategy."""
    exchanges = 4 * iterations + 1
    msgs = [0] * spec.ranks
    nbytes = [0] * spec.ranks
    moving = world > 1 or spec.transport in ("loopback", "loopback-split")
    if moving:
        for r in range(spec.ranks):
            sends = rank_routes(plan, r).sends
            msgs[r] = len({d.recv_rank for d in sends}) * exchanges
            nbytes[r] = sum(d.length for d in sends) * plan.datasize * 8 * exchanges
    coll = 0
    if world > 1 and iterations > 0:
        first = 1 if spec.use_graph and iterations > 1 else 0
        topology = build_topology(spec.case)
        chunk = poll_interval(topology, spec.case.planes, iterations)
        coll = -(-(iterations - first) // chunk) + 3
    return msgs, nbytes, coll


def _output_targets(spec):
    """(directory, WriteMode) pairs: out_dir with spec.io, then extra_outputs."""
    from .outio import WriteMode
    targets = []
    if spec.out_dir is not None:
        targets.append((spec.out_dir, WriteMode.BUFFERED if spec.io is None else WriteMode(spec.io)))
    for out_dir, mode in spec.extra_outputs:
        targets.append((out_dir, WriteMode(mode)))
    return targets


def _write_outputs(ranks, out):
    """Every rank's records of every target, packed on its GPU (outio.py)."""
    layouts, targets = out
    t0 = time.perf_counter()
    for out_dir, mode in targets:
        for dr in ranks:
            outio.write_output(dr, layouts, mode, out_dir)
    return time.perf_counter() - t0


def _execute_single(spec, topology, partition, plan, iterations, out=((), ())):
    """All blocks on this process's GPU, one engine, graph-replayed iterations."""
    import torch
    device = spec.device if spec.device is not None else torch.cuda.current_device()
    dr = _new_rank(spec, topology, partition, plan, 0, device, None, iterations)
    try:
        torch.cuda.synchronize(dr.device)
        t0 = time.perf_counter()
        dr.prime()
        if iterations > 0:
            StatusPoller(dr, poll_interval(topology, spec.case.planes, iterations)).run(iterations, spec.use_graph)
        torch.cuda.synchronize(dr.device)
        t1 = time.perf_counter()
        LAST_RUN.clear()
        LAST_RUN.update(iterations_issued=dr.iterations_done(), fused=dr.fused, small=bool(dr.layout.small))
        raise_divergence(dr.divergence())
        fields = dr.fields(0, pinned_out=spec.output)
        hist = _history(dr, iterations)
        norms = _norm_totals(_global_sumsq([dr], len(topology.blocks), iterations), iterations, dr.stream())
        torch.cuda.synchronize(dr.device)
        dr.timings.update(compute=t1 - t0, download=time.perf_counter() - t1)
        dr.timings.update(output=_write_outputs([dr], out))
        LAST_TIMINGS.clear()
        LAST_TIMINGS.update(dr.timings)
    finally:
        dr.close()
    return fields, hist, norms, t1 - t0


def _execute_distributed(spec, topology, partition, plan, iterations, dist, world, out=((), ())):
    """One rank per process/GPU; remote halos over NCCL inside the engine.

    Every job-level exchange after setup goes through the engine's NCCL
    communicator -- the divergence consensus (MIN all-reduce of the status
    keys), the norm sums (SUM all-reduce, then the device fold) and the force
    history (all-gather + rank-ordered fold) -- and every wait on it runs
    under a CommGuard: NCCL async errors, a peer's failure notice and a
    timeout abort the communicator and raise, instead of leaving ranks
    blocked (the reference aborts its fabric: runtime.py:133-144, 345-364)."""
    import torch
    rank = dist.get_rank()
    device = spec.device if spec.device is not None else rank % torch.cuda.device_count()
    torch.cuda.set_device(device)
    comm = make_comm(rank, world, device)
    guard = CommGuard(comm, rank, _store(dist))
    dr = None
    try:
        try:
            dr = _new_rank(spec, topology, partition, plan, rank, device, comm, iterations)
            gblocks = GlobalBlocks(topology)
            torch.cuda.synchronize(dr.device)
            t0 = time.perf_counter()
            dr.prime()
            job_keys = _job_keys(dr, gblocks, comm)
            if iterations > 0:
                # the first iteration eagerly: NCCL sets up its peer connections
                # outside the graph capture that records the rest
                first = 1 if spec.use_graph and iterations > 1 else 0
                if first:
                    dr.iterate(first, use_graph=False)
                chunk = poll_interval(topology, spec.case.planes, iterations)
                StatusPoller(dr, chunk, reduce=job_keys, wait=guard.wait).run(iterations - first,
                                                                              spec.use_graph)
            keys = job_keys(dr.status)
            guard.sync()
            loop_s = time.perf_counter() - t0
            raise_divergence(decode_status(keys.cpu().numpy().view(np.uint64), gblocks))
            fields = dr.fields(0, pinned_out=spec.output)
            if iterations > 0:
                hist = _reduce_history(dr, dr.force_history_array(iterations), world)
                gs = _global_sumsq([dr], len(gblocks.blocks), iterations)
                native.check(dr.lib.hbgpu_comm_allreduce(comm, _ptr(gs), _ptr(gs), gs.numel(),
                                                         native.REDUCE_SUM_F64, dr.stream()),
                             "hbgpu_comm_allreduce")
                guard.sync()
                norms = _norm_totals(gs, iterations, dr.stream())
                hist = hist.cpu().numpy()
            else:
                hist, norms = _history(dr, 0), []
            guard.sync()
            _write_outputs([dr], out)
            if out[1]:
                dist.barrier()
        except (DivergenceError, StrictRerun, RankFailure):
            raise
        except BaseException as exc:   # noqa: BLE001 - this rank failed: tell the peers
            guard.notify_failure()
            if isinstance(exc, (CollectiveError, RunAborted)):
                raise
            raise RankFailure(rank, exc) from exc
    finally:
        if dr is not None:
            dr.close()
        if not guard.aborted:
            native.load().hbgpu_comm_destroy(comm)
    return fields, hist, norms, loop_s


def _store(dist):
    try:
        return dist.distributed_c10d._get_default_store()
    except Exception:
        return None


def _job_keys(dr, gblocks, comm):
    """Status keys -> the job-wide per-block keys (one per global block,
    all-ones where nothing happened): scatter into a global array, MIN
    all-reduce (unsigned) over the engine's communicator."""
    torch = dr.torch
    gids = torch.tensor([b.id for b in dr.layout.blocks], dtype=torch.long, device=dr.device)
    buf = torch.full((len(gblocks.blocks),), -1, dtype=torch.int64, device=dr.device)

    def reduce(status):
        buf.fill_(-1)
        buf[gids] = status
        native.check(dr.lib.hbgpu_comm_allreduce(comm, _ptr(buf), _ptr(buf), buf.numel(), native.REDUCE_MIN_U64,
                                                 dr.stream()), "hbgpu_comm_allreduce")
        return buf

    return reduce


class CommGuard:
    """Bounded waits for a multi-GPU run.

    wait(event) returns once the event completed.  While waiting it polls
    (1) the communicator's asynchronous error state, (2) the job's failure
    notice (a key in torch.distributed's store, written by the first rank
    that fails) and (3) a deadline, TIMEOUT seconds as the reference's
    runtime.py:29.  Any of them aborts the NCCL communicator (its pending
    operations fail, so this rank's stream drains) and raises: CollectiveError
    for an NCCL error or a timeout, RankFailure(failed_rank, RunAborted) when
    a peer reported its failure.  notify_failure() is the failing rank's
    side: post the notice (first writer wins), abort the communicator."""

    TIMEOUT = 120.0
    KEY = "hbgpu/failed_rank"
    POLL_S = 50e-6

    def __init__(self, comm, rank, store, timeout=None, async_error=None, abort=None):
        self.comm, self.rank, self.store = comm, rank, store
        self.timeout = self.TIMEOUT if timeout is None else timeout
        self._async_error = async_error or self._nccl_async_error
        self._abort = abort or self._nccl_abort
        self.aborted = False

    def _nccl_async_error(self):
        lib = native.load()
        if lib.hbgpu_comm_async_error(self.comm) != 0:
            return lib.hbgpu_last_error().decode(errors="replace")
        return None

    def _nccl_abort(self):
        native.load().hbgpu_comm_abort(self.comm)

    def abort(self):
        if not self.aborted:
            self.aborted = True
            self._abort()

    def failed_peer(self):
        if self.store is None:
            return None
        try:
            if self.store.check([self.KEY]):
                return int(self.store.get(self.KEY))
        except Exception:
            return None
        return None

    def notify_failure(self):
        if self.store is not None:
            try:
                self.store.compare_set(self.KEY, "", str(self.rank))
            except Exception:
                pass
        self.abort()

    def check(self):
        msg = self._async_error()
        if msg is not None:
            self.abort()
            raise CollectiveError(f"rank {self.rank}: {msg}")
        peer = self.failed_peer()
        if peer is not None and peer != self.rank:
            self.abort()
            raise RankFailure(peer, RunAborted(f"rank {self.rank} aborted: rank {peer} failed"))

    def wait(self, event):
        deadline = time.monotonic() + self.timeout
        while not event.query():
            self.check()
            if time.monotonic() > deadline:
                self.abort()
                raise CollectiveError(f"rank {self.rank}: device work did not complete within "
                                      f"{self.timeout:.0f} s (a peer stopped?)")
            time.sleep(self.POLL_S)
        self.check()

    def sync(self):
        """wait() for everything issued so far on torch's current stream (the
        engine joins its work back onto it; the collectives run on it)."""
        import torch
        ev = torch.cuda.Event()
        ev.record()
        self.wait(ev)


def _execute_loopback(spec, topology, partition, plan, iterations, out=((), ())):
    """spec.ranks engines on this GPU, one per rank of the reference partition,
    stepped stage by stage; the remote halo payloads move between their send
    and receive buffers by device copies in place of NCCL.  This runs the
    multi-GPU data path -- fused pack in the stage kernel, per-peer segments,
    unpack -- on one device."""
    import torch
    device = spec.device if spec.device is not None else torch.cuda.current_device()
    nr = spec.ranks
    ranks = []
    try:
        for r in range(nr):
            ranks.append(_new_rank(spec, topology, partition, plan, r, device, None, iterations))
        lib = native.load()
        recv_index = [{peer: (off, cnt) for peer, off, cnt in dr.layout.recvs} for dr in ranks]

        def transport():
            for r, dr in enumerate(ranks):
                for peer, off, cnt in dr.layout.sends:
                    roff, rcnt = recv_index[peer][r]
                    if rcnt != cnt:
                        raise ProtocolError(f"rank {r} -> {peer}: {cnt} != {rcnt} doubles")
                    ranks[peer].recvbuf[roff:roff + cnt].copy_(dr.sendbuf[off:off + cnt])

        def phase(p, exchange):
            if split and 0 <= p < 4 and (not ranks[0].fused or p in (1, 3)):
                # the multi-GPU engine's overlapped schedule (hb_runtime.cu
                # run_split): boundary tiles + remote packs, then the payload
                # transfer on a side stream concurrently with the interior
                # tiles, then the unpack once both are done
                for dr in ranks:
                    native.check(lib.hbgpu_engine_step_split(dr.engine, p, 0, dr.stream()),
                                 "hbgpu_engine_step_split")
                fork = torch.cuda.Event()
                fork.record()
                with torch.cuda.stream(side):
                    side.wait_event(fork)
                    transport()
                join = torch.cuda.Event()
                join.record(side)
                for dr in ranks:
                    native.check(lib.hbgpu_engine_step_split(dr.engine, p, 1, dr.stream()),
                                 "hbgpu_engine_step_split")
                torch.cuda.current_stream().wait_event(join)
                for dr in ranks:
                    native.check(lib.hbgpu_engine_unpack(dr.engine, p, dr.stream()), "hbgpu_engine_unpack")
                return
            for dr in ranks:
                native.check(lib.hbgpu_engine_step(dr.engine, p, dr.stream()), "hbgpu_engine_step")
            if exchange:
                transport()
                for dr in ranks:
                    native.check(lib.hbgpu_engine_unpack(dr.engine, p, dr.stream()), "hbgpu_engine_unpack")

        # spec.transport "loopback-split": every pass phase as the overlapped
        # boundary / transfer + interior / unpack schedule of the NCCL engine
        split = spec.transport == "loopback-split"
        side = torch.cuda.Stream(device)
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        phase(-1, True)
        chunk = poll_interval(topology, spec.case.planes, max(1, iterations))
        for it in range(iterations):
            for st in range(4):
                phase(st, True)
            phase(4, False)
            if (it + 1) % chunk == 0 and first_event(dr.divergence() for dr in ranks) is not None:
                break
        torch.cuda.synchronize(device)
        loop_s = time.perf_counter() - t0
        raise_divergence(first_event(dr.divergence() for dr in ranks))
        fields = {}
        for dr in ranks:
            fields.update(dr.fields(0, pinned_out=spec.output))
        norms = _norm_totals(_global_sumsq(ranks, len(topology.blocks), iterations), iterations,
                             ranks[0].stream())
        if iterations > 0:
            stacked = torch.stack([dr.force_history_array(iterations).reshape(-1) for dr in ranks])
            count = stacked.shape[1]
            folded = torch.empty(count, dtype=torch.float64, device=stacked.device)
            if count:
                native.check(lib.hbgpu_ordered_fold(_ptr(stacked), nr, count, _ptr(folded), ranks[0].stream()),
                             "hbgpu_ordered_fold")
            hist = folded.cpu().numpy().reshape(iterations, 3, spec.case.planes, spec.case.nbody)
        else:
            hist = _history(ranks[0], 0)
        torch.cuda.synchronize(device)
        _write_outputs(ranks, out)
    finally:
        for dr in ranks:
            dr.close()
    return fields, hist, norms, loop_s


def _reduce_history(dr, hist, world):
    """All-gather every rank's force history and fold it in rank order."""
    import torch
    count = hist.numel()
    if count == 0:
        return hist
    stacked = torch.empty(world * count, dtype=torch.float64, device=dr.device)
    src = hist.contiguous().view(-1)
    native.check(dr.lib.hbgpu_comm_allgather(dr.comm, _ptr(src), _ptr(stacked), count, dr.stream()),
                 "hbgpu_comm_allgather")
    out = torch.empty(count, dtype=torch.float64, device=dr.device)
    native.check(dr.lib.hbgpu_ordered_fold(_ptr(stacked), world, count, _ptr(out), dr.stream()),
                 "hbgpu_ordered_fold")
    return out.view_as(hist)
