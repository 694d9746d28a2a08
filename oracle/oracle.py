"""CPU oracle for the HB residual-and-smoothing loop -- TEST INFRASTRUCTURE ONLY.

This module restates the reference (`hbproxy`, /root/reference/pkg/src/hbproxy)
algorithm for the hot path so that the CUDA path can be checked against it on
hosts where the reference itself is absent (the GPU box).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import it; the product package never does.

Pinning: tests/test_oracle_golden.py checks this restatement against golden
vectors produced by running the reference itself (tests/golden/make_golden.py),
including the reference's full-run fingerprints.

What is restated, and from where:
  spectral_matrix      hbcore.py:74-96
  initial_values       hbcore.py:148-162
  forcing_values       hbcore.py:165-177
  residual / update    hbcore.py:184-245  (C, oracle/hb_oracle.c)
  divergence locator   hbcore.py:279-284
  face views           hbcore.py:291-322
  compute_forces       hbcore.py:359-382
  halo exchange        exchange.py:121-149 (plan), 195-202, 260-261 (copy)
  run loop             driver.py:110-149   (priming exchange, 4 RK stages,
                                            forces once per iteration)
  rank-ordered sum     runtime.py:290-294

The residual norm is NOT part of the reference: it is
defined here as sqrt(fsum over blocks ascending of R**2) for the residual
evaluated in stage one of each iteration.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

NPDE = 4
NU = 0.05
ADVECTION = 1.0
RK_ALPHAS = (0.25, 1.0 / 3.0, 0.5, 1.0)
TWO_PI = 2.0 * math.pi

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None


def build():
    """Compile oracle/hb_oracle.c (plain gcc, see oracle/Makefile)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "hb_oracle.c"))):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.c_void_p
        lg = ctypes.c_long
        L.oracle_residual.argtypes = [dp, dp, dp, ctypes.c_double, ctypes.c_double, dp,
                                      lg, lg, lg, lg, lg, lg, lg, lg]
        L.oracle_residual.restype = None
        L.oracle_update.argtypes = [dp, dp, dp, ctypes.c_double, ctypes.c_int,
                                    lg, lg, lg, lg, lg, lg, lg, lg]
        L.oracle_update.restype = ctypes.c_double
        L.oracle_stage_many.argtypes = [ctypes.c_int, dp, dp, dp, dp, dp, dp, dp, dp, dp,
                                        lg, lg, ctypes.c_double, ctypes.c_int, ctypes.c_int, dp]
        L.oracle_stage_many.restype = ctypes.c_int
        L.oracle_stage_lean.argtypes = [ctypes.c_int, dp, dp, dp, dp, dp, dp, dp, dp, dp,
                                        lg, lg, ctypes.c_double, ctypes.c_int, ctypes.c_int, dp, dp]
        L.oracle_stage_lean.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data


# ---------------------------------------------------------------------------
# Operator pieces
# ---------------------------------------------------------------------------

def spectral_matrix(nharms, omega):
    """hbcore.py:74-96: D[j,k] = (omega/2)(-1)^d / sin(pi d / N), d wrapped."""
    n = 2 * nharms + 1
    mat = np.zeros((n, n))
    for j in range(n):
        for k in range(n):
            if j != k:
                d = (j - k + nharms) % n - nharms
                mat[j, k] = 0.5 * omega * (-1.0) ** d / math.sin(math.pi * d / n)
    return mat


def cell_centres(spec):
    xc = spec.x0 + (np.arange(1, spec.ni + 1) - 0.5) * spec.h
    yc = spec.y0 + (np.arange(1, spec.nj + 1) - 0.5) * spec.h
    return xc, yc


def initial_values(spec, planes, npde=NPDE):
    """hbcore.py:148-162 over the full interior: 0.1 sin(2pi x+.35p) cos(2pi y-.2n)."""
    xc, yc = cell_centres(spec)
    a = np.sin(TWO_PI * xc[None, :] + 0.35 * np.arange(npde, dtype=np.float64)[:, None])
    b = np.cos(TWO_PI * yc[None, :] - 0.2 * np.arange(0, planes, dtype=np.float64)[:, None])
    return 0.1 * a[None, :, None, :] * b[:, None, :, None]


def forcing_values(spec, planes, npde=NPDE):
    """hbcore.py:165-177: amp(n) (1 + .25p) sin(2pi x) sin(2pi y)."""
    xc, yc = cell_centres(spec)
    sxy = np.sin(TWO_PI * xc)[None, :] * np.sin(TWO_PI * yc)[:, None]
    amp = np.zeros(planes)
    if planes > 1:
        amp[1] = 0.8
    if planes > 2:
        amp[2] = -0.5
    pfac = 1.0 + 0.25 * np.arange(npde, dtype=np.float64)
    out = amp[:, None, None, None] * pfac[None, :, None, None] * sxy[None, None, :, :]
    return np.ascontiguousarray(out)


def residual_into(q, dmat, src, h, out, n_lo, n_hi, j_lo, j_hi):
    """_residual_kernel with the host-side coefficient arithmetic of hbcore.py:255-258."""
    P, npde, nj2, ni2 = q.shape
    lib().oracle_residual(_ptr(q), _ptr(np.ascontiguousarray(dmat)), _ptr(src),
                          NU / (h * h), ADVECTION / (2.0 * h), _ptr(out),
                          P, npde, nj2, ni2, n_lo, n_hi, j_lo, j_hi)


def update(q, q0, resid, coef, snapshot, n_lo, n_hi, j_lo, j_hi):
    P, npde, nj2, ni2 = q.shape
    return lib().oracle_update(_ptr(q), _ptr(q0), _ptr(resid), coef, int(bool(snapshot)),
                               P, npde, nj2, ni2, n_lo, n_hi, j_lo, j_hi)


def divergence_location(q):
    """hbcore.py:279-284: lexicographically first non-finite interior value ->
    (i, j, p, n) with 1-based i/j."""
    interior = q[:, :, 1:-1, 1:-1]
    bad = np.argwhere(~np.isfinite(interior))
    n, p, j, i = (int(v) for v in bad[0])
    return i + 1, j + 1, p, n


# ---------------------------------------------------------------------------
# Faces, exchange and forces
# ---------------------------------------------------------------------------

def face_interior(q, face, lo, hi):
    nj, ni = q.shape[2] - 2, q.shape[3] - 2
    return {"south": lambda: q[:, :, 1, lo:hi + 1], "north": lambda: q[:, :, nj, lo:hi + 1],
            "west": lambda: q[:, :, lo:hi + 1, 1], "east": lambda: q[:, :, lo:hi + 1, ni]}[face]()


def face_halo(q, face, lo, hi):
    nj, ni = q.shape[2] - 2, q.shape[3] - 2
    return {"south": lambda: q[:, :, 0, lo:hi + 1], "north": lambda: q[:, :, nj + 1, lo:hi + 1],
            "west": lambda: q[:, :, lo:hi + 1, 0], "east": lambda: q[:, :, lo:hi + 1, ni + 1]}[face]()


def exchange(qs, cuts):
    """All cut directions of one exchange (every block local): direction 0
    fills side_a's halo from side_b, direction 1 the reverse, a reversed cut
    flipping the side_b range (exchange.py:133-144, 195-202)."""
    for cut in cuts:
        a, b = cut.side_a, cut.side_b
        src = face_interior(qs[b.block], b.face, b.lo, b.hi)
        if cut.reversed:
            src = src[:, :, ::-1]
        face_halo(qs[a.block], a.face, a.lo, a.hi)[...] = src
        src = face_interior(qs[a.block], a.face, a.lo, a.hi)
        dst = face_halo(qs[b.block], b.face, b.lo, b.hi)
        if cut.reversed:
            dst = dst[:, :, ::-1]
        dst[...] = src


def compute_forces(qs, blocks, planes, nbody):
    """hbcore.py:359-382: strict left-to-right sum of h*q over body faces."""
    out = np.zeros((3, planes, nbody))
    for spec in sorted(blocks, key=lambda s: s.id):
        q = qs[spec.id]
        for face, body in spec.body_faces:
            extent = spec.ni if face in ("north", "south") else spec.nj
            view = face_interior(q, face, 1, extent)
            for n in range(planes):
                for k in range(3):
                    total = out[k, n, body]
                    for v in view[n, k].tolist():
                        total += spec.h * v
                    out[k, n, body] = total
    return out


def ordered_sum(buffers):
    """runtime.py:290-294: acc = buf[0] + buf[1] + ... in ascending rank order."""
    acc = np.array(buffers[0], dtype=np.float64, copy=True)
    for b in buffers[1:]:
        acc += b
    return acc


def partition_blocks(blocks, nranks):
    """mesh.py:352-373: greedy LPT, descending cells, ties ascending id/rank."""
    import heapq
    order = sorted(blocks, key=lambda b: (-(b.ni * b.nj), b.id))
    heap = [(0, r) for r in range(nranks)]
    assign = [0] * len(blocks)
    for b in order:
        load, r = heapq.heappop(heap)
        assign[b.id] = r
        heapq.heappush(heap, (load + b.ni * b.nj, r))
    return tuple(assign)


# ---------------------------------------------------------------------------
# Run loop
# ---------------------------------------------------------------------------

class OracleDivergence(Exception):
    def __init__(self, iteration, stage, block, i, j, p, n):
        self.iteration, self.stage = iteration, stage
        self.block, self.i, self.j, self.p, self.n = block, i, j, p, n
        super().__init__(f"non-finite value in block {block} at (i={i}, j={j}, pde={p}, "
                         f"plane={n}) [iteration {iteration}, stage {stage}]")


@dataclass
class OracleResult:
    fields: dict
    forces: np.ndarray             # (3, planes, nbody): cl, cd, cm
    norms: list = field(default_factory=list)
    force_history: list = field(default_factory=list)
    loop_s: float = 0.0


class OracleSolver:
    """Single-rank restatement of driver._rank_program (driver.py:110-149),
    steppable so bench.py can time iterations.

    `case` is any object with the reference CaseConfig attributes.  `initial`
    optionally maps a BlockSpec to the (planes, npde, nj, ni) initial interior
    (the hbcore.initial_values hook); default is the reference's IC.
    """

    def __init__(self, case, initial=None, nthreads=None, record_norms=True,
                 record_forces=False):
        self.case = case
        self.planes = planes = 2 * case.nharms + 1
        self.npde = npde = case.npde
        self.blocks = blocks = sorted(case.blocks, key=lambda s: s.id)
        self.nthreads = nthreads or max(1, len(os.sched_getaffinity(0)))
        self.dmat = np.ascontiguousarray(spectral_matrix(case.nharms, case.omega))
        self.qs, self.q0s, self.rs, self.srcs = {}, {}, {}, {}
        for s in blocks:
            self.qs[s.id] = np.zeros((planes, npde, s.nj + 2, s.ni + 2))
            self.q0s[s.id] = np.zeros_like(self.qs[s.id])
            self.rs[s.id] = np.zeros((planes, npde, s.nj, s.ni))
            self.srcs[s.id] = forcing_values(s, planes, npde)
            ic = initial(s, planes, npde) if initial is not None else initial_values(s, planes, npde)
            self.qs[s.id][:, :, 1:s.nj + 1, 1:s.ni + 1] = ic
        self.alpha_dtau = [a * case.dtau for a in RK_ALPHAS]
        arr = lambda vals, t: np.array(vals, dtype=t)  # noqa: E731
        self._q = arr([_ptr(self.qs[s.id]) for s in blocks], np.uintp)
        self._q0 = arr([_ptr(self.q0s[s.id]) for s in blocks], np.uintp)
        self._r = arr([_ptr(self.rs[s.id]) for s in blocks], np.uintp)
        self._s = arr([_ptr(self.srcs[s.id]) for s in blocks], np.uintp)
        self._ni = arr([s.ni for s in blocks], np.int64)
        self._nj = arr([s.nj for s in blocks], np.int64)
        self._nu = arr([NU / (s.h * s.h) for s in blocks], np.float64)
        self._adv = arr([ADVECTION / (2.0 * s.h) for s in blocks], np.float64)
        self._accs = np.zeros(len(blocks) * planes)
        self.record_norms, self.record_forces = record_norms, record_forces
        self.result = OracleResult(fields=self.qs, forces=np.zeros((3, planes, case.nbody)))
        self.done = 0

    def prime(self):
        exchange(self.qs, self.case.cuts)  # priming exchange (driver.py:129)

    def iterate(self, iterations):
        L = lib()
        nb = len(self.blocks)
        for _ in range(iterations):
            for stage in range(4):
                bad = L.oracle_stage_many(nb, _ptr(self._q), _ptr(self._q0), _ptr(self._r),
                                          _ptr(self._s), _ptr(self._ni), _ptr(self._nj),
                                          _ptr(self._nu), _ptr(self._adv), _ptr(self.dmat),
                                          self.planes, self.npde, self.alpha_dtau[stage],
                                          int(stage == 0), self.nthreads, _ptr(self._accs))
                if stage == 0 and self.record_norms:
                    self.result.norms.append(_norm(self.rs[s.id] for s in self.blocks))
                if bad:
                    for s in self.blocks:
                        if not np.all(np.isfinite(self.qs[s.id][:, :, 1:-1, 1:-1])):
                            raise OracleDivergence(self.done, stage, s.id,
                                                   *divergence_location(self.qs[s.id]))
                exchange(self.qs, self.case.cuts)
            forces = compute_forces(self.qs, self.blocks, self.planes, self.case.nbody)
            self.result.forces = forces
            if self.record_forces:
                self.result.force_history.append(forces.copy())
            self.done += 1
        return self.result

    @property
    def units_per_iteration(self):
        return sum(s.ni * s.nj for s in self.blocks) * self.planes * 4


class LeanOracleSolver(OracleSolver):
    """The same run loop holding only q and q0 per block (BASELINE C3/C4 at
    full size: C4 needs 38.8 GB instead of the reference's 77.5 GB).  The
    stage is oracle_stage_lean (hb_oracle.c): forcing formed on the fly as
    (amp[n] pfac[p]) * sxy -- bitwise forcing_values() -- and a 2-row residual
    scratch per (block, pde).  Norms: per-block compensated sums of R**2,
    combined with math.fsum (rtol 1e-12 against the fsum definition)."""

    def __init__(self, case, initial=None, nthreads=None, record_norms=True,
                 record_forces=False):
        self.case = case
        self.planes = planes = 2 * case.nharms + 1
        self.npde = npde = case.npde
        self.blocks = blocks = sorted(case.blocks, key=lambda s: s.id)
        self.nthreads = nthreads or max(1, len(os.sched_getaffinity(0)))
        self.dmat = np.ascontiguousarray(spectral_matrix(case.nharms, case.omega))
        amp = np.zeros(planes)
        if planes > 1:
            amp[1] = 0.8
        if planes > 2:
            amp[2] = -0.5
        pfac = 1.0 + 0.25 * np.arange(npde, dtype=np.float64)
        self.ap = np.ascontiguousarray(amp[:, None] * pfac[None, :])   # (planes, npde)
        self.qs, self.q0s, self.sxys = {}, {}, {}
        for s in blocks:
            self.qs[s.id] = np.zeros((planes, npde, s.nj + 2, s.ni + 2))
            self.q0s[s.id] = np.zeros_like(self.qs[s.id])
            xc, yc = cell_centres(s)
            self.sxys[s.id] = np.ascontiguousarray(
                np.sin(TWO_PI * xc)[None, :] * np.sin(TWO_PI * yc)[:, None])
            ic = initial(s, planes, npde) if initial is not None else initial_values(s, planes, npde)
            self.qs[s.id][:, :, 1:s.nj + 1, 1:s.ni + 1] = ic
        self.alpha_dtau = [a * case.dtau for a in RK_ALPHAS]
        arr = lambda vals, t: np.array(vals, dtype=t)  # noqa: E731
        self._q = arr([_ptr(self.qs[s.id]) for s in blocks], np.uintp)
        self._q0 = arr([_ptr(self.q0s[s.id]) for s in blocks], np.uintp)
        self._sxy = arr([_ptr(self.sxys[s.id]) for s in blocks], np.uintp)
        self._ni = arr([s.ni for s in blocks], np.int64)
        self._nj = arr([s.nj for s in blocks], np.int64)
        self._nu = arr([NU / (s.h * s.h) for s in blocks], np.float64)
        self._adv = arr([ADVECTION / (2.0 * s.h) for s in blocks], np.float64)
        self._sumsq = np.zeros(len(blocks))
        self._bad = np.zeros(len(blocks), dtype=np.int32)
        self.record_norms, self.record_forces = record_norms, record_forces
        self.result = OracleResult(fields=self.qs, forces=np.zeros((3, planes, case.nbody)))
        self.done = 0

    def iterate(self, iterations):
        L = lib()
        nb = len(self.blocks)
        for _ in range(iterations):
            for stage in range(4):
                want_norm = stage == 0 and self.record_norms
                bad = L.oracle_stage_lean(nb, _ptr(self._q), _ptr(self._q0), _ptr(self._sxy),
                                          _ptr(self._ni), _ptr(self._nj), _ptr(self._nu),
                                          _ptr(self._adv), _ptr(self.dmat), _ptr(self.ap),
                                          self.planes, self.npde, self.alpha_dtau[stage],
                                          int(stage == 0), self.nthreads,
                                          _ptr(self._sumsq) if want_norm else None,
                                          _ptr(self._bad))
                if want_norm:
                    try:
                        self.result.norms.append(math.sqrt(math.fsum(self._sumsq.tolist())))
                    except (OverflowError, ValueError):
                        self.result.norms.append(math.inf)
                if bad:
                    for k, s in enumerate(self.blocks):
                        if self._bad[k]:
                            raise OracleDivergence(self.done, stage, s.id,
                                                   *divergence_location(self.qs[s.id]))
                exchange(self.qs, self.case.cuts)
            forces = compute_forces(self.qs, self.blocks, self.planes, self.case.nbody)
            self.result.forces = forces
            if self.record_forces:
                self.result.force_history.append(forces.copy())
            self.done += 1
        return self.result


def run(case, iterations=None, initial=None, nthreads=None, record_norms=True,
        record_forces=False, lean=False):
    """Single-rank restatement of driver.run_case: prime, iterate, return fields/forces.
    lean=True holds only q and q0 (LeanOracleSolver)."""
    import time
    iterations = case.iterations if iterations is None else iterations
    cls = LeanOracleSolver if lean else OracleSolver
    solver = cls(case, initial, nthreads, record_norms, record_forces)
    t0 = time.perf_counter()
    solver.prime()
    result = solver.iterate(iterations)
    result.loop_s = time.perf_counter() - t0
    return result


def _norm(resids):
    """sqrt(exactly rounded sum of R**2) over blocks ascending; inf/nan once
    the run has diverged."""
    with np.errstate(over="ignore", invalid="ignore"):
        parts = [(r * r).ravel() for r in resids]
    try:
        return math.sqrt(math.fsum(math.fsum(p) for p in parts))
    except OverflowError:
        return math.inf


def fingerprint(fields, forces):
    """sha256[:16] over fields (blocks ascending, halos included) then cl/cd/cm."""
    import hashlib
    h = hashlib.sha256()
    for b in sorted(fields):
        h.update(np.ascontiguousarray(fields[b]).tobytes())
    for k in range(3):
        h.update(np.ascontiguousarray(forces[k]).tobytes())
    return h.hexdigest()[:16]
