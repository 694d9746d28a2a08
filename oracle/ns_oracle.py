"""CPU checker for the north-star HB Euler / NS path -- TEST INFRASTRUCTURE ONLY.

Drives oracle/ns_oracle.c (a restatement of the specification in
paper_1304_7654_b200/nsflow.py, written independently of hb_ns.cu) through the
same run loop as the GPU solver: per RK stage, cut halos (two layers, numpy
copies), boundary + corner halos, the local time step at stage 1, the spatial
residual, the HB source + update; forces after each iteration.

Parity is UNPINNED: the reference (hbproxy) has no flux physics
(hbcore.py:3-13), so nothing pins this checker to a reference
output.  Only tests/ may import it.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "build", "libnsoracle.so")
_lib = None
RK_ALPHAS = (0.25, 1.0 / 3.0, 0.5, 1.0)
NG = 2


class NSBlockC(ctypes.Structure):
    _fields_ = [("ni", ctypes.c_int), ("nj", ctypes.c_int), ("P", ctypes.c_int), ("Pg", ctypes.c_int),
                ("x", ctypes.c_void_p), ("y", ctypes.c_void_p), ("xt", ctypes.c_void_p), ("yt", ctypes.c_void_p),
                ("kinds", ctypes.c_int * 4),
                ("xc", ctypes.c_void_p), ("yc", ctypes.c_void_p), ("vol", ctypes.c_void_p),
                ("six", ctypes.c_void_p), ("siy", ctypes.c_void_p), ("gi", ctypes.c_void_p),
                ("sjx", ctypes.c_void_p), ("sjy", ctypes.c_void_p), ("gj", ctypes.c_void_p)]


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "ns_oracle.c")
        if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        L = ctypes.CDLL(_LIB)
        vp, bp = ctypes.c_void_p, ctypes.POINTER(NSBlockC)
        L.ns_geometry.argtypes = [bp]
        L.ns_boundaries.argtypes = [bp, vp, vp]
        L.ns_residual.argtypes = [bp, vp, vp, ctypes.c_double]
        L.ns_timestep.argtypes = [bp, vp, vp, ctypes.c_double, ctypes.c_double, ctypes.c_double]
        L.ns_update.argtypes = [bp, vp, vp, vp, vp, vp, vp, ctypes.c_double, ctypes.c_int,
                                ctypes.POINTER(ctypes.c_longdouble)]
        L.ns_update.restype = ctypes.c_int
        L.ns_forces.argtypes = [bp, vp, vp, vp, vp]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


class OracleNSBlock:
    def __init__(self, case, blk):
        P, ni, nj = case.planes, blk.ni, blk.nj
        self.spec, self.P = blk, P
        self.x = np.ascontiguousarray(blk.x, dtype=np.float64)
        self.y = np.ascontiguousarray(blk.y, dtype=np.float64)
        self.xt = None if blk.xt is None else np.ascontiguousarray(blk.xt, dtype=np.float64)
        self.yt = None if blk.yt is None else np.ascontiguousarray(blk.yt, dtype=np.float64)
        Pg = self.x.shape[0]
        e = lambda *s: np.zeros(s)  # noqa: E731
        self.geo = {"xc": e(Pg, nj + 4, ni + 4), "yc": e(Pg, nj + 4, ni + 4), "vol": e(Pg, nj + 4, ni + 4),
                    "six": e(Pg, nj + 4, ni + 5), "siy": e(Pg, nj + 4, ni + 5), "gi": e(Pg, nj + 4, ni + 5),
                    "sjx": e(Pg, nj + 5, ni + 4), "sjy": e(Pg, nj + 5, ni + 4), "gj": e(Pg, nj + 5, ni + 4)}
        c = NSBlockC()
        c.ni, c.nj, c.P, c.Pg = ni, nj, P, Pg
        c.x, c.y, c.xt, c.yt = _p(self.x), _p(self.y), _p(self.xt), _p(self.yt)
        for k in range(4):
            c.kinds[k] = blk.kinds[k]
        for k, v in self.geo.items():
            setattr(c, k, _p(v))
        self.c = c
        lib().ns_geometry(ctypes.byref(c))
        if self.xt is None:
            del self.geo["gi"], self.geo["gj"]
        self.slots = [np.zeros((P, 4, nj + 4, ni + 4)) for _ in range(3)]
        self.r = np.zeros((P, 4, nj, ni))
        self.dt = np.zeros((nj, ni))


def _interior(q, blk, side, k, lo, hi):
    ni, nj = blk.ni, blk.nj
    if side == "south":
        return q[:, :, k + 1, lo + 1:hi + 2]
    if side == "north":
        return q[:, :, nj + 2 - k, lo + 1:hi + 2]
    if side == "west":
        return q[:, :, lo + 1:hi + 2, k + 1]
    return q[:, :, lo + 1:hi + 2, ni + 2 - k]


def _halo(q, blk, side, k, lo, hi):
    ni, nj = blk.ni, blk.nj
    if side == "south":
        return q[:, :, 2 - k, lo + 1:hi + 2]
    if side == "north":
        return q[:, :, nj + 1 + k, lo + 1:hi + 2]
    if side == "west":
        return q[:, :, lo + 1:hi + 2, 2 - k]
    return q[:, :, lo + 1:hi + 2, ni + 1 + k]


def cut_exchange(blocks, cuts, slot):
    """Two halo layers of every cut, both directions (plain copies)."""
    for c in cuts:
        A, B = blocks[c.a], blocks[c.b]
        qa, qb = A.slots[slot], B.slots[slot]
        for k in (1, 2):
            _halo(qa, A.spec, c.face_a, k, c.lo, c.hi)[...] = _interior(qb, B.spec, c.face_b, k, c.lo, c.hi)
            _halo(qb, B.spec, c.face_b, k, c.lo, c.hi)[...] = _interior(qa, A.spec, c.face_a, k, c.lo, c.hi)


class NSDivergence(Exception):
    def __init__(self, block, iteration, stage):
        self.block, self.iteration, self.stage = block, iteration, stage
        super().__init__(f"non-finite state in block {block} at iteration {iteration}, stage {stage}")


class OracleNS:
    def __init__(self, case, initial=None):
        from paper_1304_7654_b200 import nsflow
        self.case = case
        self.blocks = {b.id: OracleNSBlock(case, b) for b in case.blocks}
        self.order = sorted(self.blocks)
        self.winf = np.ascontiguousarray(nsflow.freestream(case))
        self.dmat = np.ascontiguousarray(nsflow.spectral_matrix(case))
        for bid, ob in self.blocks.items():
            ob.slots[0][...] = initial(ob.spec) if initial is not None else nsflow.initial_state(case, ob.spec)
        self.norms, self.forces = [], []
        self.done = 0

    def fill(self, slot):
        L = lib()
        cut_exchange(self.blocks, self.case.cuts, slot)
        for bid in self.order:
            ob = self.blocks[bid]
            L.ns_boundaries(ctypes.byref(ob.c), _p(ob.slots[slot]), _p(self.winf))

    def iterate(self, iterations):
        L = lib()
        case = self.case
        onh = case.omega * case.nharms
        for _ in range(iterations):
            sumsq = ctypes.c_longdouble(0.0)
            for st, (si, so) in enumerate(((0, 1), (1, 2), (2, 1), (1, 0))):
                self.fill(si)
                for bid in self.order:
                    ob = self.blocks[bid]
                    if st == 0:
                        L.ns_timestep(ctypes.byref(ob.c), _p(ob.slots[0]), _p(ob.dt), case.mu, case.cfl, onh)
                    L.ns_residual(ctypes.byref(ob.c), _p(ob.slots[si]), _p(ob.r), case.mu)
                    bad = L.ns_update(ctypes.byref(ob.c), _p(ob.slots[si]), _p(ob.slots[0]), _p(ob.slots[so]),
                                      _p(ob.r), _p(ob.dt), _p(self.dmat), RK_ALPHAS[st], int(st == 0),
                                      ctypes.byref(sumsq))
                    if bad:
                        raise NSDivergence(bid, self.done, st)
                if st == 0:
                    self.norms.append(math.sqrt(float(sumsq.value)))
            self.forces.append(self.force_coefficients())
            self.done += 1
        return self

    def force_coefficients(self):
        """(P, 2) (cl, cd): wall pressure forces folded over blocks ascending,
        rotated into the snapshot's freestream axes."""
        P = self.case.planes
        fxy = np.zeros((P, 2))
        for bid in self.order:
            ob = self.blocks[bid]
            lib().ns_forces(ctypes.byref(ob.c), _p(ob.slots[0]), None, None, _p(fxy))
        ang = np.radians(self.case.dalpha_deg) * np.sin(2 * np.pi * np.arange(P) / P)
        ca, sa = np.cos(ang), np.sin(ang)
        cd = fxy[:, 0] * ca + fxy[:, 1] * sa
        cl = fxy[:, 1] * ca - fxy[:, 0] * sa
        return np.stack([cl, cd], axis=1)

    def fields(self):
        return {bid: ob.slots[0] for bid, ob in self.blocks.items()}


def run(case, iterations=None, initial=None):
    o = OracleNS(case, initial)
    o.iterate(case.iterations if iterations is None else iterations)
    return o
