"""Case builders, the bundled catalog, and the BASELINE.json workloads.

The four topology builders and the six catalog cases reproduce the
reference's (cases.py:39-147): same block origins, cut lists and bodies, so
block/halo indexing is identical.  The catalog is generated in-process rather
than shipped as .cfg text (the reference's .cfg files are themselves the
output of its case_text over these builders, cases.py:156-183).

BASELINE.json's five configurations describe Euler/Navier-Stokes physics the
reference operator cannot express.  `baseline_workload`
maps each onto the reference operator with the configuration's block layout,
cell counts, snapshot count and iteration count, plus a
seeded freestream-like initial state.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .casefile import parse_case, case_text
from .topology import BlockSpec, CaseConfig, CutSide, CutSpec


def _bodies_by_block(bodies):
    table = {}
    for blk, face, body in bodies:
        table.setdefault(blk, []).append((face, body))
    return table


def _row(nblocks, ni, nj, h, bodies):
    faces = _bodies_by_block(bodies)
    return [BlockSpec(id=k, ni=ni, nj=nj, x0=k * ni * h, y0=0.0, h=h,
                      body_faces=tuple(faces.get(k, ()))) for k in range(nblocks)]


def _case(nharms, iterations, dtau, omega, nbody, blocks, cuts, name):
    return CaseConfig(nharms=nharms, npde=4, iterations=iterations, dtau=dtau,
                      omega=omega, nbody=nbody, blocks=blocks, cuts=cuts, name=name)


def ring_case(nblocks, ni, nj, nharms, *, h, dtau, omega=1.0, iterations=10,
              nbody=0, bodies=(), name=""):
    """Blocks in a row, block k's east face joined to block (k+1) mod n's west face."""
    if nblocks < 2:
        raise ValueError("a ring needs at least 2 blocks")
    cuts = [CutSpec(CutSide(k, "east", 1, nj), CutSide((k + 1) % nblocks, "west", 1, nj))
            for k in range(nblocks)]
    return _case(nharms, iterations, dtau, omega, nbody,
                 _row(nblocks, ni, nj, h, bodies), cuts, name)


def pair_case(ni, nj, nharms, *, h, dtau, omega=1.0, iterations=10,
              nbody=0, bodies=(), reversed_cut=False, name=""):
    """Two blocks side by side sharing one east/west cut."""
    cuts = [CutSpec(CutSide(0, "east", 1, nj), CutSide(1, "west", 1, nj),
                    reversed=reversed_cut)]
    return _case(nharms, iterations, dtau, omega, nbody,
                 _row(2, ni, nj, h, bodies), cuts, name)


def stacked_pair_case(ni, nj, nharms, *, h, dtau, omega=1.0, iterations=1,
                      nbody=0, bodies=(), name=""):
    """Two blocks stacked in y sharing one north/south cut of length ni."""
    faces = _bodies_by_block(bodies)
    blocks = [BlockSpec(id=k, ni=ni, nj=nj, x0=0.0, y0=k * nj * h, h=h,
                        body_faces=tuple(faces.get(k, ()))) for k in range(2)]
    cuts = [CutSpec(CutSide(0, "north", 1, ni), CutSide(1, "south", 1, ni))]
    return _case(nharms, iterations, dtau, omega, nbody, blocks, cuts, name)


def lattice_case(nbx, nby, ni, nj, nharms, *, h, dtau, omega=1.0, iterations=10,
                 nbody=0, bodies=(), name=""):
    """nbx x nby lattice (block id = row*nbx + col): all east/west cuts row by
    row, then all north/south cuts."""
    faces = _bodies_by_block(bodies)
    blocks = [BlockSpec(id=r * nbx + c, ni=ni, nj=nj, x0=c * ni * h, y0=r * nj * h, h=h,
                        body_faces=tuple(faces.get(r * nbx + c, ())))
              for r in range(nby) for c in range(nbx)]
    cuts = [CutSpec(CutSide(r * nbx + c, "east", 1, nj), CutSide(r * nbx + c + 1, "west", 1, nj))
            for r in range(nby) for c in range(nbx - 1)]
    cuts += [CutSpec(CutSide(r * nbx + c, "north", 1, ni),
                     CutSide((r + 1) * nbx + c, "south", 1, ni))
             for r in range(nby - 1) for c in range(nbx)]
    return _case(nharms, iterations, dtau, omega, nbody, blocks, cuts, name)


# ---------------------------------------------------------------------------
# Bundled catalog (reference cases.py:116-153)
# ---------------------------------------------------------------------------

def tc_tiny():
    return pair_case(4, 4, nharms=1, h=0.25, dtau=0.05, iterations=10,
                     nbody=1, bodies=((0, "south", 0),), name="tc-tiny")


def tc1_mini():
    return ring_case(32, 32, 32, nharms=7, h=0.03125, dtau=0.004, iterations=20,
                     nbody=2, bodies=((0, "south", 0), (16, "south", 1)), name="tc1-mini")


def tc2_mini():
    return lattice_case(8, 8, 32, 32, nharms=4, h=0.03125, dtau=0.004, iterations=10,
                        nbody=1, bodies=((0, "south", 0),), name="tc2-mini")


def cut2500():
    return stacked_pair_case(2500, 4, nharms=1, h=0.01, dtau=0.0001, iterations=1,
                             nbody=1, bodies=((0, "south", 0),), name="cut2500")


def tc1_full():
    return ring_case(512, 32, 16, nharms=31, h=0.03125, dtau=0.004, iterations=100,
                     nbody=2, bodies=((0, "south", 0), (256, "south", 1)), name="tc1-full")


def tc2_full():
    return lattice_case(64, 32, 64, 32, nharms=17, h=0.015625, dtau=0.002, iterations=100,
                        nbody=1, bodies=((0, "south", 0),), name="tc2-full")


BUILDERS = {"tc-tiny": tc_tiny, "tc1-mini": tc1_mini, "tc2-mini": tc2_mini,
            "cut2500": cut2500, "tc1-full": tc1_full, "tc2-full": tc2_full}


def builtin_case_names():
    return tuple(BUILDERS)


def load_builtin(name):
    """A catalog case, round-tripped through the text format like a file load."""
    if name not in BUILDERS:
        raise KeyError(name)
    return parse_case(case_text(BUILDERS[name]()), source=f"<builtin {name}>", name=name)


# ---------------------------------------------------------------------------
# BASELINE.json workloads C0..C4 on the reference operator
# ---------------------------------------------------------------------------

GAMMA = 1.4
SEED_BASE = 13047654


@dataclass(frozen=True)
class Workload:
    """A BASELINE configuration expressed on the reference operator."""

    key: str
    case: CaseConfig
    mach: float
    pitch_deg: float
    description: str

    def initial(self, spec, planes, npde=4):
        return seeded_initial(spec, planes, npde, self.mach, self.pitch_deg)

    @property
    def units_per_iteration(self):
        """Cell-snapshot RK-stage updates per iteration (4 stages)."""
        return sum(b.cells() for b in self.case.blocks) * self.case.planes * 4


def freestream(planes, mach, pitch_deg):
    """q_inf(n) = (1, M cos a_n, M sin a_n, 1/(g(g-1)) + M^2/2), a_n = da sin(2 pi n/P)."""
    n = np.arange(planes, dtype=np.float64)
    alpha = math.radians(pitch_deg) * np.sin(2.0 * math.pi * n / planes)
    out = np.empty((planes, 4))
    out[:, 0] = 1.0
    out[:, 1] = mach * np.cos(alpha)
    out[:, 2] = mach * np.sin(alpha)
    out[:, 3] = 1.0 / (GAMMA * (GAMMA - 1.0)) + 0.5 * mach * mach
    return out


def seeded_initial(spec, planes, npde, mach, pitch_deg):
    """q_inf(n)[p] * (1 + 0.01 U(-1, 1)), U from default_rng(13047654 + block id).

    Keyed by block id, so it is independent of the block -> GPU partition.
    """
    rng = np.random.default_rng(SEED_BASE + spec.id)
    u = rng.uniform(-1.0, 1.0, size=(planes, npde, spec.nj, spec.ni))
    u *= 0.01
    u += 1.0
    u *= freestream(planes, mach, pitch_deg)[:, :npde, None, None]
    return u


def _dtau(h):
    # dtau * nu / h^2 = 0.2048, the ratio of the bundled tc1-mini case
    return 4.096 * h * h


def baseline_workload(key, iterations=None):
    """C0..C4 of BASELINE.json on the reference operator."""
    key = key.upper()
    if key == "C0":
        h = 1.0 / 64
        case = _case(1, 100, _dtau(h), 1.0, 0,
                     [BlockSpec(0, 64, 32, 0.0, 0.0, h)], [], "C0")
        wl = Workload("C0", case, 0.5, 1.0, "1 block 64x32, N_H=1 (P=3), 100 it")
    elif key == "C1":
        h = 1.0 / 512
        case = lattice_case(2, 2, 256, 128, 2, h=h, dtau=_dtau(h), iterations=200,
                            nbody=2, bodies=((0, "south", 0), (1, "south", 1)), name="C1")
        wl = Workload("C1", case, 0.3, 0.0, "2x2 blocks of 256x128, N_H=2 (P=5), 200 it")
    elif key == "C2":
        h = 1.0 / 512
        blk = BlockSpec(0, 512, 256, 0.0, 0.0, h, body_faces=(("south", 0),))
        cuts = [CutSpec(CutSide(0, "east", 1, 256), CutSide(0, "west", 1, 256))]
        case = _case(4, 500, _dtau(h), 0.12, 1, [blk], cuts, "C2")
        wl = Workload("C2", case, 0.6, 5.0,
                      "1 block 512x256 O-grid wrap (self-cut), N_H=4 (P=9), 500 it")
    elif key == "C3":
        h = 1.0 / 4096
        case = lattice_case(4, 2, 1024, 512, 3, h=h, dtau=_dtau(h), iterations=200,
                            nbody=4, bodies=tuple((c, "south", c) for c in range(4)),
                            name="C3")
        wl = Workload("C3", case, 0.4, 0.0, "4x2 blocks of 1024x512, N_H=3 (P=7), 200 it")
    elif key == "C4":
        h = 1.0 / 8192
        case = lattice_case(8, 8, 1024, 1024, 4, h=h, dtau=_dtau(h), iterations=50,
                            name="C4")
        wl = Workload("C4", case, 0.5, 2.0, "8x8 blocks of 1024x1024, N_H=4 (P=9), 50 it")
    else:
        raise KeyError(f"unknown BASELINE workload {key!r} (C0..C4)")
    if iterations is not None:
        wl.case.iterations = iterations
    return wl
