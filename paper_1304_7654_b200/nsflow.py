"""North-star physics: the HB Euler / laminar
Navier-Stokes residual-and-smoothing loop on curvilinear structured blocks.

The reference has none of this (hbcore.py:3-13 is a linear advection-
diffusion proxy; SPEC.md:8, 182 list flux physics as a non-goal; PAPER.md:
158-166 promises the HB NS formulation but the text is absent).  This module
and hb_ns.cu implement a standard formulation, specified below; the CPU
checker oracle/ns_oracle.c is an independent restatement of the same
specification.  **Parity is unpinned**: there is no reference output to pin
either side to; GPU == oracle bitwise is what the tests require.

Specification (every operation a separately rounded IEEE fp64 mul / add /
div / sqrt, in the order written; no FMA)
---------------------------------------------------------------------------
State per cell and HB snapshot n: W = (rho, rho u, rho v, rho E), gamma = 1.4,
p = (gamma - 1) (rho E - 0.5 (rho u * u + rho v * v)) with u = rho u / rho,
c = sqrt(gamma p / rho).  Freestream rho = 1, c = 1 (p = 1/gamma), speed M at
the snapshot's angle alpha_n = dalpha sin(2 pi n / P).  Viscosity mu = M / Re
(reference length 1), Pr = 0.72.

Geometry (host, numpy, from node coordinates with two extrapolated ghost
node layers): cell centres = 0.25 ((x00 + x10) + (x11 + x01)); cell area
V = 0.5 ((x11 - x00)(y01 - y10) - (y11 - y00)(x01 - x10)); i-face normal
(area-weighted, pointing +i) S = (y_top - y_bot, x_bot - x_top) of the face
from node (i, j-1) to (i, j); j-face S = (y_left - y_right, x_right - x_left)
of the face from node (i-1, j) to (i, j).  Rigidly moving meshes (C2's
pitching airfoil) carry per-snapshot normals and the face grid flux
G = x_t Sx + y_t Sy.

Face flux (i or j face between cells L and R, with LL, RR the next cells
out along the same index; S, G the face metrics):
  convective   Fc = 0.5 (F(W_L) + F(W_R)),  F(W) = W (u.S - G) + p (0, Sx, Sy, u.S)
  JST          lambda_X = |u_X.S - G| + c_X |S|,  lambda = 0.5 (lambda_L + lambda_R)
               nu_X = |p_{X+1} - 2 p_X + p_{X-1}| / (p_{X+1} + 2 p_X + p_{X-1})
               eps2 = K2 lambda max(nu_L, nu_R),  eps4 = max(0, K4 lambda - eps2)
               D = eps2 (W_R - W_L) - eps4 (((W_RR - 3 W_R) + 3 W_L) - W_LL)
  viscous (NS) face gradients of u, v and e = p / ((gamma-1) rho) on the
               "diamond": d/dxi = phi_R - phi_L, d/deta = 0.25 ((phi_L+ + phi_R+)
               - (phi_L- + phi_R-)) from the cells beside L and R across the
               face's tangential index; x/y derivatives through the Jacobian of
               the cell centres; tau and q = -(mu gamma / Pr) grad e;
               Fv = (0, tau_xx Sx + tau_xy Sy, tau_xy Sx + tau_yy Sy,
                     (u_f tau_xx + v_f tau_xy - q_x) Sx + (u_f tau_xy + v_f tau_yy - q_y) Sy)
  face flux    Ff = (Fc - D) - Fv
Residual  R = ((Ff_{i+1/2} - Ff_{i-1/2}) + Ff_{j+1/2}) - Ff_{j-1/2}
              + V sum_{m ascending} D[n][m] W_m            (HB source)
Local time step (from the iteration's start state, all snapshots):
  dt = min_n CFL V / (((lambda_i + lambda_j) + lambda_v) + omega N_H V),
  lambda_i = 0.5 (lambda(S_{i-1/2}) + lambda(S_{i+1/2})) with the cell's own
  state, lambda_v = (2 gamma mu / (Pr rho)) (|S_i|^2 + |S_j|^2) / V (NS only).
4-stage RK (alphas 1/4, 1/3, 1/2, 1):  W^(s) = W^0 - (alpha_s dt / V) R(W^(s-1)).
Boundaries (two halo layers, filled before every residual): far-field =
freestream of the snapshot; no-slip wall = (rho, -rho u, -rho v, rho E) of the
mirrored interior cell; slip wall = the interior state with its velocity
(relative to the wall) reflected about the face normal; cuts = the paired
interior layers; corner halos = the i-halo cell of the nearest interior row.
Residual norm: sqrt(sum over blocks, snapshots, cells of R_rho^2) of stage 1.
Forces: per snapshot, cl / cd = sum over wall faces (blocks ascending, face
order) of p S rotated into the snapshot's lift / drag axes.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GAMMA = 1.4
PR = 0.72
K2 = 0.5
K4 = 1.0 / 64.0
CFL = 1.5
NG = 2            # halo layers

# face kinds (per block side: south, north, west, east)
FARFIELD, NOSLIP, SLIP, CUT = 0, 1, 2, 3
SIDES = ("south", "north", "west", "east")


@dataclass
class NSBlock:
    id: int
    ni: int
    nj: int
    # node coordinates, shape (P_geo, nj+1+2NG, ni+1+2NG): snapshot-major when
    # the mesh moves (P_geo = P), else P_geo = 1
    x: np.ndarray
    y: np.ndarray
    kinds: tuple = (FARFIELD, FARFIELD, FARFIELD, FARFIELD)
    # grid velocity field (per snapshot) as functions of node position, or None
    xt: np.ndarray | None = None
    yt: np.ndarray | None = None


@dataclass
class NSCut:
    """side_a of block a (face, 1-based range lo..hi) <-> side_b of block b."""
    a: int
    face_a: str
    b: int
    face_b: str
    lo: int
    hi: int


@dataclass
class NSCase:
    name: str
    nharms: int
    mach: float
    dalpha_deg: float
    reynolds: float | None          # None: Euler
    omega: float
    blocks: list
    cuts: list = field(default_factory=list)
    iterations: int = 100
    cfl: float = CFL

    @property
    def planes(self):
        return 2 * self.nharms + 1

    @property
    def mu(self):
        return 0.0 if self.reynolds is None else self.mach / self.reynolds


# ---------------------------------------------------------------------------
# meshes (BASELINE.json configs, physics versions)
# ---------------------------------------------------------------------------

def _extend(X):
    """Two ghost node layers on every side by linear extrapolation."""
    for _ in range(NG):
        X = np.concatenate([2 * X[:, :1] - X[:, 1:2], X, 2 * X[:, -1:] - X[:, -2:-1]], axis=1)
        X = np.concatenate([2 * X[:1] - X[1:2], X, 2 * X[-1:] - X[-2:-1]], axis=0)
    return X


def sinusoidal_mesh(ni, nj, x0=0.0, y0=0.0, lx=1.0, ly=None, amp=0.05):
    """The unit square (or its [x0, x0+lx] x [y0, y0+ly] piece) mapped by
    x += amp sin(2 pi y), y += amp sin(2 pi x) (configs 0 and 4)."""
    ly = lx * nj / ni if ly is None else ly
    X, Y = np.meshgrid(x0 + lx * np.arange(ni + 1) / ni, y0 + ly * np.arange(nj + 1) / nj)
    x = X + amp * np.sin(2 * np.pi * Y)
    y = Y + amp * np.sin(2 * np.pi * X)
    return _extend(x)[None], _extend(y)[None]


def tanh_mesh(ni, nj, x0, y0, lx, ly, beta=2.0, ytot=None, yoff=0.0):
    """Rectangle piece whose y coordinate is clustered toward the bottom wall
    y = 0 by tanh stretching (configs 1 and 3): y = H (1 + tanh(beta (eta -
    1)) / tanh(beta)) over the whole height H, eta uniform."""
    ytot = ly if ytot is None else ytot
    eta = (yoff + ly * np.arange(nj + 1) / nj) / ytot
    yy = ytot * (1.0 + np.tanh(beta * (eta - 1.0)) / np.tanh(beta))
    xx = x0 + lx * np.arange(ni + 1) / ni
    X, Y = np.meshgrid(xx, yy)
    return _extend(X)[None], _extend(Y)[None]


def naca0012(t):
    """Half-thickness of NACA 0012 (closed trailing edge) at chord station t."""
    return 0.6 * (0.2969 * np.sqrt(t) - 0.1260 * t - 0.3516 * t ** 2 + 0.2843 * t ** 3 - 0.1036 * t ** 4)


def ogrid_mesh(ni, nj, radius=20.0, stretch=1.02, planes=1, pitch_deg=0.0, k=0.1, mach=0.6):
    """O-grid around NACA 0012 (config 2): i runs around the airfoil
    (periodic, a self-cut), j outward with geometric radial spacing (ratio
    `stretch`) to a circle of `radius` chords about mid-chord.  With
    pitch_deg > 0 the whole mesh rotates rigidly about the quarter chord,
    alpha(t) = pitch sin(omega t), omega = 2 k M (chord 1); snapshot n sits
    at t_n = 2 pi n / (P omega); node velocities are returned as xt, yt."""
    # clockwise around the airfoil, so that (i, j = outward) is right-handed
    th = -2 * np.pi * np.arange(ni + 1) / ni
    t = 0.5 * (1.0 + np.cos(th))                       # TE -> LE -> TE
    xs = t
    ys = np.where(np.sin(th) >= 0, 1.0, -1.0) * naca0012(t)
    xo = 0.5 + radius * np.cos(th)
    yo = radius * np.sin(th)                           # lower surface first
    g = stretch ** np.arange(nj + 1)
    s = (g - 1.0) / (g[-1] - 1.0)                      # 0 at the wall, 1 outside
    x = xs[None, :] + s[:, None] * (xo - xs)[None, :]
    y = ys[None, :] + s[:, None] * (yo - ys)[None, :]
    x, y = _extend(x), _extend(y)
    if pitch_deg == 0.0:
        return x[None], y[None], None, None
    omega = 2.0 * k * mach
    xs_, ys_, xt_, yt_ = [], [], [], []
    for n in range(planes):
        tn = 2 * np.pi * n / (planes * omega)
        a = math.radians(pitch_deg) * math.sin(omega * tn)
        ad = math.radians(pitch_deg) * omega * math.cos(omega * tn)
        ca, sa = math.cos(-a), math.sin(-a)           # nose-up pitch: clockwise rotation
        dx, dy = x - 0.25, y
        xr = 0.25 + ca * dx - sa * dy
        yr = sa * dx + ca * dy
        xs_.append(xr)
        ys_.append(yr)
        # d/dt of the rotation: omega_z = -ad about (0.25, 0)
        xt_.append(ad * (yr - 0.0))
        yt_.append(-ad * (xr - 0.25))
    return np.stack(xs_), np.stack(ys_), np.stack(xt_), np.stack(yt_)


def ns_workload(key, iterations=None, scale=1):
    """BASELINE.json configs with their physics.  `scale`
    divides the cell counts (tests run small versions of the same setups)."""
    key = key.upper()
    if key == "C0":
        ni, nj = 64 // scale, 32 // scale
        x, y = sinusoidal_mesh(ni, nj, ly=0.5)
        case = NSCase("C0-euler", 1, 0.5, 1.0, None, 1.0, [NSBlock(0, ni, nj, x, y)], iterations=100)
    elif key in ("C1", "C3"):
        nbx, nby = (2, 2) if key == "C1" else (4, 2)
        ni, nj = ((256, 128) if key == "C1" else (1024, 512))
        ni, nj = ni // scale, nj // scale
        mach, re, nh = (0.3, 1e4, 2) if key == "C1" else (0.4, 1e5, 3)
        lx, ly = 1.0, 0.5
        blocks = []
        for r in range(nby):
            for c in range(nbx):
                x, y = tanh_mesh(ni, nj, c * lx, 0.0, lx, ly, ytot=nby * ly, yoff=r * ly)
                kinds = [FARFIELD] * 4
                if r == 0:
                    kinds[0] = NOSLIP
                if r > 0:
                    kinds[0] = CUT
                if r < nby - 1:
                    kinds[1] = CUT
                if c > 0:
                    kinds[2] = CUT
                if c < nbx - 1:
                    kinds[3] = CUT
                blocks.append(NSBlock(r * nbx + c, ni, nj, x, y, tuple(kinds)))
        cuts = [NSCut(r * nbx + c, "east", r * nbx + c + 1, "west", 1, nj)
                for r in range(nby) for c in range(nbx - 1)]
        cuts += [NSCut(r * nbx + c, "north", (r + 1) * nbx + c, "south", 1, ni)
                 for r in range(nby - 1) for c in range(nbx)]
        case = NSCase(f"{key}-ns", nh, mach, 0.0, re, 1.0, blocks, cuts,
                      iterations=200 if key == "C1" else 200)
    elif key == "C2":
        ni, nj = 512 // scale, 256 // scale
        P = 9
        x, y, xt, yt = ogrid_mesh(ni, nj, planes=P, pitch_deg=5.0, mach=0.6)
        blk = NSBlock(0, ni, nj, x, y, (SLIP, FARFIELD, CUT, CUT), xt, yt)
        case = NSCase("C2-euler-pitching", 4, 0.6, 0.0, None, 2 * 0.1 * 0.6, [blk],
                      [NSCut(0, "east", 0, "west", 1, nj)], iterations=500)
    elif key == "C4":
        ni = nj = 1024 // scale
        blocks = []
        for r in range(8):
            for c in range(8):
                x, y = sinusoidal_mesh(ni, nj, x0=c / 8, y0=r / 8, lx=1 / 8, ly=1 / 8)
                kinds = [FARFIELD if r == 0 else CUT, FARFIELD if r == 7 else CUT,
                         FARFIELD if c == 0 else CUT, FARFIELD if c == 7 else CUT]
                blocks.append(NSBlock(r * 8 + c, ni, nj, x, y, tuple(kinds)))
        cuts = [NSCut(r * 8 + c, "east", r * 8 + c + 1, "west", 1, nj) for r in range(8) for c in range(7)]
        cuts += [NSCut(r * 8 + c, "north", (r + 1) * 8 + c, "south", 1, ni) for r in range(7) for c in range(8)]
        case = NSCase("C4-euler", 4, 0.5, 2.0, None, 1.0, blocks, cuts, iterations=50)
    else:
        raise KeyError(key)
    if iterations is not None:
        case.iterations = iterations
    return case


# ---------------------------------------------------------------------------
# geometry (the specification's formulas, numpy element-wise: each op one
# IEEE rounding, the written order)
# ---------------------------------------------------------------------------

def metrics(block):
    """Cell centres (incl. ghosts), areas, face normals: arrays over the
    extended index range.  Shapes (Pg = 1 or P):
      xc, yc   (Pg, nj+2NG, ni+2NG)      cell (j, i) at [j+NG-1, i+NG-1]
      vol      (Pg, nj+2NG, ni+2NG)
      six, siy (Pg, nj+2NG, ni+2NG+1)    i-face between cells i and i+1
      sjx, sjy (Pg, nj+2NG+1, ni+2NG)    j-face between cells j and j+1
    """
    x, y = block.x, block.y
    x00, x10, x11, x01 = x[:, :-1, :-1], x[:, :-1, 1:], x[:, 1:, 1:], x[:, 1:, :-1]
    y00, y10, y11, y01 = y[:, :-1, :-1], y[:, :-1, 1:], y[:, 1:, 1:], y[:, 1:, :-1]
    xc = 0.25 * ((x00 + x10) + (x11 + x01))
    yc = 0.25 * ((y00 + y10) + (y11 + y01))
    vol = 0.5 * ((x11 - x00) * (y01 - y10) - (y11 - y00) * (x01 - x10))
    # i-face at node column I: from node (I, J-1) to (I, J)
    six = y[:, 1:, :] - y[:, :-1, :]
    siy = x[:, :-1, :] - x[:, 1:, :]
    # j-face at node row J: from node (I-1, J) to (I, J)
    sjx = y[:, :, :-1] - y[:, :, 1:]
    sjy = x[:, :, 1:] - x[:, :, :-1]
    out = {"xc": xc, "yc": yc, "vol": vol, "six": six, "siy": siy, "sjx": sjx, "sjy": sjy}
    if block.xt is not None:
        # face grid flux: average of the face's two node velocities . S
        xt, yt = block.xt, block.yt
        gi = (0.5 * (xt[:, 1:, :] + xt[:, :-1, :])) * six + (0.5 * (yt[:, 1:, :] + yt[:, :-1, :])) * siy
        gj = (0.5 * (xt[:, :, :-1] + xt[:, :, 1:])) * sjx + (0.5 * (yt[:, :, :-1] + yt[:, :, 1:])) * sjy
        out["gi"], out["gj"] = gi, gj
    return {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in out.items()}


def freestream(case):
    """W_inf per snapshot, shape (P, 4)."""
    P = case.planes
    out = np.zeros((P, 4))
    for n in range(P):
        a = math.radians(case.dalpha_deg) * math.sin(2 * math.pi * n / P)
        u, v = case.mach * math.cos(a), case.mach * math.sin(a)
        p = 1.0 / GAMMA
        out[n] = (1.0, u, v, p / (GAMMA - 1.0) + 0.5 * (u * u + v * v))
    return out


def initial_state(case, block, seed=13047654):
    """Freestream with a seeded 1% uniform perturbation per state variable
    (BASELINE.json), halos zero: shape (P, 4, nj+2NG, ni+2NG)."""
    P = case.planes
    winf = freestream(case)
    rng = np.random.default_rng(seed + block.id)
    q = np.zeros((P, 4, block.nj + 2 * NG, block.ni + 2 * NG))
    pert = 1.0 + 0.01 * rng.uniform(-1.0, 1.0, size=(P, 4, block.nj, block.ni))
    q[:, :, NG:-NG, NG:-NG] = winf[:, :, None, None] * pert
    return q


def circulant_antisymmetric(mat):
    from .hbop import circulant_antisymmetric as ca
    return ca(mat)


def spectral_matrix(case):
    from .hbop import spectral_matrix as sm
    return np.ascontiguousarray(sm(case.nharms, case.omega).matrix)


# ---------------------------------------------------------------------------
# the GPU run (libhbgpu hbns_* + hbgpu_halo for the cut halos)
# ---------------------------------------------------------------------------

RK_ALPHAS = (0.25, 1.0 / 3.0, 0.5, 1.0)
TILE_I, TILE_J = 32, 8        # hbns_stage tiles (include/hbns.h HBNS_TILE_I/J)


def ns_partition(case, nranks):
    """Blocks -> ranks, the proxy path's greedy LPT rule (topology.
    partition_blocks): blocks in descending cell count (ties: lower id) each
    to the least-loaded rank (ties: lower rank).  Returns owner[block id]."""
    import heapq
    if not 1 <= nranks <= len(case.blocks):
        raise ValueError(f"{nranks} ranks for {len(case.blocks)} blocks")
    loads = [(0, r) for r in range(nranks)]
    owner = {}
    for b in sorted(case.blocks, key=lambda b: (-b.ni * b.nj, b.id)):
        load, r = heapq.heappop(loads)
        owner[b.id] = r
        heapq.heappush(loads, (load + b.ni * b.nj, r))
    return owner


class HaloPlan:
    """The cut-halo moves of one rank (hbgpu_halo directions, both halo
    layers, both ways per cut), in one global order -- cuts as listed, layer
    1 then 2, a <- b then b <- a -- which every rank enumerates alike:
      local   both blocks on this rank: slot -> slot;
      pack    source here, destination on peer q: slot -> send buffer;
      unpack  source on peer q, destination here: receive buffer -> slot.
    A peer's payload is its directions in that order, each element-major
    (the 4P values of a face cell contiguous).  sends / recvs: (peer,
    offset, count) in doubles, peers ascending."""

    def __init__(self, case, offsets, owner=None, rank=0):
        from . import native
        P = case.planes
        nv = 4 * P
        blocks = {b.id: b for b in case.blocks}
        owner = owner or {b.id: 0 for b in case.blocks}

        def cell(b, face, k, e, halo):
            ni, nj = b.ni, b.nj
            if face == "south":
                return (e, 1 - k) if halo else (e, k)
            if face == "north":
                return (e, nj + k) if halo else (e, nj + 1 - k)
            if face == "west":
                return (1 - k, e) if halo else (k, e)
            return (ni + k, e) if halo else (ni + 1 - k, e)

        def off(b, i, j):
            return offsets[b.id] + (j + 1) * (b.ni + 4) + (i + 1)

        local, pack, unpack = [], {}, {}
        for c in case.cuts:
            A, B = blocks[c.a], blocks[c.b]
            n = c.hi - c.lo + 1
            for k in (1, 2):
                for dst, dface, src, sface in ((A, c.face_a, B, c.face_b), (B, c.face_b, A, c.face_a)):
                    ps, pd = owner[src.id], owner[dst.id]
                    if rank not in (ps, pd):
                        continue
                    si, sj = cell(src, sface, k, c.lo, False)
                    di, dj = cell(dst, dface, k, c.lo, True)
                    ses = 1 if sface in ("south", "north") else src.ni + 4
                    des = 1 if dface in ("south", "north") else dst.ni + 4
                    svs = (src.nj + 4) * (src.ni + 4)
                    dvs = (dst.nj + 4) * (dst.ni + 4)
                    if ps == rank and pd == rank:
                        local.append((off(src, si, sj), ses, svs, off(dst, di, dj), des, dvs, n, 0, 0, 0))
                    elif ps == rank:
                        pack.setdefault(pd, []).append((off(src, si, sj), ses, svs, n))
                    else:
                        unpack.setdefault(ps, []).append((off(dst, di, dj), des, dvs, n))
        rows_pack, rows_unpack, self.sends, self.recvs = [], [], [], []
        o = 0
        for q in sorted(pack):
            start = o
            for so, ses, svs, n in pack[q]:
                rows_pack.append((so, ses, svs, o, nv, 1, n, 0, 1, 0))   # dst_kind 1: send buffer
                o += n * nv
            self.sends.append((q, start, o - start))
        self.nsend = o
        o = 0
        for q in sorted(unpack):
            start = o
            for do, des, dvs, n in unpack[q]:
                rows_unpack.append((o, nv, 1, do, des, dvs, n, 2, 0, 0))  # src_kind 2: receive buffer
                o += n * nv
            self.recvs.append((q, start, o - start))
        self.nrecv = o
        dt = native.HALO_DIR_DTYPE
        # the first exchange launch: local copies and packs (one hbgpu_halo)
        self.first = np.array(local + rows_pack, dtype=dt) if local or rows_pack else np.zeros(0, dt)
        self.unpack = np.array(rows_unpack, dtype=dt) if rows_unpack else np.zeros(0, dt)
        self.nlocal = len(local)


def _halo_rows(case, offsets):
    """hbgpu_halo directions of every cut, both ways, both halo layers (one
    rank holding every block)."""
    return HaloPlan(case, offsets).first


def wall_layout(case):
    """Global wall-face order of the force folds (blocks ascending, sides
    south / north / west / east, face cells ascending): per block the
    position of its first wall face, and the total."""
    off, n = {}, 0
    for b in sorted(case.blocks, key=lambda b: b.id):
        off[b.id] = n
        for side in range(4):
            if b.kinds[side] in (NOSLIP, SLIP):
                n += b.ni if side < 2 else b.nj
    return off, n


def _ns_types():
    """ctypes mirrors of hbns_block / hbns_args (include/hbns.h)."""
    import ctypes
    vp, i32, i64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double

    class Block(ctypes.Structure):
        _fields_ = [("w_off", i64), ("r_off", i64), ("dt_off", i64), ("c_off", i64), ("fi_off", i64),
                    ("fj_off", i64), ("part_off", i64), ("ni", i32), ("nj", i32), ("kinds", i32 * 4),
                    ("gid", i32), ("wall_off", i32)]

    class Args(ctypes.Structure):
        _fields_ = [("w", vp * 3), ("r", vp), ("dt", vp), ("xc", vp), ("yc", vp), ("vol", vp),
                    ("six", vp), ("siy", vp), ("gi", vp), ("sjx", vp), ("sjy", vp), ("gj", vp),
                    ("blocks", vp), ("winf", vp), ("dmat", vp), ("status", vp), ("norm_part", vp),
                    ("norms", vp), ("forces", vp), ("blk_norms", vp), ("wall_prod", vp), ("iter_dev", vp), ("mu", f64), ("cfl", f64), ("omega_nh", f64), ("kq", f64),
                    ("nblocks", i32), ("P", i32), ("Pg", i32), ("moving", i32), ("max_len", i32),
                    ("max_cells", i32), ("max_ni", i32), ("max_nj", i32), ("nglobal", i32), ("nwall", i32),
                    ("stage", i32), ("flags", i32)]
    return Block, Args


class NSRun:
    """The HB Euler / NS loop of one rank's blocks on one GPU: the blocks
    resident in three state pools, the RK stages launched on torch's current
    stream (hb_ns.cu), cut halos by hbgpu_halo.

    owner (block id -> rank, ns_partition) and rank select this rank's
    blocks; with several ranks, each stage's cut halos are an exchange --
    exchange_begin (local copies + packs), the transport moving `sends` /
    `recvs` between the ranks' send and receive buffers, exchange_end
    (unpacks) -- and the residual norms and wall forces are kept as per-block
    sums and per-face products in global order (blk_norms, wall_prod), to be
    summed over the ranks and folded like one rank's (run_ns_ranks)."""

    def __init__(self, case, max_iters, initial=None, device=None, owner=None, rank=0):
        import ctypes
        import torch
        from . import native
        self.lib = native.require_cuda()
        self.torch, self._ct = torch, ctypes
        self.case = case
        self.max_iters = max_iters
        self.rank = rank
        owner = owner or {b.id: 0 for b in case.blocks}
        self.multi = len(set(owner.values())) > 1
        dev = self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        P = case.planes
        all_blocks = sorted(case.blocks, key=lambda b: b.id)
        gid = {b.id: k for k, b in enumerate(all_blocks)}
        wall_off, nwall = wall_layout(case)
        blocks = self.blocks = [b for b in all_blocks if owner[b.id] == rank]
        if not blocks:
            raise ValueError(f"rank {rank} owns no block")
        geos = [metrics(b) for b in blocks]
        Pg = geos[0]["xc"].shape[0]
        moving = "gi" in geos[0]
        Block, Args = _ns_types()
        max_cells = max(b.ni * b.nj for b in blocks)
        ctas = max(-(-b.ni // TILE_I) * -(-b.nj // TILE_J) for b in blocks)   # tiles per block
        table = (Block * len(blocks))()
        self.w_off = {}
        wsz = r_off = dt_off = c_off = fi_off = fj_off = 0
        pools = {k: [] for k in ("xc", "yc", "vol", "six", "siy", "gi", "sjx", "sjy", "gj")}
        for k, (b, g) in enumerate(zip(blocks, geos)):
            e = table[k]
            e.w_off, e.r_off, e.dt_off = wsz, r_off, dt_off
            e.c_off, e.fi_off, e.fj_off = c_off, fi_off, fj_off
            e.part_off = k * ctas
            e.ni, e.nj = b.ni, b.nj
            # the stage kernel indexes inside one snapshot of a block in 32 bits
            if 4 * (b.nj + 4) * (b.ni + 4) >= 2 ** 31:
                from .exceptions import ConfigError
                raise ConfigError(f"block {b.id}: {b.ni} x {b.nj} cells exceed the NS kernel's 32-bit plane offsets")
            for sd in range(4):
                e.kinds[sd] = b.kinds[sd]
            e.gid, e.wall_off = gid[b.id], wall_off[b.id]
            self.w_off[b.id] = wsz
            wsz += P * 4 * (b.nj + 4) * (b.ni + 4)
            r_off += P * 4 * b.nj * b.ni
            dt_off += b.nj * b.ni
            c_off += g["xc"].size
            fi_off += g["six"].size
            fj_off += g["sjx"].size
            for name in pools:
                if name in g:
                    pools[name].append(g[name].ravel())
        f64 = torch.float64
        self.slots = [torch.zeros(wsz, dtype=f64, device=dev) for _ in range(3)]
        for b in blocks:
            q = initial(b) if initial is not None else initial_state(case, b)
            self.slot_view(0, b).copy_(torch.from_numpy(np.ascontiguousarray(q)))
        self.r = torch.zeros(max(1, r_off), dtype=f64, device=dev)
        self.dt = torch.zeros(max(1, dt_off), dtype=f64, device=dev)
        self.geo = {k: (torch.from_numpy(np.concatenate(v)).to(dev) if v else torch.zeros(1, dtype=f64, device=dev))
                    for k, v in pools.items()}
        self.t_blocks = torch.frombuffer(bytearray(bytes(table)), dtype=torch.uint8).to(dev)
        self.winf = torch.from_numpy(np.ascontiguousarray(freestream(case))).to(dev)
        dmat_host = spectral_matrix(case).copy()
        self.dmat = torch.from_numpy(dmat_host).to(dev)
        # HBNS_FLAG_D_CIRCULANT: the update may share D products between rows m +- k
        self.d_circulant = bool(circulant_antisymmetric(dmat_host))
        self.status = torch.full((len(blocks),), -1, dtype=torch.int64, device=dev)
        self.norm_part = torch.zeros(len(blocks) * ctas, dtype=f64, device=dev)
        self.norms = torch.zeros(max(1, max_iters), dtype=f64, device=dev)
        self.forces = torch.zeros(max(1, max_iters) * P * 2, dtype=f64, device=dev)
        self.nglobal, self.nwall = len(all_blocks), nwall
        if self.multi:
            self.blk_norms = torch.zeros(max(1, max_iters) * len(all_blocks), dtype=f64, device=dev)
            self.wall_prod = torch.zeros(max(1, max_iters * P * 2 * nwall), dtype=f64, device=dev)
        plan = self.plan = HaloPlan(case, self.w_off, owner, rank)
        self.t_first = torch.from_numpy(plan.first.view(np.uint8).copy()).to(dev) if len(plan.first) else None
        self.t_unpack = torch.from_numpy(plan.unpack.view(np.uint8).copy()).to(dev) if len(plan.unpack) else None
        self.first_len = int(plan.first["length"].max()) if len(plan.first) else 0
        self.unpack_len = int(plan.unpack["length"].max()) if len(plan.unpack) else 0
        self.iter_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        self.graph = None
        self.sendbuf = torch.zeros(max(1, plan.nsend), dtype=f64, device=dev)
        self.recvbuf = torch.zeros(max(1, plan.nrecv), dtype=f64, device=dev)
        a = Args()
        for k in range(3):
            a.w[k] = self.slots[k].data_ptr()
        a.r, a.dt = self.r.data_ptr(), self.dt.data_ptr()
        for name in pools:
            setattr(a, name, self.geo[name].data_ptr())
        a.blocks, a.winf, a.dmat = self.t_blocks.data_ptr(), self.winf.data_ptr(), self.dmat.data_ptr()
        a.status, a.norm_part = self.status.data_ptr(), self.norm_part.data_ptr()
        a.norms, a.forces = self.norms.data_ptr(), self.forces.data_ptr()
        if self.multi:
            a.blk_norms, a.wall_prod = self.blk_norms.data_ptr(), self.wall_prod.data_ptr()
        else:
            a.iter_dev = self.iter_dev.data_ptr()
        a.mu, a.cfl, a.omega_nh = case.mu, case.cfl, case.omega * case.nharms
        a.kq = (case.mu * GAMMA) / PR    # the specification's (mu gamma) / Pr, one IEEE mul and div
        a.nblocks, a.P, a.Pg, a.moving = len(blocks), P, Pg, int(moving)
        a.flags = 1 if self.d_circulant else 0   # HBNS_FLAG_D_CIRCULANT
        a.max_len = max(max(b.ni, b.nj) for b in blocks)
        a.max_cells = max_cells
        a.max_ni, a.max_nj = max(b.ni for b in blocks), max(b.nj for b in blocks)
        a.nglobal, a.nwall = len(all_blocks), nwall
        self.args = a
        self.done = 0

    def slot_view(self, slot, b):
        P = self.case.planes
        n = P * 4 * (b.nj + 4) * (b.ni + 4)
        off = self.w_off[b.id]
        return self.slots[slot][off:off + n].view(P, 4, b.nj + 4, b.ni + 4)

    def _stream(self):
        return self._ct.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def _vp(self, t):
        return self._ct.c_void_p(t.data_ptr())

    def exchange_begin(self, slot):
        """Cut halos of `slot`: local copies, and the packs of the payloads
        this rank sends."""
        from . import native
        if self.t_first is not None:
            native.check(self.lib.hbgpu_halo(self._vp(self.slots[slot]), self._vp(self.sendbuf), None,
                                             self._vp(self.t_first), len(self.plan.first), self.first_len,
                                             self.case.planes, self._stream()), "hbgpu_halo (ns cuts)")

    def exchange_end(self, slot):
        """Unpack the received payloads into `slot`'s halos."""
        from . import native
        if self.t_unpack is not None:
            native.check(self.lib.hbgpu_halo(self._vp(self.slots[slot]), None, self._vp(self.recvbuf),
                                             self._vp(self.t_unpack), len(self.plan.unpack), self.unpack_len,
                                             self.case.planes, self._stream()), "hbgpu_halo (ns unpack)")

    def stage(self, st):
        """Boundary halos of stage st's input, then the fused stage kernel."""
        from . import native
        si, so = STAGE_SLOTS[st]
        self.args.stage = st   # the launch copies the arguments (and a graph keeps the copy)
        ap, s = self._ct.byref(self.args), self._stream()
        native.check(self.lib.hbns_boundaries(ap, si, s), "hbns_boundaries")
        native.check(self.lib.hbns_stage(ap, si, so, RK_ALPHAS[st], self.done, int(st == 0), s), "hbns_stage")

    def finish_iteration(self):
        from . import native
        native.check(self.lib.hbns_forces(self._ct.byref(self.args), self.done, self._stream()), "hbns_forces")
        self.done += 1

    def _one_iteration(self):
        for st in range(4):
            self.exchange_begin(STAGE_SLOTS[st][0])
            self.stage(st)
        self.finish_iteration()

    def iterate(self, iterations, use_graph=True):
        """`iterations` iterations of a run whose blocks are all on this rank.
        use_graph: the first iteration runs eagerly and is then captured once
        as a CUDA graph (its ~20 launches; the iteration index lives in a
        device counter), which every later iteration replays."""
        if self.multi:
            raise ValueError("a multi-rank NSRun iterates through run_ns_ranks / run_ns_distributed")
        if self.done + iterations > self.max_iters:
            raise ValueError(f"{iterations} more iterations exceed max_iters={self.max_iters}")
        torch = self.torch
        for _ in range(iterations):
            if not use_graph or (self.graph is None and self.done == 0):
                self._one_iteration()
                continue
            if self.graph is None:
                side = torch.cuda.Stream(self.device)
                side.wait_stream(torch.cuda.current_stream(self.device))
                self.graph = torch.cuda.CUDAGraph()
                with torch.cuda.stream(side), torch.cuda.graph(self.graph, stream=side):
                    done = self.done
                    self._one_iteration()
                    self.done = done   # capture launches nothing
                torch.cuda.current_stream(self.device).wait_stream(side)
            self.graph.replay()
            self.done += 1
        return self

    def divergence(self):
        """The first non-finite value: earliest (iteration, stage), then the
        lowest block id, then the first (snapshot, variable, j, i) --
        (block, i, j, variable, snapshot, iteration, stage), or None."""
        return _first_divergence(self.status.cpu().numpy().view(np.uint64), self.blocks)

    def fields(self):
        return {b.id: self.slot_view(0, b).cpu().numpy() for b in self.blocks}

    def norm_history(self):
        return self.norms[:self.done].cpu().tolist()

    def force_history(self):
        """(iterations, P, 2) (cl, cd) in the snapshot's freestream axes."""
        return _lift_drag(self.case, self.forces[:self.done * self.case.planes * 2].cpu().numpy(), self.done)


def _first_divergence(keys, blocks):
    """Decode per-block status keys ((gstage << 40) | lin, all-ones: none)."""
    hits = []
    for b, key in zip(blocks, keys):
        key = int(key)
        if key == (1 << 64) - 1:
            continue
        gstage, lin = key >> 40, key & ((1 << 40) - 1)
        hits.append((gstage, b.id, lin, b))
    if not hits:
        return None
    gstage, bid, lin, b = min(hits, key=lambda h: h[:3])
    nk = lin // (b.ni * b.nj)
    return bid, lin % b.ni + 1, (lin // b.ni) % b.nj + 1, nk % 4, nk // 4, (gstage - 1) // 4, (gstage - 1) % 4


def _raise_divergence(d):
    from .exceptions import DivergenceError
    err = DivergenceError(*d[:5])
    err.iteration, err.stage = d[5], d[6]
    raise err


# stage s reads slot STAGE_SLOTS[s][0], writes STAGE_SLOTS[s][1] (0 = W^0)
STAGE_SLOTS = ((0, 1), (1, 2), (2, 1), (1, 0))


def _lift_drag(case, fxy, iterations):
    P = case.planes
    fxy = np.asarray(fxy).reshape(iterations, P, 2)
    ang = np.radians(case.dalpha_deg) * np.sin(2 * np.pi * np.arange(P) / P)
    ca, sa = np.cos(ang), np.sin(ang)
    cd = fxy[:, :, 0] * ca + fxy[:, :, 1] * sa
    cl = fxy[:, :, 1] * ca - fxy[:, :, 0] * sa
    return np.stack([cl, cd], axis=2)


class NSRanksResult:
    """A multi-rank run's results, the job-wide view: fields of every block,
    the residual norms and wall forces folded exactly as one rank's, the
    first divergence in block order."""

    def __init__(self, case, runs, norms, forces, iterations):
        self.case, self.runs, self._norms, self._forces, self.done = case, runs, norms, forces, iterations

    def fields(self):
        out = {}
        for r in self.runs:
            out.update(r.fields())
        return out

    def norm_history(self):
        return self._norms.cpu().tolist()

    def force_history(self):
        return _lift_drag(self.case, self._forces.cpu().numpy(), self.done)

    def divergence(self):
        keys = np.concatenate([r.status.cpu().numpy().view(np.uint64) for r in self.runs])
        return _first_divergence(keys, [b for r in self.runs for b in r.blocks])


def _fold_job(case, lib, blk_norms, wall_prod, iterations, stream, ctypes_mod):
    """Job-wide norms (hbgpu_norm_totals over global block ids) and wall
    forces (hbns_wall_fold over the global wall-face order) from the summed
    per-block sums and per-face products."""
    import torch
    from . import native
    P = case.planes
    nb = len(case.blocks)
    norms = torch.zeros(max(1, iterations), dtype=torch.float64, device=blk_norms.device)
    forces = torch.zeros(max(1, iterations * P * 2), dtype=torch.float64, device=blk_norms.device)
    vp = ctypes_mod.c_void_p
    if iterations:
        native.check(lib.hbgpu_norm_totals(vp(blk_norms.data_ptr()), iterations, nb, vp(norms.data_ptr()), stream),
                     "hbgpu_norm_totals")
        native.check(lib.hbns_wall_fold(vp(wall_prod.data_ptr()), iterations, P, wall_layout(case)[1],
                                        vp(forces.data_ptr()), stream), "hbns_wall_fold")
    return norms[:iterations], forces[:iterations * P * 2]


def run_ns_ranks(case, iterations=None, nranks=2, initial=None):
    """The case split over `nranks` ranks (ns_partition) run as engines of one
    process on one GPU, their cut-halo payloads moved by device copies
    (loopback transport) -- the exchange a multi-GPU run does over NCCL
    (run_ns_distributed), step for step.  Returns an NSRanksResult."""
    import ctypes
    import torch
    iterations = case.iterations if iterations is None else iterations
    owner = ns_partition(case, nranks)
    runs = [NSRun(case, max(1, iterations), initial, owner=owner, rank=r) for r in range(nranks)]
    if nranks == 1:
        runs[0].iterate(iterations)
        torch.cuda.synchronize()
        res = NSRanksResult(case, runs, runs[0].norms[:iterations], runs[0].forces[:iterations * case.planes * 2],
                            iterations)
    else:
        send_at = [{q: (o, c) for q, o, c in r.plan.sends} for r in runs]
        for _ in range(iterations):
            for st in range(4):
                si = STAGE_SLOTS[st][0]
                for r in runs:
                    r.exchange_begin(si)
                for r in runs:   # the transport: peer send-buffer segments -> receive buffer
                    for q, off, cnt in r.plan.recvs:
                        so, sc = send_at[q][r.rank]
                        if sc != cnt:
                            raise RuntimeError(f"rank {q} -> {r.rank}: {sc} != {cnt} doubles")
                        r.recvbuf[off:off + cnt].copy_(runs[q].sendbuf[so:so + sc])
                for r in runs:
                    r.exchange_end(si)
                    r.stage(st)
            for r in runs:
                r.finish_iteration()
        blk = sum(r.blk_norms for r in runs)       # one nonzero contributor per entry: exact
        prod = sum(r.wall_prod for r in runs)
        norms, forces = _fold_job(case, runs[0].lib, blk, prod, iterations, runs[0]._stream(), ctypes)
        torch.cuda.synchronize()
        res = NSRanksResult(case, runs, norms, forces, iterations)
    d = res.divergence()
    if d is not None:
        _raise_divergence(d)
    return res


def run_ns_distributed(case, iterations=None, initial=None):
    """One rank of a multi-GPU run under torchrun (one process per GPU,
    torch.distributed initialised): this rank's blocks (ns_partition), the
    cut-halo payloads of every stage over NCCL (grouped ncclSend/ncclRecv per
    peer, hbgpu_comm_exchange), then the per-block norm sums and per-face
    force products summed over the ranks (ncclAllReduce; exact, one
    contributor per entry) and folded as one rank's.  Every rank returns the
    job-wide norms and forces and its own blocks' fields."""
    import ctypes
    import torch
    import torch.distributed as dist
    from . import native
    from .blockops import HaloContext
    from .solver import make_comm
    iterations = case.iterations if iterations is None else iterations
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.cuda.current_device()
    if world == 1:
        return run_ns_ranks(case, iterations, 1, initial)
    owner = ns_partition(case, world)
    run = NSRun(case, max(1, iterations), initial, owner=owner, rank=rank)
    comm = make_comm(rank, world, dev)
    try:
        ctx = HaloContext(rank, comm=comm)
        for _ in range(iterations):
            for st in range(4):
                si = STAGE_SLOTS[st][0]
                run.exchange_begin(si)
                ctx.transfer(run.sendbuf, run.plan.sends, run.recvbuf, run.plan.recvs)
                run.exchange_end(si)
                run.stage(st)
            run.finish_iteration()
        s = run._stream()
        for t in (run.blk_norms, run.wall_prod):
            native.check(run.lib.hbgpu_comm_allreduce(comm, ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(t.data_ptr()),
                                                      t.numel(), native.REDUCE_SUM_F64, s), "hbgpu_comm_allreduce")
        keys = torch.full((len(case.blocks),), -1, dtype=torch.int64, device=run.device)
        keys[torch.tensor(_gids(case, run.blocks), device=run.device)] = run.status
        native.check(run.lib.hbgpu_comm_allreduce(comm, ctypes.c_void_p(keys.data_ptr()),
                                                  ctypes.c_void_p(keys.data_ptr()), keys.numel(),
                                                  native.REDUCE_MIN_U64, s), "hbgpu_comm_allreduce")
        norms, forces = _fold_job(case, run.lib, run.blk_norms, run.wall_prod, iterations, s, ctypes)
        torch.cuda.synchronize()
    finally:
        native.load().hbgpu_comm_destroy(comm)
    res = NSRanksResult(case, [run], norms, forces, iterations)
    d = _first_divergence(keys.cpu().numpy().view(np.uint64), sorted(case.blocks, key=lambda b: b.id))
    if d is not None:
        _raise_divergence(d)
    return res


def _gids(case, blocks):
    order = {b.id: k for k, b in enumerate(sorted(case.blocks, key=lambda b: b.id))}
    return [order[b.id] for b in blocks]


def run_ns(case, iterations=None, initial=None, poll=16):
    """Run a case on the GPU; returns the NSRun (fields, norms, forces).
    The status keys are read every `poll` iterations: a non-finite state
    stops the run there and raises DivergenceError (block, i, j, variable,
    snapshot; .iteration and .stage) for the first offending stage."""
    iterations = case.iterations if iterations is None else iterations
    r = NSRun(case, max(1, iterations), initial)
    done = 0
    while done < iterations:
        step = min(poll, iterations - done)
        r.iterate(step)
        done += step
        d = r.divergence()   # synchronises
        if d is not None:
            _raise_divergence(d)
    r.torch.cuda.synchronize()
    return r
