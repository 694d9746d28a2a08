"""The HB model operator's host-side pieces: constants, the time-spectral
matrix D, the RK scheme, and the initial-state / forcing tables.

Everything transcendental is evaluated here, on the host, with the same numpy
/ math expressions as the reference (hbcore.py:74-177), and the bits are
uploaded: the GPU never recomputes sin/cos, so its inputs are the reference's
inputs bit for bit on the same host.

The forcing array of the reference, amp[n] * pfac[p] * sxy[j, i] evaluated
left to right (hbcore.py:165-177), is stored factored as a per-(plane, pde)
scalar ap[n][p] = amp[n] * pfac[p] and, per block, the two vectors
sin(2 pi x_i) and sin(2 pi y_j) whose rounded product is the reference's
sxy[j, i]; the device forms the sxy table from them once (one rounded multiply
per element) and the stage kernel forms ap * sxy with one more, which
reproduces the reference's array exactly, signed zeros included.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .exceptions import DomainError

NPDE = 4
NU = 0.05
ADVECTION = 1.0
RK_ALPHAS = (0.25, 1.0 / 3.0, 0.5, 1.0)
TWO_PI = 2.0 * math.pi


@dataclass(frozen=True)
class SpectralDeriv:
    """The dense (2 N_H + 1)^2 time-spectral derivative matrix."""

    matrix: np.ndarray
    omega: float
    nharms: int

    @property
    def planes(self):
        return 2 * self.nharms + 1

    @property
    def period(self):
        return TWO_PI / self.omega


def spectral_matrix(nharms, omega):
    """D[j, k] = (omega / 2) (-1)^d / sin(pi d / N) for j != k, 0 on the diagonal.

    d = j - k wrapped into [-N_H, N_H] (N = 2 N_H + 1), which makes D exactly
    antisymmetric in floating point (reference hbcore.py:74-96).
    """
    if nharms < 0:
        raise DomainError(f"nharms must be >= 0, got {nharms}")
    if omega <= 0:
        raise DomainError(f"omega must be > 0, got {omega}")
    size = 2 * nharms + 1
    mat = np.zeros((size, size), dtype=np.float64)
    for row in range(size):
        for col in range(size):
            if row != col:
                d = (row - col + nharms) % size - nharms
                mat[row, col] = 0.5 * omega * (-1.0) ** d / math.sin(math.pi * d / size)
    mat.setflags(write=False)
    return SpectralDeriv(matrix=mat, omega=omega, nharms=nharms)


def circulant_antisymmetric(mat):
    """True when D[(m+k)%P][m] is bitwise D[k][0] and -D[(m-k)%P][m], and the
    diagonal is +0.0.

    spectral_matrix has this structure exactly (the wrapped d of ref
    hbcore.py:88-94 makes D a function of d alone, with D(-d) = -D(d)); the
    stage kernel relies on it to multiply by N_H constants and to share one
    product between two rows.
    """
    mat = np.ascontiguousarray(mat, dtype=np.float64)
    size = mat.shape[0]
    bits = mat.view(np.uint64)
    idx = np.arange(size)
    if np.any(bits[idx, idx] != 0):
        return False
    for k in range(1, size // 2 + 1):
        plus = bits[(idx + k) % size, idx]
        minus = bits[(idx - k) % size, idx]
        if np.any(plus != bits[k, 0]) or np.any(plus != (minus ^ np.uint64(1 << 63))):
            return False
    return True


@dataclass(frozen=True)
class RKScheme:
    """q_s = q_0 - alpha_s dtau R(q_{s-1}), alphas (1/4, 1/3, 1/2, 1)."""

    dtau: float
    alphas: tuple = RK_ALPHAS

    def __post_init__(self):
        if self.alphas[-1] != 1.0:
            raise DomainError("last stage coefficient must be 1")
        if self.dtau < 0:
            raise DomainError("dtau must be >= 0")

    def stage_coefficients(self):
        """alpha_s * dtau, rounded on the host in double (driver.py:118)."""
        return [a * self.dtau for a in self.alphas]


def cell_centres(spec):
    xc = spec.x0 + (np.arange(1, spec.ni + 1) - 0.5) * spec.h
    yc = spec.y0 + (np.arange(1, spec.nj + 1) - 0.5) * spec.h
    return xc, yc


def initial_values(spec, planes, npde, n_lo, n_hi, j_lo, j_hi):
    """The reference's deterministic initial state on a plane/row sub-range:
    0.1 sin(2 pi x + 0.35 p) cos(2 pi y - 0.2 n) (hbcore.py:148-162).

    run_case looks this function up at call time, so it is a patch point
    exactly like the reference's.
    """
    xc = spec.x0 + (np.arange(1, spec.ni + 1) - 0.5) * spec.h
    yc = spec.y0 + (np.arange(j_lo, j_hi) - 0.5) * spec.h
    sx = np.sin(TWO_PI * xc[None, :] + 0.35 * np.arange(npde, dtype=np.float64)[:, None])
    cy = np.cos(TWO_PI * yc[None, :] - 0.2 * np.arange(n_lo, n_hi, dtype=np.float64)[:, None])
    return 0.1 * sx[None, :, None, :] * cy[:, None, :, None]


def forcing_amplitudes(planes, npde=NPDE):
    """ap[n][p] = amp[n] * (1 + 0.25 p); amp = 0.8 on plane 1, -0.5 on plane 2."""
    amp = np.zeros(planes)
    if planes > 1:
        amp[1] = 0.8
    if planes > 2:
        amp[2] = -0.5
    pfac = 1.0 + 0.25 * np.arange(npde, dtype=np.float64)
    return np.ascontiguousarray(amp[:, None] * pfac[None, :])


def forcing_vectors(spec):
    """(sin(2 pi x_i), sin(2 pi y_j)): the two factors of the forcing table."""
    xc, yc = cell_centres(spec)
    return np.sin(TWO_PI * xc), np.sin(TWO_PI * yc)


def forcing_table(spec):
    """sxy[j, i] = sin(2 pi x_i) * sin(2 pi y_j) as the reference forms it
    (hbcore.py:169): one rounded product per element -- what the device
    table built from forcing_vectors holds."""
    sx, sy = forcing_vectors(spec)
    return np.ascontiguousarray(sx[None, :] * sy[:, None])


def forcing_values(spec, planes, npde=NPDE):
    """The full (planes, npde, nj, ni) forcing array, for API compatibility."""
    ap = forcing_amplitudes(planes, npde)
    return np.ascontiguousarray(ap[:, :, None, None] * forcing_table(spec)[None, None])


def stencil_coefficients(h):
    """(NU / h^2, ADVECTION / (2 h)) rounded exactly as hbcore.py:256-258."""
    return NU / (h * h), ADVECTION / (2.0 * h)
