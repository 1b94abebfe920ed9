"""D3Q19 lattice constants, flow parameters and the scalar per-node API.

Mirrors the reference's `sparselbm.lattice` (pkg/src/sparselbm/lattice.py)
with the D2Q9 tables replaced by D3Q19 ones (indices 0-8 keep the D2Q9
numbering).  `equilibrium`, `moments` and `bgk_collide` call
the library's host functions, which are compiled from the same source
(csrc/d3q19.cuh) as the device kernel.

    direction : 0 rest | 1 +x 2 +y 3 -x 4 -y | 5 (+,+) 6 (-,+) 7 (-,-) 8 (+,-)
                9 +z 10 -z | 11 (+x,+z) 12 (-x,-z) 13 (-x,+z) 14 (+x,-z)
                15 (+y,+z) 16 (-y,-z) 17 (-y,+z) 18 (+y,-z)
"""

from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _lib

Q = 19
D = 3

CX = np.array([0, 1, 0, -1, 0, 1, -1, -1, 1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0], dtype=np.int8)
CY = np.array([0, 0, 1, 0, -1, 1, 1, -1, -1, 0, 0, 0, 0, 0, 0, 1, -1, -1, 1], dtype=np.int8)
CZ = np.array([0, 0, 0, 0, 0, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 1, -1], dtype=np.int8)
OPP = np.array([0, 3, 4, 1, 2, 7, 8, 5, 6, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17],
               dtype=np.int8)
W_EXACT = tuple([Fraction(1, 3)] + [Fraction(1, 18)] * 4 + [Fraction(1, 36)] * 4
                + [Fraction(1, 18)] * 2 + [Fraction(1, 36)] * 8)
W = np.array([float(w) for w in W_EXACT], dtype=np.float64)

# D2Q9 direction k <- D3Q19 directions with the same (c_x, c_y)
PROJECTION_D2Q9 = ((0, 9, 10), (1, 11, 14), (2, 15, 18), (3, 12, 13),
                   (4, 16, 17), (5,), (6,), (7,), (8,))


@dataclass(frozen=True)
class LatticeModel:
    d: int = D
    q: int = Q
    dx: float = 1.0
    dt: float = 1.0

    @property
    def velocities(self):
        return np.stack([CX, CY, CZ], axis=1).astype(np.int64)

    @property
    def weights(self):
        return W.copy()

    @property
    def weights_exact(self):
        return W_EXACT

    @property
    def opposite(self):
        return OPP.copy()


D3Q19 = LatticeModel()


@dataclass(frozen=True)
class FlowParams:
    """Characteristic flow numbers in lattice units (reference lattice.py:72-115):
    Re = U L / nu and omega = 1 / (3 nu + 1/2)."""

    U: float
    L: float
    Re: float
    nu: float
    omega: float

    def __post_init__(self):
        if not all(np.isfinite([self.U, self.L, self.Re, self.nu, self.omega])):
            raise ValueError("flow parameters must be finite")
        if abs(self.Re - self.U * self.L / self.nu) > 1e-12 * abs(self.Re):
            raise ValueError(f"inconsistent parameters: Re={self.Re} but U*L/nu="
                             f"{self.U * self.L / self.nu}")
        expected = omega_from_viscosity(self.nu)
        if abs(self.omega - expected) > 1e-12 * expected:
            raise ValueError(f"omega={self.omega} does not match nu={self.nu}")
        if not 0.0 < self.omega < 2.0:
            raise ValueError(f"omega must lie in (0, 2), got {self.omega}")

    @classmethod
    def from_reynolds(cls, U, L, Re):
        nu = viscosity_from_reynolds(U, L, Re)
        return cls(U=U, L=L, Re=Re, nu=nu, omega=omega_from_viscosity(nu))

    @classmethod
    def from_viscosity(cls, U, L, nu):
        if nu <= 0:
            raise ValueError(f"viscosity must be positive, got {nu}")
        if U <= 0 or L <= 0:
            raise ValueError("U and L must be positive")
        return cls(U=U, L=L, Re=U * L / nu, nu=nu, omega=omega_from_viscosity(nu))


def omega_from_viscosity(nu):
    if not np.isfinite(nu) or nu <= 0:
        raise ValueError(f"viscosity must be positive and finite, got {nu}")
    return 1.0 / (3.0 * nu + 0.5)


def viscosity_from_reynolds(U, L, Re):
    for name, val in (("U", U), ("L", L), ("Re", Re)):
        if not np.isfinite(val) or val <= 0:
            raise ValueError(f"{name} must be positive and finite, got {val}")
    return U * L / Re


def opposite_direction(i):
    if not 0 <= i < Q:
        raise ValueError(f"direction index out of range: {i}")
    return int(OPP[i])


def _vec3(v):
    v = np.asarray(v, dtype=np.float64).ravel()
    if v.size == 2:
        v = np.append(v, 0.0)
    if v.size != 3:
        raise ValueError(f"expected a 2- or 3-vector, got {v}")
    return np.ascontiguousarray(v)


def equilibrium(rho, v, dtype=np.float64):
    """f_i = w_i rho (1 + 3 c.v + 4.5 (c.v)^2 - 1.5 v.v) with the kernel's
    expression tree (lattice.py:136-147)."""
    v = _vec3(v)
    if not (np.isfinite(rho) and np.all(np.isfinite(v))):
        raise ValueError("equilibrium inputs must be finite")
    if float(v @ v) >= 1.0:
        raise ValueError(f"velocity magnitude must stay below 1, got {v}")
    out = np.empty(Q)
    _lib.check(_lib.scalar_call("lbm19_feq", dtype, float(rho), _lib.dptr(v), _lib.dptr(out)))
    return out


def moments(f, dtype=np.float64):
    """Density and velocity of a 19-vector; v = 0 when rho == 0 (lattice.py:150-163)."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    if f.shape != (Q,):
        raise ValueError(f"expected {Q} distribution values, got shape {f.shape}")
    if not np.all(np.isfinite(f)):
        raise ValueError("distribution values must be finite")
    rho = np.zeros(1)
    u = np.zeros(3)
    _lib.check(_lib.scalar_call("lbm19_moments", dtype, _lib.dptr(f), _lib.dptr(rho), _lib.dptr(u)))
    return float(rho[0]), u


def bgk_collide(f, omega, dtype=np.float64):
    """One BGK relaxation of a node's 19 values towards f_eq(moments(f))."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    if f.shape != (Q,) or not np.all(np.isfinite(f)):
        raise ValueError("expected 19 finite distribution values")
    out = np.empty(Q)
    _lib.check(_lib.scalar_call("lbm19_collide", dtype, _lib.dptr(f), float(omega), _lib.dptr(out)))
    return out
