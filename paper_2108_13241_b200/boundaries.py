"""Scalar boundary-closure API (reference pkg/src/sparselbm/boundaries.py:33-134),
D3Q19.  The closures themselves are the library's host functions, compiled
from the same csrc/d3q19.cuh source the step kernel inlines.

Face with inward normal n and wall velocity u (Hecht & Harting 2010):
    rho   = (sum_{c.n=0} f + 2 sum_{c.n<0} f) / (1 - u.n)
    f_n   = f_-n + rho u.n / 3
    f_n+t = f_-n-t + rho (u.n + u.t) / 6 - N_t,
    N_t   = 1/2 sum_{c.n=0} f (c.t) - rho u.t / 3
"""

from dataclasses import dataclass

import numpy as np

from . import _lib
from .lattice import OPP, Q, moments
from .layouts import NodeType, Orientation

_NORMAL = {Orientation.WEST: (0, 1), Orientation.EAST: (0, -1),
           Orientation.SOUTH: (1, 1), Orientation.NORTH: (1, -1),
           Orientation.BOTTOM: (2, 1), Orientation.TOP: (2, -1)}


@dataclass(frozen=True)
class BcOutcome:
    f: np.ndarray
    rho: float
    velocity: np.ndarray


def bounce_back_gather(f_pre_at_node, missing_direction):
    """Value streaming in from a solid/out-of-domain upstream node: the node's
    own previous f_opp(i) (reference boundaries.py:41-51)."""
    i = int(missing_direction)
    if not 1 <= i < Q:
        raise ValueError(f"direction must be a moving direction 1..18, got {i}")
    f = np.asarray(f_pre_at_node, dtype=np.float64)
    if f.shape != (Q,):
        raise ValueError(f"expected {Q} distribution values, got shape {f.shape}")
    return float(f[OPP[i]])


def _parse_orientation(o):
    if isinstance(o, Orientation):
        if o == Orientation.NONE:
            raise ValueError("wall orientation must name a face")
        return o
    if isinstance(o, (int, np.integer)):
        return _parse_orientation(Orientation(int(o)))
    key = str(o).strip().upper()
    table = {"N": Orientation.NORTH, "NORTH": Orientation.NORTH, "S": Orientation.SOUTH,
             "SOUTH": Orientation.SOUTH, "E": Orientation.EAST, "EAST": Orientation.EAST,
             "W": Orientation.WEST, "WEST": Orientation.WEST, "T": Orientation.TOP,
             "TOP": Orientation.TOP, "B": Orientation.BOTTOM, "BOTTOM": Orientation.BOTTOM}
    if key not in table:
        raise ValueError(f"unknown wall orientation {o!r}")
    return table[key]


def _vec3(u):
    u = np.asarray(u, dtype=np.float64).ravel()
    if u.size == 2:
        u = np.append(u, 0.0)
    if u.size != 3:
        raise ValueError("wall velocity must be a 2- or 3-vector")
    return np.ascontiguousarray(u)


def zou_he_velocity(f_known, wall_orientation, u_wall, dtype=np.float64):
    orient = _parse_orientation(wall_orientation)
    f = np.ascontiguousarray(f_known, dtype=np.float64)
    if f.shape != (Q,):
        raise ValueError(f"expected {Q} distribution values, got shape {f.shape}")
    u = _vec3(u_wall)
    if float(u @ u) >= 1.0:
        raise ValueError(f"wall velocity magnitude must stay below 1, got {u}")
    a, s = _NORMAL[orient]
    if 1.0 - s * u[a] == 0.0:
        raise ValueError(f"imposed normal velocity makes the {orient.name} closure singular")
    out = np.empty(Q)
    _lib.check(_lib.scalar_call("lbm19_zou_he_velocity", dtype, _lib.dptr(f), int(orient),
                                _lib.dptr(u), _lib.dptr(out)))
    rho, _ = moments(out)
    return BcOutcome(f=out, rho=rho, velocity=u.copy())


def zou_he_pressure(f_known, wall_orientation, rho_wall, dtype=np.float64):
    orient = _parse_orientation(wall_orientation)
    if not np.isfinite(rho_wall) or rho_wall <= 0:
        raise ValueError(f"imposed density must be positive, got {rho_wall}")
    f = np.ascontiguousarray(f_known, dtype=np.float64)
    if f.shape != (Q,):
        raise ValueError(f"expected {Q} distribution values, got shape {f.shape}")
    out = np.empty(Q)
    _lib.check(_lib.scalar_call("lbm19_zou_he_pressure", dtype, _lib.dptr(f), int(orient),
                                float(rho_wall), _lib.dptr(out)))
    _, u = moments(out)
    return BcOutcome(f=out, rho=float(rho_wall), velocity=u)


def resolve_boundary(type_tag, orientation, bc_index, gathered_f, boundary_values):
    """Apply a node's closure to its gathered distributions (reference
    boundaries.py:87-110)."""
    f = np.asarray(gathered_f, dtype=np.float64)
    tag = NodeType(int(type_tag))
    if tag in (NodeType.FLUID, NodeType.BOUNCE_BACK_WALL):
        return f.copy()
    if tag == NodeType.SOLID:
        raise ValueError("solid nodes are never resolved")
    if bc_index < 0:
        raise ValueError("boundary node has no boundary-value entry")
    if tag == NodeType.VELOCITY_BC:
        return zou_he_velocity(f, orientation, boundary_values.velocity(bc_index)).f
    return zou_he_pressure(f, orientation, boundary_values.pressure(bc_index)).f
