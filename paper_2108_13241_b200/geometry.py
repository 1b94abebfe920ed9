"""3-D geometry builders for the benchmark configurations (host side, run
once per geometry; not on the hot path).

Conventions carried over from the reference (pkg/src/sparselbm/geometry.py:1-30):
* domain walls are wet boundary nodes (bounce-back, velocity or pressure),
  never solid, so an empty cavity or channel has porosity 1;
* obstacles are solid interiors wrapped in a one-node bounce-back ring (the
  3-D ring is the 26-neighbour dilation), so no FLUID node touches SOLID;
* boundary ownership at edges and corners: velocity > pressure > bounce-back.

Builders: `build_cavity` (C1), `build_channel` (C2/C5), `build_duct_z`
(C5 along z), `build_porous_random` (C3, random spheres),
`build_vascular` (C4, seeded bifurcating tube tree).
"""

from dataclasses import dataclass, field

import numpy as np

from .layouts import BoundaryValueTable, NodeDescriptorField, NodeType, Orientation

POROSITY_TOLERANCE = 0.02


class GeometryError(ValueError):
    """Invalid build parameters or conflicting boundary assignments."""


@dataclass
class Provenance:
    case: str
    params: dict = field(default_factory=dict)
    seed: int | None = None


@dataclass
class Geometry:
    descriptors: NodeDescriptorField
    boundary_values: BoundaryValueTable
    porosity: float
    provenance: Provenance

    @property
    def dims(self):
        return self.descriptors.dims

    @property
    def periodic(self):
        return self.descriptors.periodic

    def refresh_porosity(self):
        self.porosity = porosity(self)
        return self.porosity


def porosity(geometry):
    d = geometry.descriptors
    return d.non_solid_count() / d.type_tag.size


def from_arrays(case, type_tag, boundary_values=None, bc_index=None, orientation=None,
                params=None, seed=None, periodic=(False, False, False)):
    """Assemble a Geometry from raw (nz, ny, nx) descriptor arrays
    (reference geometry.py:93-106)."""
    desc = NodeDescriptorField(type_tag, bc_index=bc_index, orientation=orientation,
                               periodic=periodic)
    table = boundary_values if boundary_values is not None else BoundaryValueTable()
    _validate_bc_assignments(desc, table)
    geom = Geometry(descriptors=desc, boundary_values=table, porosity=0.0,
                    provenance=Provenance(case=case, params=dict(params or {}), seed=seed))
    geom.refresh_porosity()
    return geom


def _validate_bc_assignments(desc, table):
    tags = desc.type_tag
    is_bc = (tags == NodeType.VELOCITY_BC) | (tags == NodeType.PRESSURE_BC)
    if np.any(tags > NodeType.PRESSURE_BC):
        raise GeometryError("node type out of range")
    if np.any(desc.orientation > Orientation.BOTTOM):
        raise GeometryError("orientation out of range")
    if not is_bc.any():
        return
    if np.any(is_bc & (desc.bc_index < 0)):
        raise GeometryError("velocity/pressure node without a boundary value")
    if np.any(is_bc & (desc.orientation == Orientation.NONE)):
        raise GeometryError("velocity/pressure node without a wall orientation")
    idx = desc.bc_index[is_bc]
    if int(idx.max()) >= len(table):
        raise GeometryError("bc_index points past the boundary value table")
    if len(table) > 255:
        raise GeometryError("at most 255 boundary-table entries are supported")
    for tag, kind in ((NodeType.VELOCITY_BC, BoundaryValueTable.KIND_VELOCITY),
                      (NodeType.PRESSURE_BC, BoundaryValueTable.KIND_PRESSURE)):
        for i in np.unique(desc.bc_index[tags == tag]):
            if table.kind(int(i)) != kind:
                raise GeometryError(f"boundary entry {i} has the wrong kind for {tag.name}")


def _empty(n_x, n_y, n_z):
    shape = (n_z, n_y, n_x)
    return (np.full(shape, NodeType.FLUID, dtype=np.uint8),
            np.full(shape, -1, dtype=np.int32), np.zeros(shape, dtype=np.uint8))


def build_cavity(n_x, n_y, n_z, U_lid):
    """Lid-driven cavity: the y = n_y - 1 face (edges included) imposes
    velocity (U_lid, 0, 0); the other five faces are bounce-back
    (reference geometry.py:125-150)."""
    if min(n_x, n_y, n_z) < 8:
        raise GeometryError(f"cavity needs at least 8^3 nodes, got {n_x}x{n_y}x{n_z}")
    types, bc_index, orient = _empty(n_x, n_y, n_z)
    types[:, 0, :] = NodeType.BOUNCE_BACK_WALL
    types[:, :, 0] = NodeType.BOUNCE_BACK_WALL
    types[:, :, n_x - 1] = NodeType.BOUNCE_BACK_WALL
    types[0, :, :] = NodeType.BOUNCE_BACK_WALL
    types[n_z - 1, :, :] = NodeType.BOUNCE_BACK_WALL
    table = BoundaryValueTable()
    lid = table.add_velocity(U_lid, 0.0, 0.0)
    types[:, n_y - 1, :] = NodeType.VELOCITY_BC
    bc_index[:, n_y - 1, :] = lid
    orient[:, n_y - 1, :] = Orientation.NORTH
    return from_arrays("cavity", types, table, bc_index, orient,
                       params={"U": repr(float(U_lid)), "L": str(n_y - 1)})


class VelocityInlet:
    def __init__(self, v):
        v = tuple(float(c) for c in v)
        self.v = v + (0.0,) * (3 - len(v))


class PressureInlet:
    def __init__(self, rho):
        self.rho = float(rho)


def build_channel(n_x, n_y, n_z, inlet, outlet_rho=1.0, periodic_z=True):
    """Straight channel along x: inlet face x = 0, constant-pressure outlet
    x = n_x - 1, bounce-back walls at y = 0 / n_y - 1 and -- unless the span
    is periodic -- at z = 0 / n_z - 1 (reference geometry.py:162-203)."""
    if not (n_x >= 8 and n_y >= 8 and n_z >= 1):
        raise GeometryError(f"channel too small: {n_x}x{n_y}x{n_z}")
    types, bc_index, orient = _empty(n_x, n_y, n_z)
    types[:, 0, :] = NodeType.BOUNCE_BACK_WALL
    types[:, n_y - 1, :] = NodeType.BOUNCE_BACK_WALL
    if not periodic_z:
        types[0, :, :] = NodeType.BOUNCE_BACK_WALL
        types[n_z - 1, :, :] = NodeType.BOUNCE_BACK_WALL
    table = BoundaryValueTable()
    if isinstance(inlet, VelocityInlet):
        inlet_idx = table.add_velocity(*inlet.v)
        inlet_type = NodeType.VELOCITY_BC
        case, params = "chan_v", {"inlet_v": repr(inlet.v)}
    elif isinstance(inlet, PressureInlet):
        inlet_idx = table.add_pressure(inlet.rho)
        inlet_type = NodeType.PRESSURE_BC
        case, params = "chan_p", {"inlet_rho": repr(inlet.rho)}
    else:
        raise GeometryError("inlet must be VelocityInlet or PressureInlet")
    outlet_idx = table.add_pressure(outlet_rho)
    params["outlet_rho"] = repr(float(outlet_rho))
    types[:, :, n_x - 1] = NodeType.PRESSURE_BC
    bc_index[:, :, n_x - 1] = outlet_idx
    orient[:, :, n_x - 1] = Orientation.EAST
    types[:, :, 0] = inlet_type
    bc_index[:, :, 0] = inlet_idx
    orient[:, :, 0] = Orientation.WEST
    return from_arrays(case, types, table, bc_index, orient, params=params,
                       periodic=(False, False, bool(periodic_z)))


def build_duct_z(n_x, n_y, n_z, u_in=0.05, outlet_rho=1.0):
    """Square duct along z (config C5): bounce-back x/y faces, velocity inlet
    at z = 0 (orientation BOTTOM), pressure outlet at z = n_z - 1 (TOP)."""
    types, bc_index, orient = _empty(n_x, n_y, n_z)
    types[:, 0, :] = types[:, n_y - 1, :] = NodeType.BOUNCE_BACK_WALL
    types[:, :, 0] = types[:, :, n_x - 1] = NodeType.BOUNCE_BACK_WALL
    table = BoundaryValueTable()
    inl = table.add_velocity(0.0, 0.0, u_in)
    out = table.add_pressure(outlet_rho)
    types[n_z - 1] = NodeType.PRESSURE_BC
    bc_index[n_z - 1] = out
    orient[n_z - 1] = Orientation.TOP
    types[0] = NodeType.VELOCITY_BC
    bc_index[0] = inl
    orient[0] = Orientation.BOTTOM
    return from_arrays("duct_z", types, table, bc_index, orient,
                       params={"u_in": repr(float(u_in)), "outlet_rho": repr(float(outlet_rho))})


def dilate26(mask):
    """26-neighbour (3x3x3) binary dilation without wrap."""
    out = mask.copy()
    for axis in range(3):
        src = out.copy()
        sl_a = [slice(None)] * 3
        sl_b = [slice(None)] * 3
        sl_a[axis], sl_b[axis] = slice(1, None), slice(None, -1)
        out[tuple(sl_a)] |= src[tuple(sl_b)]
        out[tuple(sl_b)] |= src[tuple(sl_a)]
    return out


def _porous_shell(n_x, n_y, n_z, rho_in=1.016, rho_out=1.0):
    """Pressure inlet x = 0, pressure outlet x = n_x - 1, bounce-back y and z
    faces (reference geometry.py:281-299 in 3-D)."""
    types, bc_index, orient = _empty(n_x, n_y, n_z)
    table = BoundaryValueTable()
    inlet = table.add_pressure(rho_in)
    outlet = table.add_pressure(rho_out)
    types[:, 0, :] = types[:, n_y - 1, :] = NodeType.BOUNCE_BACK_WALL
    types[0, :, :] = types[n_z - 1, :, :] = NodeType.BOUNCE_BACK_WALL
    types[:, :, 0] = NodeType.PRESSURE_BC
    bc_index[:, :, 0] = inlet
    orient[:, :, 0] = Orientation.WEST
    types[:, :, n_x - 1] = NodeType.PRESSURE_BC
    bc_index[:, :, n_x - 1] = outlet
    orient[:, :, n_x - 1] = Orientation.EAST
    return types, bc_index, orient, table


def _apply_solids(types, solid):
    solid = solid & (types == NodeType.FLUID)   # walls win over solids
    types[solid] = NodeType.SOLID
    ring = dilate26(solid) & ~solid & (types == NodeType.FLUID)
    types[ring] = NodeType.BOUNCE_BACK_WALL


REGULAR_GRID = 8


def build_porous_regular(n, phi_target, dims=None):
    """Regular sphere packing (reference build_porous_regular,
    geometry.py:315-370, in 3-D): an 8 x 8 x 8 array of equal spheres on a
    uniform grid (spacing n/8, offset n/16) whose radius is chosen by
    bisection to hit the target porosity within 0.02; same walls and
    pressure drop as build_porous_random."""
    if not 0.3 <= phi_target <= 1.0:
        raise GeometryError(f"regular arrays cover porosity 0.3..1.0, got {phi_target}")
    n_x, n_y, n_z = dims if dims is not None else (n, n, n)
    if min(n_x, n_y, n_z) < 8 * REGULAR_GRID:
        raise GeometryError(f"domain too small for an 8x8x8 sphere array: {(n_x, n_y, n_z)}")
    sp = (n_x / REGULAR_GRID, n_y / REGULAR_GRID, n_z / REGULAR_GRID)
    cx = np.round((np.arange(REGULAR_GRID) + 0.5) * sp[0]).astype(np.int64)
    cy = np.round((np.arange(REGULAR_GRID) + 0.5) * sp[1]).astype(np.int64)
    cz = np.round((np.arange(REGULAR_GRID) + 0.5) * sp[2]).astype(np.int64)
    # squared distance to the nearest sphere centre, separable per axis
    dx = np.min((np.arange(n_x)[:, None] - cx[None, :]) ** 2, axis=1)
    dy = np.min((np.arange(n_y)[:, None] - cy[None, :]) ** 2, axis=1)
    dz = np.min((np.arange(n_z)[:, None] - cz[None, :]) ** 2, axis=1)
    d2 = dz[:, None, None] + dy[None, :, None] + dx[None, None, :]

    def achieved(radius):
        types, bc_index, orient, table = _porous_shell(n_x, n_y, n_z)
        if radius > 0:
            _apply_solids(types, (d2 <= radius * radius) & (types == NodeType.FLUID))
        return 1.0 - np.count_nonzero(types == NodeType.SOLID) / types.size, (types, bc_index, orient, table)

    lo, hi = 0.0, float(min(sp))
    phi_lo, grids = achieved(lo)
    best_err, radius = abs(phi_lo - phi_target), lo
    if best_err > POROSITY_TOLERANCE:
        phi_hi, grids_hi = achieved(hi)
        if phi_hi > phi_target + POROSITY_TOLERANCE:
            raise GeometryError(f"target porosity {phi_target} unreachable (minimum about {phi_hi:.3f})")
        if abs(phi_hi - phi_target) < best_err:
            best_err, radius, grids = abs(phi_hi - phi_target), hi, grids_hi
        for _ in range(60):
            if best_err <= POROSITY_TOLERANCE:
                break
            mid = 0.5 * (lo + hi)
            phi_mid, grids_mid = achieved(mid)
            if abs(phi_mid - phi_target) < best_err:
                best_err, radius, grids = abs(phi_mid - phi_target), mid, grids_mid
            if phi_mid > phi_target:
                lo = mid
            else:
                hi = mid
    types, bc_index, orient, table = grids
    return from_arrays("porous_regular", types, table, bc_index, orient,
                       params={"phi_target": repr(float(phi_target)), "radius": repr(float(radius))})


def build_porous_random(n, phi_target, seed, radius_range=(4, 32), dims=None,
                        max_attempts=200_000):
    """Random-sphere porous medium (config C3; reference
    build_porous_random, geometry.py:373-417, in 3-D).  Spheres with radii
    uniform in `radius_range` are placed until the porosity falls inside
    phi_target +- 0.02; a candidate that overshoots is rejected and the radius
    cap halves.  The porosity is tracked incrementally (solid count inside the
    interior), so the build is O(sum of sphere volumes), deterministic per seed.
    """
    if not 0.1 <= phi_target <= 1.0:
        raise GeometryError(f"random packings cover porosity 0.1..1.0, got {phi_target}")
    n_x, n_y, n_z = dims if dims is not None else (n, n, n)
    if min(n_x, n_y, n_z) < 16:
        raise GeometryError("domain too small for random spheres")
    rng = np.random.default_rng(seed)
    r_lo, r_hi = radius_range
    types, bc_index, orient, table = _porous_shell(n_x, n_y, n_z)
    interior = types == NodeType.FLUID
    solid = np.zeros_like(interior)
    total = types.size
    n_solid = 0
    phi = 1.0
    attempts = 0
    cap = r_hi
    while phi > phi_target + POROSITY_TOLERANCE and attempts < max_attempts:
        attempts += 1
        r = int(rng.integers(r_lo, cap + 1))
        cx = int(rng.integers(1, n_x - 1))
        cy = int(rng.integers(1, n_y - 1))
        cz = int(rng.integers(1, n_z - 1))
        x0, x1 = max(1, cx - r), min(n_x - 2, cx + r)
        y0, y1 = max(1, cy - r), min(n_y - 2, cy + r)
        z0, z1 = max(1, cz - r), min(n_z - 2, cz + r)
        zz, yy, xx = np.ogrid[z0:z1 + 1, y0:y1 + 1, x0:x1 + 1]
        ball = (xx - cx) ** 2 + (yy - cy) ** 2 + (zz - cz) ** 2 <= r * r
        box = (slice(z0, z1 + 1), slice(y0, y1 + 1), slice(x0, x1 + 1))
        new = ball & ~solid[box] & interior[box]
        added = int(np.count_nonzero(new))
        phi_trial = 1.0 - (n_solid + added) / total
        if phi_trial < phi_target - POROSITY_TOLERANCE:
            cap = max(r_lo, r // 2)
            continue
        solid[box] |= new
        n_solid += added
        phi = phi_trial
    _apply_solids(types, solid)
    return from_arrays("porous_random", types, table, bc_index, orient,
                       params={"phi_target": repr(float(phi_target)),
                               "radius_range": repr(tuple(radius_range))},
                       seed=int(seed))


def _capsule(lumen, p0, p1, r):
    """Mark nodes within distance r of the segment p0-p1 (clipped)."""
    n_z, n_y, n_x = lumen.shape
    lo = np.floor(np.minimum(p0, p1) - r).astype(int)
    hi = np.ceil(np.maximum(p0, p1) + r).astype(int)
    lo = np.maximum(lo, 0)
    hi = np.minimum(hi, [n_x - 1, n_y - 1, n_z - 1])
    if np.any(lo > hi):
        return
    zz, yy, xx = np.ogrid[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1]
    d = p1 - p0
    L2 = float(d @ d)
    px, py, pz = xx - p0[0], yy - p0[1], zz - p0[2]
    t = (px * d[0] + py * d[1] + pz * d[2]) / (L2 if L2 > 0 else 1.0)
    t = np.clip(t, 0.0, 1.0)
    qx, qy, qz = px - t * d[0], py - t * d[1], pz - t * d[2]
    inside = qx * qx + qy * qy + qz * qz <= r * r
    lumen[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1] |= inside


def _grow(lumen, rng, p, direction, r, length, depth, r_min):
    end = p + direction * length
    _capsule(lumen, p, end, r)
    if depth == 0 or r * 0.79 < r_min:
        return
    # two children: Murray's law radius, rotated about a random axis
    axis = rng.normal(size=3)
    axis -= direction * (axis @ direction)
    axis /= np.linalg.norm(axis) + 1e-12
    for sign in (1.0, -1.0):
        ang = sign * rng.uniform(0.35, 0.7)
        c, s = np.cos(ang), np.sin(ang)
        dnew = direction * c + np.cross(axis, direction) * s
        dnew /= np.linalg.norm(dnew)
        _grow(lumen, rng, end, dnew, r * 0.79, length * rng.uniform(0.7, 0.9),
              depth - 1, r_min)


def build_vascular(n, seed, fluid_fraction=0.05, dims=None, r_root=None, depth=6):
    """Seeded bifurcating tube forest (config C4): lumen FLUID, a one-node
    bounce-back ring, everything else SOLID.  Trees enter through the x = 0
    face; lumen nodes on the x = 0 face are a pressure inlet (rho 1.01), lumen
    nodes on any other face a pressure outlet (rho 1.0) oriented to that face.
    Trees are added until the non-solid fraction reaches `fluid_fraction`."""
    n_x, n_y, n_z = dims if dims is not None else (n, n, n)
    rng = np.random.default_rng(seed)
    r0 = r_root if r_root is not None else max(2.5, min(n_x, n_y, n_z) / 40.0)
    lumen = np.zeros((n_z, n_y, n_x), dtype=bool)
    total = lumen.size
    trees = 0
    frac = 0.0
    while frac < fluid_fraction and trees < 4096:
        trees += 1
        p = np.array([0.0, rng.uniform(0.15, 0.85) * (n_y - 1),
                      rng.uniform(0.15, 0.85) * (n_z - 1)])
        d = np.array([1.0, rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3)])
        d /= np.linalg.norm(d)
        _grow(lumen, rng, p, d, r0, 0.3 * n_x, depth, 1.0)
        if trees % 4 == 0:   # non-solid = lumen + its ring
            frac = np.count_nonzero(dilate26(lumen)) / total
    types = np.full((n_z, n_y, n_x), NodeType.SOLID, dtype=np.uint8)
    ring = dilate26(lumen) & ~lumen
    types[lumen] = NodeType.FLUID
    types[ring] = NodeType.BOUNCE_BACK_WALL
    bc_index = np.full(types.shape, -1, dtype=np.int32)
    orient = np.zeros(types.shape, dtype=np.uint8)
    table = BoundaryValueTable()
    inlet = table.add_pressure(1.01)
    outlet = table.add_pressure(1.0)
    # faces in reverse priority order so x = 0 (inlet) wins at shared edges
    faces = [((slice(None), slice(None), n_x - 1), Orientation.EAST),
             ((slice(None), 0, slice(None)), Orientation.SOUTH),
             ((slice(None), n_y - 1, slice(None)), Orientation.NORTH),
             ((0, slice(None), slice(None)), Orientation.BOTTOM),
             ((n_z - 1, slice(None), slice(None)), Orientation.TOP)]
    for sl, o in faces:
        sel = lumen[sl]
        t = types[sl]
        b = bc_index[sl]
        oo = orient[sl]
        t[sel] = NodeType.PRESSURE_BC
        b[sel] = outlet
        oo[sel] = o
    sl = (slice(None), slice(None), 0)
    sel = lumen[sl]
    types[sl][sel] = NodeType.PRESSURE_BC
    bc_index[sl][sel] = inlet
    orient[sl][sel] = Orientation.WEST
    return from_arrays("vascular", types, table, bc_index, orient,
                       params={"fluid_fraction": repr(float(fluid_fraction)),
                               "trees": str(trees)}, seed=int(seed))
