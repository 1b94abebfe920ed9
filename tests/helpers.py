"""Shared test fixtures: golden-vector loading, the projection bridge
 and 3-D geometry generators mirroring the reference's
random mixed-BC geometry (pkg/tests/conftest.py:20-69)."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GOLDEN_CASES = ["mixed_s1", "mixed_s2", "mixed_s3", "cavity48_f64", "cavity48_f32",
                "chan_v", "chan_p", "porous64", "box_perturbed"]
PROJECTION = ((0, 9, 10), (1, 11, 14), (2, 15, 18), (3, 12, 13), (4, 16, 17),
              (5,), (6,), (7,), (8,))

SOLID, FLUID, WALL, VEL, PRES = 0, 1, 2, 3, 4
NORTH, SOUTH, EAST, WEST, TOP, BOTTOM = 1, 2, 3, 4, 5, 6


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def project(f19):
    """Sum D3Q19 populations over c_z onto the 9 D2Q9 directions."""
    f19 = np.asarray(f19, dtype=np.float64)
    return np.stack([sum(f19[j] for j in P) for P in PROJECTION])


def extruded_case(g, nz):
    """3-D arrays of a 2-D golden case extruded along a periodic z axis."""
    ext = lambda a: np.ascontiguousarray(np.repeat(np.asarray(a)[None], nz, axis=0))
    bc_vel = np.concatenate([g["bc_vel"], np.zeros((len(g["bc_vel"]), 1))], axis=1)
    rho0 = g["rho0"]
    v0 = (g["v0x"], g["v0y"], 0.0)
    if rho0.ndim:
        rho0 = ext(rho0)
        v0 = (ext(g["v0x"]), ext(g["v0y"]), 0.0)
    else:
        rho0, v0 = float(rho0), (float(g["v0x"]), float(g["v0y"]), 0.0)
    return dict(types=ext(g["types"]), orient=ext(g["orient"]), bc_index=ext(g["bc_index"]),
                bc_kind=g["bc_kind"], bc_vel=bc_vel, bc_rho=g["bc_rho"],
                omega=float(g["omega"]), steps=int(g["steps"]),
                dtype=np.dtype(str(g["dtype"])), rho0=rho0, v0=v0,
                periodic=(False, False, True))


def random_mixed_geometry3(seed, n=(12, 10, 8), solid_fraction=0.12, periodic_z=False):
    """Every boundary kind on a small box: velocity inlet (west), pressure
    outlet (east), moving lid (north), bounce-back floor (south), velocity /
    pressure z faces (bottom / top) unless z is periodic, random solid
    blobs with 26-neighbour bounce-back rings inside."""
    nx, ny, nz = n
    rng = np.random.default_rng(seed)
    types = np.full((nz, ny, nx), FLUID, dtype=np.uint8)
    bc = np.full(types.shape, -1, dtype=np.int32)
    orient = np.zeros(types.shape, dtype=np.uint8)
    kinds, vel, rho = [], [], []

    def add_v(v):
        kinds.append(0), vel.append(v), rho.append(0.0)
        return len(kinds) - 1

    def add_p(r):
        kinds.append(1), vel.append((0.0, 0.0, 0.0)), rho.append(r)
        return len(kinds) - 1

    inlet = add_v((0.04, 0.01, 0.005))
    lid = add_v((0.03, 0.0, 0.01))
    outlet = add_p(1.002)
    bottom = add_v((0.0, 0.0, 0.02))
    top = add_p(0.998)

    def face(sl, t, b, o):
        types[sl], bc[sl], orient[sl] = t, b, o

    types[:, 0, :] = WALL
    if not periodic_z:
        face((nz - 1, slice(None), slice(None)), PRES, top, TOP)
        face((0, slice(None), slice(None)), VEL, bottom, BOTTOM)
    face((slice(None), slice(None), nx - 1), PRES, outlet, EAST)
    face((slice(None), ny - 1, slice(None)), VEL, lid, NORTH)
    face((slice(None), slice(None), 0), VEL, inlet, WEST)
    # velocity beats pressure beats bounce-back at shared edges
    face((slice(None), ny - 1, 0), VEL, lid, NORTH)
    solid = np.zeros(types.shape, dtype=bool)
    zlo = 0 if periodic_z else 2
    zhi = nz if periodic_z else nz - 2
    solid[zlo:zhi, 2:-2, 2:-2] = rng.random((zhi - zlo, ny - 4, nx - 4)) < solid_fraction
    types[solid] = SOLID
    ring = np.zeros_like(solid)
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                sh = np.roll(solid, (dz, dy, dx), axis=(0, 1, 2))
                if not periodic_z:
                    if dz == 1:
                        sh[0] = False
                    if dz == -1:
                        sh[-1] = False
                if dy == 1:
                    sh[:, 0] = False
                if dy == -1:
                    sh[:, -1] = False
                if dx == 1:
                    sh[:, :, 0] = False
                if dx == -1:
                    sh[:, :, -1] = False
                ring |= sh
    ring &= ~solid & (types == FLUID)
    types[ring] = WALL
    return dict(types=types, orient=orient, bc_index=bc, bc_kind=np.array(kinds, np.uint8),
                bc_vel=np.array(vel, float), bc_rho=np.array(rho, float),
                periodic=(False, False, periodic_z))


def to_geometry(case, name="case"):
    """Wrap raw arrays into the package's Geometry."""
    from paper_2108_13241_b200 import BoundaryValueTable, from_arrays
    t = BoundaryValueTable()
    for k, v, r in zip(case["bc_kind"], case["bc_vel"], case["bc_rho"]):
        if k == 0:
            t.add_velocity(*v)
        else:
            t.add_pressure(r)
    return from_arrays(name, case["types"], t, case["bc_index"], case["orient"],
                       periodic=case["periodic"])


def oracle_sim(case, omega, dtype):
    from oracle.step19 import OracleSim
    return OracleSim(case["types"], case["orient"], case["bc_index"], case["bc_kind"],
                     case["bc_vel"], case["bc_rho"], omega, dtype=dtype,
                     periodic=case["periodic"])
