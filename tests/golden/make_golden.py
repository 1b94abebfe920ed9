"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
D2Q9 solver (`sparselbm`, /root/reference/pkg) in this container.

Run:  python tests/golden/make_golden.py      (needs /root/reference; the
fixtures it writes are committed, so nothing at test time reads the
reference tree).

Every case records the reference geometry arrays, the boundary table, omega,
the canonical (9, n_y, n_x) state after `initialize` and after N steps, the
reference's macroscopic fields and total mass.  The D3Q19 oracle and the GPU
kernel reproduce these through the projection bridge: the
geometry is extruded along a periodic z axis and the 19 populations are
summed over c_z onto the 9 D2Q9 directions.

Cases (reference call sites in brackets):
  mixed_s{1,2,3}   random mixed-BC 16x16 geometry, nu 0.1, 25 steps, f64
                   [pkg/tests/conftest.py:20-69, test_kernel.py:106-116]
  cavity48_f64/32  build_cavity(48, 48, 0.1), nu 0.06, 50 steps
                   [test_kernel.py:132-140, 248-255]
  chan_v           build_channel(48, 16, VelocityInlet((0.05, 0))), nu 0.25, 60 steps
  chan_p           build_channel(48, 16, PressureInlet(1.016)), nu 0.25, 60 steps
  porous64         build_porous_random(64, 0.6, seed=9), nu 0.3, 20 steps
                   [test_kernel.py:119-129]
  box_perturbed    closed 24x24 box, random rho/u perturbation (rng 8), 200 steps
                   [test_kernel.py:235-245]
plus the Ghia (1982) Re = 100 centreline table the reference ships
(pkg/src/sparselbm/data/ghia1982_reference.txt) for the physics check.

Pointer-tile index fixtures (`tiles_<case>.npz`, `python make_golden.py
--tiles`): the reference's own `layouts.allocate(..., "pointer_tile", ...)`
tile rank grid (compacted row-major rank of tiles holding >= 1 non-solid
node, -1 = not allocated; pkg/src/sparselbm/layouts.py:389-401) and its
slot_of map (rank * 256 + row-major intra-tile index, :263-269, 396-399),
plus the fully allocated `tile` layout's slot_of, for porous64 and the
mixed-BC seeds 1-3.
"""

import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"


def _import_reference():
    tmp = tempfile.mkdtemp(prefix="refpkg_")
    dst = os.path.join(tmp, "pkg")
    shutil.copytree(REF, dst)
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tmp, "numba_cache"))
    sys.path.insert(0, os.path.join(dst, "src"))
    sys.path.insert(0, os.path.join(dst, "tests"))
    import sparselbm as slb  # noqa: E402
    import conftest as refconf  # noqa: E402
    return slb, refconf


def canonical(slb, sim):
    n_x, n_y = sim.geometry.dims
    out = np.zeros((9, n_y, n_x), dtype=sim.dtype)
    slots = sim.field.slot_of
    ok = slots >= 0
    for i in range(9):
        out[i][ok] = sim.field.pre[i][slots[ok]]
    return out


def record(slb, name, geom, nu, steps, scalar=np.float64, rho0=1.0, v0=(0.0, 0.0),
           U=0.1):
    n_x, n_y = geom.dims
    params = slb.FlowParams.from_viscosity(U=U, L=n_y - 1, nu=nu)
    sim = slb.Simulation(geom, params, layout="dense", scalar=scalar)
    sim.initialize(rho0=rho0, v0=v0)
    f_init = canonical(slb, sim)
    m0 = slb.total_mass(sim)
    sim.run(steps)
    f_final = canonical(slb, sim)
    rho, vx, vy = sim.macroscopic_fields()
    kinds, vel, rhos = geom.boundary_values.as_arrays(np.float64)
    d = geom.descriptors
    out = dict(types=d.type_tag, orient=d.orientation, bc_index=d.bc_index,
               masks9=d.neighbor_mask, bc_kind=kinds, bc_vel=vel, bc_rho=rhos,
               omega=np.float64(params.omega), steps=np.int64(steps),
               dtype=np.array(np.dtype(scalar).name),
               f_init=f_init, f_final=f_final, rho=rho, vx=vx, vy=vy,
               mass0=np.float64(m0), mass_final=np.float64(slb.total_mass(sim)),
               rho0=np.asarray(rho0, dtype=np.float64),
               v0x=np.asarray(v0[0], dtype=np.float64),
               v0y=np.asarray(v0[1], dtype=np.float64))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, geom.dims, steps, np.dtype(scalar).name, "mass", m0, "->",
          out["mass_final"])


def record_tiles(slb, name, geom):
    from sparselbm import layouts as L
    d = geom.descriptors
    pt = L.allocate(geom.dims, "pointer_tile", np.float64, d.type_tag)
    full = L.allocate(geom.dims, "tile", np.float64, d.type_tag)
    out = dict(types=d.type_tag, tile_edge=np.int64(L.TILE_EDGE),
               tile_rank=pt._tile_rank, slot_of=pt.slot_of,
               allocated_tiles=np.int64(pt.allocated_tiles),
               n_slots=np.int64(pt.n_slots), tile_slot_of=full.slot_of)
    np.savez_compressed(os.path.join(HERE, f"tiles_{name}.npz"), **out)
    print("tiles", name, geom.dims, "allocated", pt.allocated_tiles, "of",
          full.allocated_tiles)


def main_tiles():
    slb, refconf = _import_reference()
    for seed in (1, 2, 3):
        record_tiles(slb, f"mixed_s{seed}", refconf.random_mixed_geometry(seed))
    record_tiles(slb, "porous64", slb.build_porous_random(64, 0.6, seed=9))
    # sparse enough that some 16x16 tiles are all solid (dropped)
    record_tiles(slb, "porous96_lo", slb.build_porous_random(96, 0.35, seed=4))
    # 72 = 4.5 tiles: padded edge tiles
    record_tiles(slb, "porous72_lo", slb.build_porous_random(72, 0.3, seed=5))


def main():
    slb, refconf = _import_reference()
    for seed in (1, 2, 3):
        record(slb, f"mixed_s{seed}", refconf.random_mixed_geometry(seed), 0.1, 25,
               U=0.04)
    record(slb, "cavity48_f64", slb.build_cavity(48, 48, 0.1), 0.06, 50)
    record(slb, "cavity48_f32", slb.build_cavity(48, 48, 0.1), 0.06, 50,
           scalar=np.float32)
    record(slb, "chan_v", slb.build_channel(48, 16, slb.VelocityInlet((0.05, 0.0))),
           0.25, 60)
    record(slb, "chan_p", slb.build_channel(48, 16, slb.PressureInlet(1.016)),
           0.25, 60, rho0=1.008)
    record(slb, "porous64", slb.build_porous_random(64, 0.6, seed=9), 0.3, 20)
    rng = np.random.default_rng(8)
    n = 24
    types = np.full((n, n), slb.NodeType.FLUID, dtype=np.uint8)
    types[0, :] = types[-1, :] = slb.NodeType.BOUNCE_BACK_WALL
    types[:, 0] = types[:, -1] = slb.NodeType.BOUNCE_BACK_WALL
    box = slb.from_arrays("box", types)
    rho0 = 1.0 + 0.02 * (rng.random((n, n)) - 0.5)
    v0 = (0.04 * (rng.random((n, n)) - 0.5), 0.04 * (rng.random((n, n)) - 0.5))
    record(slb, "box_perturbed", box, 0.05, 200, rho0=rho0, v0=v0)

    table = slb.load_ghia_reference()
    yv, uv = table.vertical[100]
    xh, vh = table.horizontal[100]
    np.savez_compressed(os.path.join(HERE, "ghia_re100.npz"),
                        y=np.asarray(yv), u=np.asarray(uv),
                        x=np.asarray(xh), v=np.asarray(vh))
    print("ghia rows", len(yv), len(xh))


if __name__ == "__main__":
    if "--tiles" in sys.argv:
        main_tiles()
    else:
        main()
