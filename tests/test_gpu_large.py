"""The 2^31-node path (config C5 on one GPU, A-A scheme): unsigned 32-bit slot
arithmetic beyond 2^31 slots, checked bitwise against a small column.

A Couette layer driven by a moving TOP lid over a BOTTOM wall, periodic in x
and y: every (x, y) column evolves identically, so after k steps each z plane
of the 1024 x 1024 x 2050 domain (2.15e9 nodes, > 2^31 slots) must equal the
same plane of a 32 x 32 x 2050 column bit for bit."""

import numpy as np
import pytest

import paper_2108_13241_b200 as lb
from paper_2108_13241_b200 import _lib

pytestmark = pytest.mark.gpu


def _couette(nx, ny, nz, u_lid=0.05):
    types = np.full((nz, ny, nx), lb.NodeType.FLUID, dtype=np.uint8)
    orient = np.zeros_like(types)
    bc = np.full(types.shape, -1, dtype=np.int32)
    table = lb.BoundaryValueTable()
    lid = table.add_velocity(u_lid, 0.0, 0.0)
    types[nz - 1] = lb.NodeType.VELOCITY_BC
    orient[nz - 1] = lb.Orientation.TOP
    bc[nz - 1] = lid
    types[0] = lb.NodeType.BOUNCE_BACK_WALL
    return lb.from_arrays("couette", types, table, bc, orient, periodic=(True, True, False))


def _free_device_bytes():
    try:
        import torch
        free, _ = torch.cuda.mem_get_info(0)
        return free
    except Exception:
        return 0


@pytest.mark.slow
def test_2p31_slots_aa_matches_small_column():
    nz, steps = 2050, 33
    if _lib.device_count() < 1 or _free_device_bytes() < 176e9:
        pytest.skip("needs one B200 with ~176 GB free")
    params = lb.FlowParams.from_viscosity(U=0.05, L=nz - 1, nu=0.1)
    small = lb.Simulation(_couette(32, 32, nz), params, scalar=np.float32, scheme="aa")
    small.initialize(1.0)
    small.step(steps)
    planes = [0, 1, 700, 1500, nz - 3, nz - 2, nz - 1]
    want = {z: [a[0, 0, 0] for a in small.macroscopic_box(x=(0, 1), y=(0, 1), z=z)] for z in planes}
    small.close()
    big_geom = _couette(1024, 1024, nz)
    big = lb.Simulation(big_geom, params, scalar=np.float32, scheme="aa")
    del big_geom
    assert big.stats().n_slots > 2 ** 31
    big.initialize(1.0)
    big.step(steps)
    for z in planes:
        got = big.macroscopic_box(z=z)
        for a, w in zip(got, want[z]):
            assert np.all(a == w), z
    assert np.isfinite(big.total_mass())
    big.close()
