"""GPU tile index pinned to the REFERENCE's own pointer-tile allocation
(tests/golden/tiles_*.npz, written by make_golden.py --tiles from
pkg/src/sparselbm/layouts.py:389-401 run in the container).

The reference tiles 2-D domains with 16 x 16 tiles ranked row-major over
the tiles holding >= 1 non-solid node; slot_of = rank * 256 + the row-major
intra-tile index.  The device pipeline runs the same geometry extruded to
nz = 1 with (16, 16, 1) tiles: its tile list (rank order), rank grid and
slot_of must equal the reference's bit-exactly.  With LBM_BRICK=0 the
in-tile order is the reference's row-major order, so slot_of is equal as a
whole; with the default sector bricks it is the documented brick
permutation of the same intra index (layout.cuh brick_x/brick_y)."""

import os

import numpy as np
import pytest

import paper_2108_13241_b200 as lb
from helpers import load_golden

pytestmark = pytest.mark.gpu

CASES = ["mixed_s1", "mixed_s2", "mixed_s3", "porous64", "porous96_lo", "porous72_lo"]


def _sim(types2d, layout="pointer_tile"):
    types = np.ascontiguousarray(np.asarray(types2d, dtype=np.uint8)[None])
    # descriptor values other than the type do not enter the tile index:
    # boundary nodes become walls (no table needed)
    t = types.copy()
    t[(t == 3) | (t == 4)] = 2
    geom = lb.from_arrays("tiles", t, lb.BoundaryValueTable(), periodic=(False, False, True))
    params = lb.FlowParams.from_viscosity(U=0.1, L=16, nu=0.2)
    return lb.Simulation(geom, params, layout=layout, scalar=np.float32, tile=(16, 16, 1))


def _rank_grid(tiles, gy, gx):
    rank = np.full((gy, gx), -1, dtype=np.int32)
    for r, (tx, ty, tz) in enumerate(tiles):
        assert tz == 0
        rank[ty, tx] = r
    return rank


def _brick_intra(ly, lx):
    # fp32 sector bricks on a (16, 16, 1) tile: 4 x 2 x 1 nodes, bricks
    # x-fastest (4 x 8 bricks), nodes x-fastest inside (layout.cuh)
    return ((ly >> 1) * 4 + (lx >> 2)) * 8 + (ly & 1) * 4 + (lx & 3)


@pytest.mark.parametrize("name", CASES)
def test_gpu_pointer_tiles_equal_reference(name):
    g = load_golden(f"tiles_{name}")
    assert int(g["tile_edge"]) == 16
    ref_rank, ref_slot = g["tile_rank"], g["slot_of"]
    gy, gx = ref_rank.shape
    sim = _sim(g["types"])
    tiles, nbr = sim.tile_index()
    assert len(tiles) == int(g["allocated_tiles"]) == sim.field.allocated_tiles
    rank = _rank_grid(tiles, gy, gx)
    assert np.array_equal(rank, ref_rank)
    # every kept tile's in-plane neighbours (dz = 0 row of nbr27) are the
    # reference's rank grid shifted
    for t, (tx, ty, _) in enumerate(tiles):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                qx, qy = tx + dx, ty + dy
                want = ref_rank[qy, qx] if 0 <= qx < gx and 0 <= qy < gy else -1
                assert nbr[t, 9 + (dy + 1) * 3 + (dx + 1)] == want
    slot = sim.field.slot_of[0]
    assert np.array_equal(slot < 0, ref_slot < 0)
    ok = ref_slot >= 0
    assert np.array_equal(slot[ok] // 256, ref_slot[ok] // 256)
    ys, xs = np.nonzero(ok)
    assert np.array_equal(slot[ok] % 256, _brick_intra(ys % 16, xs % 16))


@pytest.mark.parametrize("name", CASES)
def test_gpu_slot_of_equals_reference_row_major(name, monkeypatch):
    monkeypatch.setenv("LBM_BRICK", "0")  # read by lbm_create
    g = load_golden(f"tiles_{name}")
    sim = _sim(g["types"])
    assert np.array_equal(sim.field.slot_of[0], g["slot_of"])
    full = _sim(g["types"], layout="tile")
    assert np.array_equal(full.field.slot_of[0], g["tile_slot_of"])
    assert os.environ["LBM_BRICK"] == "0"
