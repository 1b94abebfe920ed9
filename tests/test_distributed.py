"""Multi-process z-slab decomposition on CPU (gloo, world size 2 and 3): the
slab split, ghost node types, neighbour wiring and boundary-plane exchange
reproduce the single-domain oracle bitwise (the multi-GPU analogue of
t/test_kernel.py:143-156)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import random_mixed_geometry3
from oracle.slab19 import SlabOracle
from oracle.step19 import OracleSim


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(periodic_z):
    return random_mixed_geometry3(7, n=(11, 9, 12), periodic_z=periodic_z)


def _worker(rank, world, port, periodic_z, steps, out_dir):
    import torch
    from paper_2108_13241_b200.distributed import neighbours, split_z
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = _case(periodic_z)
    z0, z1 = split_z(c["types"].shape[0], world)[rank]
    so = SlabOracle(c["types"], c["orient"], c["bc_index"], c["bc_kind"], c["bc_vel"],
                    c["bc_rho"], 1.25, np.float64, c["periodic"], z0, z1)
    so.initialize(1.0)
    lo, hi = neighbours(rank, world, periodic_z)

    def exchange(bottom, top):
        ops = []
        r_lo = torch.empty(bottom.shape, dtype=torch.float64)
        r_hi = torch.empty(top.shape, dtype=torch.float64)
        # my top plane feeds the upper neighbour's lower ghost and vice versa
        # tag 1: travelling up (top plane -> upper neighbour's lower ghost),
        # tag 2: travelling down; with two ranks and a periodic z both
        # neighbours are the same process, so the tags keep them apart
        if hi is not None:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(top), hi, tag=1))
            ops.append(dist.P2POp(dist.irecv, r_hi, hi, tag=2))
        if lo is not None:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(bottom), lo, tag=2))
            ops.append(dist.P2POp(dist.irecv, r_lo, lo, tag=1))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return (r_lo.numpy() if lo is not None else None,
                r_hi.numpy() if hi is not None else None)

    for _ in range(steps):
        so.step(exchange)
    np.save(os.path.join(out_dir, f"slab{rank}.npy"), so.interior)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,periodic_z", [(2, False), (2, True), (3, True)])
def test_slab_decomposition_matches_single_domain(tmp_path, world, periodic_z):
    steps = 6
    mp.spawn(_worker, args=(world, _free_port(), periodic_z, steps, str(tmp_path)), nprocs=world,
             join=True)
    c = _case(periodic_z)
    ref = OracleSim(c["types"], c["orient"], c["bc_index"], c["bc_kind"], c["bc_vel"], c["bc_rho"],
                    1.25, dtype=np.float64, periodic=c["periodic"])
    ref.initialize(1.0)
    ref.step(steps)
    got = np.concatenate([np.load(tmp_path / f"slab{r}.npy") for r in range(world)], axis=1)
    assert np.array_equal(got, ref.pre)


def test_split_and_ghost_types():
    import paper_2108_13241_b200 as lb
    from paper_2108_13241_b200.distributed import neighbours, slab_geometry, split_z
    assert split_z(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert neighbours(0, 3, False) == (None, 1)
    assert neighbours(2, 3, True) == (1, 0)
    assert neighbours(0, 1, True) == (None, None)
    g = lb.build_channel(16, 10, 12, lb.VelocityInlet((0.05, 0)))
    s0, spec = slab_geometry(g, 0, 6)
    assert s0.descriptors.type_tag.shape == (6, 10, 16)
    assert np.array_equal(spec.ghost_lo, g.descriptors.type_tag[11])   # periodic wrap
    assert np.array_equal(spec.ghost_hi, g.descriptors.type_tag[6])
    c = lb.build_duct_z(12, 12, 12)
    _, spec = slab_geometry(c, 0, 4)
    assert spec.ghost_lo is None and spec.ghost_hi is not None


def test_channel_and_duct_slab_builders_match_global():
    import paper_2108_13241_b200 as lb
    from paper_2108_13241_b200.distributed import channel_slab, duct_slab
    g, spec = duct_slab(16, 12, 5, 1, 3)
    full = lb.build_duct_z(16, 12, 15)
    assert np.array_equal(g.descriptors.type_tag, full.descriptors.type_tag[5:10])
    assert np.array_equal(spec.ghost_lo, full.descriptors.type_tag[4])
    g0, spec0 = duct_slab(16, 12, 5, 0, 3)
    assert spec0.ghost_lo is None
    assert np.array_equal(g0.descriptors.orientation, full.descriptors.orientation[0:5])
    c, cs = channel_slab(16, 12, 4, 2, 3)
    fc = lb.build_channel(16, 12, 12, lb.VelocityInlet((0.05, 0.0, 0.0)))
    assert np.array_equal(c.descriptors.type_tag, fc.descriptors.type_tag[8:12])
    assert cs.nz_global == 12 and cs.z0 == 8


def test_split_z_balanced_tile_aligned():
    from paper_2108_13241_b200.distributed import split_z_balanced
    rng = np.random.default_rng(0)
    types = np.zeros((64, 8, 8), dtype=np.uint8)
    # non-solid mass concentrated at the top: equal plane counts would be unbalanced
    for z in range(64):
        types[z].flat[: int(64 * (z / 63) ** 2)] = 1
    for parts, align in ((2, 8), (4, 8), (3, 4), (8, 8), (5, 1)):
        cuts = split_z_balanced(types, parts, align)
        assert cuts[0][0] == 0 and cuts[-1][1] == 64 and len(cuts) == parts
        assert all(a % align == 0 and b > a for a, b in cuts)
        assert all(cuts[k][1] == cuts[k + 1][0] for k in range(parts - 1))
        loads = [int(np.count_nonzero(types[a:b])) for a, b in cuts]
        # within one aligned block of the ideal share
        blk = max(int(np.count_nonzero(types[z:z + align])) for z in range(0, 64, align))
        assert max(loads) - min(loads) <= 2 * blk
    with pytest.raises(ValueError):
        split_z_balanced(types, 9, 8)
    ragged = rng.integers(0, 2, size=(30, 4, 4)).astype(np.uint8)
    cuts = split_z_balanced(ragged, 3, 8)
    assert cuts[-1] == (16, 30) or cuts[-1][1] == 30

