"""GPU z-slab halo (fused peer stores + device flags): several slab handles
on one device (same process: device pointers; two processes: CUDA IPC)
reproduce the single-domain run bitwise."""

import os
import socket

import numpy as np
import pytest

import paper_2108_13241_b200 as lb
from helpers import oracle_sim, random_mixed_geometry3, to_geometry
from paper_2108_13241_b200.distributed import (connect_local, slab_geometry, split_z,
                                                split_z_balanced)

pytestmark = pytest.mark.gpu


def _params(omega):
    return lb.FlowParams.from_viscosity(U=0.1, L=10, nu=(1.0 / omega - 0.5) / 3.0)


@pytest.mark.parametrize("nslab,periodic_z,dtype", [(2, False, np.float32), (2, True, np.float64),
                                                    (3, True, np.float32), (4, False, np.float64),
                                                    (5, True, np.float32)])
def test_slabs_in_process_bitwise(nslab, periodic_z, dtype):
    c = random_mixed_geometry3(11, n=(19, 12, 17), periodic_z=periodic_z)
    geom = to_geometry(c)
    params = _params(1.3)
    single = lb.Simulation(geom, params, scalar=dtype)
    single.initialize(1.0)
    sims = []
    for z0, z1 in split_z(17, nslab):
        g, spec = slab_geometry(geom, z0, z1)
        sims.append(lb.Simulation(g, params, scalar=dtype, slab=spec))
    connect_local(sims, periodic_z)
    for s in sims:
        s.initialize(1.0)
    for chunk in (1, 3, 16, 40):   # 40: a 32-step CUDA-graph replay (wait / boundary / signal / interior)
        single.step(chunk)
        for s in sims:
            s.step(chunk, block=False)
        for s in sims:
            s.synchronize()
        got = np.concatenate([s.canonical_state() for s in sims], axis=1)
        assert np.array_equal(got, single.canonical_state()), chunk
    # flags at the cuts are bit-exact too
    fl = np.concatenate([s.flag_words() for s in sims], axis=0)
    assert np.array_equal(fl, single.flag_words())
    ref = oracle_sim(c, params.omega, dtype)
    ref.initialize(1.0)
    ref.step(single.step_count)
    assert np.array_equal(single.canonical_state(), ref.pre)


@pytest.mark.parametrize("layout,tile,nslab,periodic_z,dtype", [
    ("pointer_tile", (8, 4, 4), 2, False, np.float32),
    ("pointer_tile", (8, 4, 4), 3, True, np.float64),
    ("pointer_tile", (4, 4, 2), 5, True, np.float32),
    ("tile", (8, 8, 4), 2, True, np.float32),
    ("pointer_tile", (8, 8, 8), 2, False, np.float64),
    ("pointer_tile", (4, 8, 16), 2, False, np.float32),
    ("pointer_tile", (8, 8, 8), 3, True, np.float32),
    ("pointer_tile", (8, 4, 8), 2, True, "wl"),
    ("pointer_tile", (8, 8, 8), 3, False, "wl")])
def test_tile_slabs_in_process_bitwise(layout, tile, nslab, periodic_z, dtype, monkeypatch):
    """Sparse z-slabs: cuts on tile planes balanced by non-solid count; the
    boundary tiles exchange through ghost planes inside the step kernel.
    "wl": the warp work list (forced), whose slab steps run the boundary tile
    planes' items first, signal, then the interior items."""
    if dtype == "wl":
        monkeypatch.setenv("LBM_STEP_VARIANT", "8")
        dtype = np.float32
    c = random_mixed_geometry3(13, n=(19, 12, 24), periodic_z=periodic_z)
    geom = to_geometry(c)
    params = _params(1.25)
    single = lb.Simulation(geom, params, layout=layout, scalar=dtype, tile=tile)
    single.initialize(1.0)
    sims = []
    cuts = split_z_balanced(geom.descriptors.type_tag, nslab, align=tile[2])
    for z0, z1 in cuts:
        assert z0 % tile[2] == 0
        g, spec = slab_geometry(geom, z0, z1)
        sims.append(lb.Simulation(g, params, layout=layout, scalar=dtype, tile=tile, slab=spec))
    connect_local(sims, periodic_z)
    for s in sims:
        s.initialize(1.0)
    for chunk in (1, 2, 13, 40):
        single.step(chunk)
        for s in sims:
            s.step(chunk, block=False)
        for s in sims:
            s.synchronize()
        got = np.concatenate([s.canonical_state() for s in sims], axis=1)
        assert np.array_equal(got, single.canonical_state()), chunk
    ref = oracle_sim(c, params.omega, dtype)
    ref.initialize(1.0)
    ref.step(single.step_count)
    assert np.array_equal(single.canonical_state(), ref.pre)


@pytest.mark.parametrize("nslab,periodic_z,dtype", [(2, False, np.float32), (3, True, np.float64),
                                                    (4, False, np.float32), (2, True, np.float32)])
def test_aa_slabs_in_process_bitwise(nslab, periodic_z, dtype):
    """A-A z-slabs: the neighbour step reads and writes the neighbouring
    slab's boundary plane directly; odd and even step counts decode to the
    single-domain AB run bitwise."""
    c = random_mixed_geometry3(14, n=(19, 12, 17), periodic_z=periodic_z)
    geom = to_geometry(c)
    params = _params(1.3)
    single = lb.Simulation(geom, params, scalar=dtype)
    single.initialize(1.0)
    sims = []
    for z0, z1 in split_z(17, nslab):
        g, spec = slab_geometry(geom, z0, z1)
        sims.append(lb.Simulation(g, params, scalar=dtype, slab=spec, scheme="aa"))
    connect_local(sims, periodic_z)
    for s in sims:
        s.initialize(1.0)
    for chunk in (1, 2, 1, 37):
        single.step(chunk)
        for s in sims:
            s.step(chunk, block=False)
        for s in sims:
            s.synchronize()
        got = np.concatenate([s.canonical_state() for s in sims], axis=1)
        assert np.array_equal(got, single.canonical_state()), (chunk, single.step_count)
        rho = np.concatenate([s.macroscopic_fields()[0] for s in sims], axis=0)
        assert np.array_equal(rho, single.macroscopic_fields()[0])
    # odd step count: state writes are refused (boundary pre_i lives in the neighbour)
    assert sims[0].step_count % 2 == 1
    with pytest.raises(RuntimeError):
        sims[0].set_state(sims[0].canonical_state())


@pytest.mark.parametrize("tile,nslab,periodic_z,dtype,variant", [
    ((8, 4, 4), 2, False, np.float32, None), ((8, 4, 4), 3, True, np.float64, None),
    ((4, 8, 8), 2, True, np.float32, "8"), ((8, 8, 8), 3, False, np.float32, "8"),
    ((4, 4, 2), 4, True, np.float32, "7")])
def test_aa_tile_slabs_in_process_bitwise(tile, nslab, periodic_z, dtype, variant, monkeypatch):
    """A-A z-slabs of pointer tiles: the neighbour step reaches into the
    neighbouring slab's tile storage through its rank grid (peer memory) and
    mirrors its cross-cut pushes for the phase-1 readback; CTA-per-tile and
    work-list kernels, odd and even step counts, graph replay (37 steps), vs
    the single-domain AB run, bitwise."""
    if variant:
        monkeypatch.setenv("LBM_STEP_VARIANT", variant)
    c = random_mixed_geometry3(15, n=(19, 12, 24), periodic_z=periodic_z)
    geom = to_geometry(c)
    params = _params(1.2)
    single = lb.Simulation(geom, params, scalar=dtype)
    single.initialize(1.0)
    sims = []
    for z0, z1 in split_z_balanced(geom.descriptors.type_tag, nslab, align=tile[2]):
        g, spec = slab_geometry(geom, z0, z1)
        sims.append(lb.Simulation(g, params, layout="pointer_tile", scalar=dtype, tile=tile, slab=spec,
                                  scheme="aa"))
    connect_local(sims, periodic_z)
    for s in sims:
        s.initialize(1.0)
    for chunk in (1, 2, 1, 37):
        single.step(chunk)
        for s in sims:
            s.step(chunk, block=False)
        for s in sims:
            s.synchronize()
        got = np.concatenate([s.canonical_state() for s in sims], axis=1)
        assert np.array_equal(got, single.canonical_state()), (chunk, single.step_count)
        rho = np.concatenate([s.macroscopic_fields()[0] for s in sims], axis=0)
        assert np.array_equal(rho, single.macroscopic_fields()[0])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, out_dir, layout="dense"):
    import torch.distributed as dist
    from paper_2108_13241_b200.distributed import connect_distributed
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = random_mixed_geometry3(12, n=(21, 10, 14), periodic_z=True)
    geom = to_geometry(c)
    z0, z1 = split_z(14, world)[rank]
    g, spec = slab_geometry(geom, z0, z1)
    scheme = "aa" if layout.endswith("-aa") else "ab"
    sim = lb.Simulation(g, _params(1.1), layout=layout.replace("-aa", ""), scalar=np.float32, slab=spec,
                        device=0, tile=(8, 4, 1), scheme=scheme)
    connect_distributed(sim, periodic_z=True)
    sim.initialize(1.0)
    sim.step(25)
    np.save(os.path.join(out_dir, f"ipc{rank}.npy"), sim.canonical_state())
    dist.barrier()
    sim.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("layout", ["dense", "pointer_tile", "dense-aa", "pointer_tile-aa"])
def test_slabs_two_processes_ipc_bitwise(tmp_path, layout):
    import torch.multiprocessing as mp
    mp.spawn(_ipc_worker, args=(2, _free_port(), str(tmp_path), layout), nprocs=2, join=True)
    c = random_mixed_geometry3(12, n=(21, 10, 14), periodic_z=True)
    single = lb.Simulation(to_geometry(c), _params(1.1), scalar=np.float32)
    single.initialize(1.0)
    single.step(25)
    got = np.concatenate([np.load(tmp_path / f"ipc{r}.npy") for r in range(2)], axis=1)
    assert np.array_equal(got, single.canonical_state())


def test_default_tile_on_slabs_is_fixed():
    """tile=None: a single domain of a low-fill medium takes 4x4x4 tiles, z-slabs
    of the same medium keep 4x4x8 (every rank cuts on the same tile planes), and
    the AB work-list slabs with that default reproduce the single domain bitwise."""
    geom = lb.build_porous_random(32, 0.15, seed=1, radius_range=(2, 6), dims=(32, 16, 32))
    params = lb.FlowParams.from_viscosity(U=0.05, L=15, nu=0.2)
    single = lb.Simulation(geom, params, layout="pointer_tile", scalar=np.float32)
    assert single.tile == (4, 4, 4)
    single.initialize(1.004)
    sims = []
    for z0, z1 in split_z_balanced(geom.descriptors.type_tag, 2, align=lb.layouts.DEFAULT_TILE[2]):
        g, spec = slab_geometry(geom, z0, z1)
        sims.append(lb.Simulation(g, params, layout="pointer_tile", scalar=np.float32, slab=spec))
        assert sims[-1].tile == (4, 4, 8)
    connect_local(sims, geom.periodic[2])
    for s in sims:
        s.initialize(1.004)
    single.step(7)
    for s in sims:
        s.step(7, block=False)    # slabs step together: a blocking step would wait on its neighbour
    for s in sims:
        s.synchronize()
    got = np.concatenate([s.canonical_state() for s in sims], axis=1)
    assert np.array_equal(got, single.canonical_state())
