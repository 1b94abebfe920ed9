"""GPU parity of the A-A in-place scheme (one PDF buffer, alternating
neighbour / node-local steps): it must give the reference's results bit for
bit, so every check is `np.array_equal` against the CPU oracle (which follows
the reference's two-buffer pull kernel, pkg/kernel.py:72-141) or against the
AB scheme of the same library."""

import numpy as np
import pytest

import paper_2108_13241_b200 as lb
from helpers import oracle_sim, random_mixed_geometry3, to_geometry

pytestmark = pytest.mark.gpu

LAYOUTS = ["dense", "bitmask_node", "tile", "pointer_tile"]


def params_for(omega):
    nu = (1.0 / omega - 0.5) / 3.0
    return lb.FlowParams.from_viscosity(U=0.1, L=10, nu=nu)


def make(case, omega, dtype, layout="dense", tile=(8, 8, 8), scheme="aa"):
    return lb.Simulation(to_geometry(case, "case"), params_for(omega), layout=layout, scalar=dtype,
                         tile=tile, scheme=scheme)


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_aa_bitwise_vs_oracle(layout, dtype, seed):
    """Odd and even step counts (both AA state phases) decode to the oracle's
    pre buffer; all six face closures, solids, periodic z (seed 2)."""
    c = random_mixed_geometry3(seed, n=(19, 12, 10), periodic_z=(seed == 2))
    omega = 1.0 / (3 * 0.08 + 0.5)
    ref = oracle_sim(c, omega, dtype)
    ref.initialize(1.0)
    sim = make(c, omega, dtype, layout, tile=(8, 4, 2) if seed == 2 else (8, 8, 8))
    sim.initialize(1.0)
    assert np.array_equal(sim.canonical_state(), ref.pre)
    for chunk in (1, 4, 1, 20, 3):
        ref.step(chunk)
        sim.step(chunk)
        assert sim.stats().parity == sim.step_count % 2
        assert np.array_equal(sim.canonical_state(), ref.pre), (layout, chunk, sim.step_count)
        rho, ux, uy, uz = sim.macroscopic_fields()
        r2, a2, b2, c2 = ref.macroscopic_fields()
        for p, q in ((rho, r2), (ux, a2), (uy, b2), (uz, c2)):
            assert np.array_equal(p, q)


@pytest.mark.parametrize("layout", ["dense", "pointer_tile"])
def test_aa_equals_ab_with_graph_replay(layout):
    """Long runs go through the captured 32-step CUDA graph; odd totals end
    in phase 1.  Mass and the decoded field view agree bitwise with AB."""
    geom = lb.build_cavity(24, 24, 16, 0.1)
    params = lb.FlowParams.from_viscosity(U=0.1, L=23, nu=0.06)
    out = {}
    for scheme in ("ab", "aa"):
        sim = lb.Simulation(geom, params, layout=layout, scalar=np.float32, scheme=scheme)
        sim.initialize(1.0)
        sim.step(75)
        out[scheme] = (sim.canonical_state(), sim.total_mass(), sim.field.pre.copy(),
                       sim.stats().device_bytes)
    assert np.array_equal(out["aa"][0], out["ab"][0])
    assert out["aa"][1] == out["ab"][1]
    assert np.array_equal(out["aa"][2], out["ab"][2])
    assert out["aa"][3] < out["ab"][3]


def test_aa_half_the_pdf_memory():
    geom = lb.build_channel(64, 32, 32, lb.VelocityInlet((0.05, 0.0, 0.0)))
    params = lb.FlowParams.from_viscosity(U=0.05, L=31, nu=0.1)
    ab = lb.Simulation(geom, params, scalar=np.float32, scheme="ab")
    aa = lb.Simulation(geom, params, scalar=np.float32, scheme="aa")
    pdf = ab.stats().plane_stride * 19 * 4
    assert ab.stats().device_bytes - aa.stats().device_bytes == pdf
    assert aa.field.payload_bytes * 2 == ab.field.payload_bytes
    assert aa.stats().scheme == 1 and ab.stats().scheme == 0


@pytest.mark.parametrize("layout", ["dense", "pointer_tile"])
def test_aa_state_io_both_phases(layout):
    """set_state / field writes in either phase land where the next step
    reads them: poke the same value into AB and AA and compare."""
    c = random_mixed_geometry3(4, n=(16, 12, 8))
    omega = 1.3
    sims = {s: make(c, omega, np.float64, layout, scheme=s) for s in ("ab", "aa")}
    rng = np.random.default_rng(0)
    for s in sims.values():
        s.initialize(1.0)
    for steps in (1, 2):  # phase 1, then phase 1 again after 2 more (odd total 3)
        for s in sims.values():
            s.step(steps)
        state = sims["ab"].canonical_state()
        live = c["types"] != 0
        noise = rng.uniform(-1e-3, 1e-3, size=state.shape) * live
        for s in sims.values():
            s.set_state(state + noise)
        assert np.array_equal(sims["aa"].canonical_state(), sims["ab"].canonical_state())
        # field view poke: one population of one fluid node
        z, y, x = [int(v[0]) for v in np.nonzero(c["types"] == 1)]
        for s in sims.values():
            v = s.field.read(x, y, z, 5)
            s.field.write(x, y, z, 5, "pre", v + 0.25)
            s.step(1)
        assert np.array_equal(sims["aa"].canonical_state(), sims["ab"].canonical_state())


def test_aa_divergence_reported_in_odd_phase():
    c = random_mixed_geometry3(1, n=(16, 12, 8))
    sim = make(c, 1.2, np.float32)
    sim.initialize(1.0)
    sim.step(3)
    f = sim.canonical_state()
    z, y, x = [int(v[-1]) for v in np.nonzero(c["types"] == 1)]
    f[7, z, y, x] = np.nan
    sim.set_state(f)
    with pytest.raises(lb.DivergenceError) as ei:
        sim.check_finite()
    assert ei.value.node == (x, y, z) and ei.value.direction == 7


def test_aa_has_no_post_buffer():
    c = random_mixed_geometry3(1, n=(12, 10, 8))
    sim = make(c, 1.2, np.float32)
    sim.initialize(1.0)
    with pytest.raises(ValueError):
        sim.canonical_state("post")
    with pytest.raises(AttributeError):
        sim.field.post


def test_aa_solid_storage_never_touched():
    geom = lb.build_porous_random(32, 0.6, seed=9, radius_range=(3, 8))
    params = lb.FlowParams.from_viscosity(U=0.1, L=31, nu=0.3)
    solid = geom.descriptors.type_tag == lb.NodeType.SOLID
    for layout in LAYOUTS:
        sim = lb.Simulation(geom, params, layout=layout, scalar=np.float32, scheme="aa")
        sim.initialize(1.0)
        for n in (1, 4):
            sim.step(n)
            assert np.all(sim.canonical_state()[:, solid] == 0.0)


def test_aa_fully_periodic_box_vs_oracle():
    """Periodic x, y and z wrap through the neighbour step's push addresses;
    a solid block with its bounce-back ring sits inside."""
    nx, ny, nz = 16, 12, 8
    types = np.ones((nz, ny, nx), dtype=np.uint8)
    types[2:6, 3:9, 4:11] = 2
    types[3:5, 4:8, 5:10] = 0
    c = dict(types=types, orient=np.zeros_like(types), bc_index=np.full(types.shape, -1, np.int32),
             bc_kind=np.zeros(0, np.uint8), bc_vel=np.zeros((0, 3)), bc_rho=np.zeros(0),
             periodic=(True, True, True))
    rng = np.random.default_rng(3)
    rho0 = 1.0 + 0.01 * rng.standard_normal(types.shape)
    v0 = tuple(0.02 * rng.standard_normal(types.shape) for _ in range(3))
    ref = oracle_sim(c, 1.1, np.float64)
    ref.initialize(rho0, v0)
    sim = make(c, 1.1, np.float64, "dense")
    sim.initialize(rho0, v0)
    for chunk in (1, 6, 33):
        ref.step(chunk)
        sim.step(chunk)
        assert np.array_equal(sim.canonical_state(), ref.pre), chunk


@pytest.mark.parametrize("layout", ["tile", "pointer_tile"])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("variant", ["8", "7"])
def test_aa_tile_kernels_bitwise(monkeypatch, layout, dtype, variant):
    """Both A-A tile kernels (warp work list: 8, one CTA per tile: 7) give
    the oracle's state bit for bit in both phases."""
    monkeypatch.setenv("LBM_STEP_VARIANT", variant)
    c = random_mixed_geometry3(3, n=(24, 16, 16), periodic_z=True)
    omega = 1.0 / (3 * 0.07 + 0.5)
    ref = oracle_sim(c, omega, dtype)
    ref.initialize(1.0)
    sim = make(c, omega, dtype, layout)
    assert bool(sim.stats().tile_work_list) == (variant == "8")
    sim.initialize(1.0)
    for chunk in (1, 6, 5):
        ref.step(chunk)
        sim.step(chunk)
        assert np.array_equal(sim.canonical_state(), ref.pre), (layout, variant, sim.step_count)
