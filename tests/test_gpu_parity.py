"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle and
the reference's golden vectors.  Bar: bitwise for flag words, tile lists and
neighbour tables AND for f_i (the kernel uses explicitly rounded
operations in the oracle's expression order, see csrc/d3q19.cuh)."""

import numpy as np
import pytest

import paper_2108_13241_b200 as lb
from helpers import (GOLDEN_CASES, extruded_case, load_golden, oracle_sim, project,
                     random_mixed_geometry3, to_geometry)
from oracle import geometry19 as G

pytestmark = pytest.mark.gpu

LAYOUTS = ["dense", "bitmask_node", "tile", "pointer_tile"]


def params_for(omega):
    nu = (1.0 / omega - 0.5) / 3.0
    return lb.FlowParams.from_viscosity(U=0.1, L=10, nu=nu)


def make(case, omega, dtype, layout="dense", tile=(8, 8, 8), name="case"):
    geom = to_geometry(case, name)
    return lb.Simulation(geom, params_for(omega), layout=layout, scalar=dtype, tile=tile)


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("periodic_z", [False, True])
def test_flag_words_bit_exact(seed, periodic_z):
    c = random_mixed_geometry3(seed, n=(21, 13, 16), periodic_z=periodic_z)
    ref = G.flag_words(c["types"], c["orient"], c["bc_index"], c["periodic"])
    for layout in LAYOUTS:
        sim = make(c, 1.2, np.float32, layout, tile=(8, 4, 8) if periodic_z else (8, 8, 8))
        assert np.array_equal(sim.flag_words(), ref), layout
        assert sim.active_node_count == int(np.count_nonzero(c["types"]))


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_step_bitwise_vs_oracle(layout, dtype, seed):
    c = random_mixed_geometry3(seed, n=(19, 12, 10), periodic_z=(seed == 2))
    omega = 1.0 / (3 * 0.08 + 0.5)
    ref = oracle_sim(c, omega, dtype)
    ref.initialize(1.0)
    sim = make(c, omega, dtype, layout, tile=(8, 4, 2) if seed == 2 else (8, 8, 8))
    sim.initialize(1.0)
    assert np.array_equal(sim.canonical_state(), ref.pre)
    for chunk in (1, 4, 20):
        ref.step(chunk)
        sim.step(chunk)
        assert np.array_equal(sim.canonical_state(), ref.pre), (layout, chunk)
    rho, ux, uy, uz = sim.macroscopic_fields()
    r2, a2, b2, c2 = ref.macroscopic_fields()
    for p, q in ((rho, r2), (ux, a2), (uy, b2), (uz, c2)):
        assert np.array_equal(p, q)


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_projection_bridge_gpu_matches_reference(name):
    g = load_golden(name)
    c = extruded_case(g, 2)
    sim = make(c, c["omega"], c["dtype"])
    sim.initialize(c["rho0"], c["v0"])
    sim.step(c["steps"])
    tol = 1e-12 if c["dtype"] == np.float64 else 2e-6
    p = project(sim.canonical_state())
    assert np.abs(p[:, 0] - g["f_final"]).max() <= tol
    assert np.abs(p[:, 1] - g["f_final"]).max() <= tol
    rho, ux, uy, uz = sim.macroscopic_fields()
    assert np.abs(rho[0] - g["rho"]).max() <= 10 * tol
    assert np.all(uz == 0.0)
    assert sim.total_mass() == pytest.approx(2 * float(g["mass_final"]),
                                             rel=1e-12 if tol < 1e-9 else 1e-6)


def test_layouts_agree_bitwise_on_cavity():
    geom = lb.build_cavity(24, 24, 16, 0.1)
    params = lb.FlowParams.from_viscosity(U=0.1, L=23, nu=0.06)
    out = {}
    for layout in LAYOUTS:
        sim = lb.Simulation(geom, params, layout=layout, scalar=np.float32)
        sim.initialize(1.0)
        sim.step(50)
        out[layout] = sim.canonical_state()
    for layout in LAYOUTS[1:]:
        assert np.array_equal(out[layout], out["dense"])


def test_tile_index_bit_exact():
    geom = lb.build_porous_random(48, 0.5, seed=3, radius_range=(3, 10), dims=(48, 40, 32))
    d = geom.descriptors
    params = lb.FlowParams.from_viscosity(U=0.1, L=40, nu=0.3)
    for layout, keep_all in (("pointer_tile", False), ("tile", True)):
        for tile in ((8, 8, 8), (16, 4, 4), (32, 2, 2)):
            sim = lb.Simulation(geom, params, layout=layout, scalar=np.float32, tile=tile)
            tiles, nbr = sim.tile_index()
            rt, rn, _ = G.tile_index(d.type_tag, tile, d.periodic, keep_all=keep_all)
            assert np.array_equal(tiles, rt)
            assert np.array_equal(nbr, rn)
            assert sim.field.allocated_tiles == len(rt)


def test_tile_index_periodic_wrap():
    c = random_mixed_geometry3(5, n=(16, 16, 16), periodic_z=True)
    sim = make(c, 1.1, np.float32, "pointer_tile", tile=(8, 8, 4))
    tiles, nbr = sim.tile_index()
    rt, rn, _ = G.tile_index(c["types"], (8, 8, 4), c["periodic"])
    assert np.array_equal(tiles, rt) and np.array_equal(nbr, rn)


def test_solid_storage_never_touched():
    geom = lb.build_porous_random(32, 0.6, seed=9, radius_range=(3, 8))
    params = lb.FlowParams.from_viscosity(U=0.1, L=31, nu=0.3)
    solid = geom.descriptors.type_tag == lb.NodeType.SOLID
    for layout in LAYOUTS:
        sim = lb.Simulation(geom, params, layout=layout, scalar=np.float32)
        sim.initialize(1.0)
        sim.step(5)
        assert np.all(sim.canonical_state("pre")[:, solid] == 0.0)
        assert np.all(sim.canonical_state("post")[:, solid] == 0.0)


def test_rest_closed_box_is_bitwise_fixed_point():
    geom = lb.build_cavity(16, 16, 16, 0.1)
    geom.descriptors.type_tag[geom.descriptors.type_tag == lb.NodeType.VELOCITY_BC] = \
        lb.NodeType.BOUNCE_BACK_WALL
    geom.descriptors.bc_index[:] = -1
    geom.descriptors.orientation[:] = 0
    params = lb.FlowParams.from_viscosity(U=0.1, L=15, nu=0.1)
    for dt in (np.float32, np.float64):
        sim = lb.Simulation(geom, params, scalar=dt)
        sim.initialize(1.0)
        before = sim.canonical_state()
        sim.run(17)
        assert np.array_equal(sim.canonical_state(), before)


def test_initialize_imposes_boundary_values():
    geom = lb.build_channel(48, 16, 8, lb.PressureInlet(1.016))
    params = lb.FlowParams.from_viscosity(U=0.1, L=15, nu=0.25)
    sim = lb.Simulation(geom, params)
    sim.initialize(rho0=1.008)
    rho, vx, vy, vz = sim.macroscopic_fields()
    assert rho[3, 8, 24] == pytest.approx(1.008, rel=1e-12)
    assert rho[3, 8, 0] == pytest.approx(1.016, rel=1e-12)
    assert rho[3, 8, 47] == pytest.approx(1.0, rel=1e-12)
    with pytest.raises(ValueError):
        sim.initialize(rho0=np.ones((4, 4, 4)))


def test_divergence_detection_names_node_and_step():
    geom = lb.build_cavity(16, 16, 12, 0.1)
    params = lb.FlowParams.from_viscosity(U=0.1, L=15, nu=0.1)
    for layout in ("dense", "pointer_tile"):
        sim = lb.Simulation(geom, params, layout=layout)
        sim.initialize(1.0)
        sim.run(3)
        slot = int(sim.field.slot_of[5, 4, 7])
        sim.field.pre[2, slot] = np.nan
        with pytest.raises(lb.DivergenceError) as err:
            sim.check_finite()
        assert err.value.node == (7, 4, 5)
        assert err.value.direction == 2
        assert err.value.step == 3
        sim.initialize(1.0)
        sim.field.pre[2, slot] = np.inf
        with pytest.raises(lb.DivergenceError):
            sim.run(20, check_divergence_every=10)


def test_run_observers_and_counters():
    geom = lb.build_cavity(16, 16, 8, 0.1)
    params = lb.FlowParams.from_viscosity(U=0.1, L=15, nu=0.1)
    sim = lb.Simulation(geom, params)
    sim.initialize(1.0)
    calls = []

    def obs(step, fields, pre):
        calls.append(step)
        with pytest.raises(ValueError):
            pre[0, 0] = 1.0
        assert fields[0].shape == (8, 16, 16)

    sim.run(100, observers=[(10, obs)])
    assert calls == list(range(10, 101, 10))
    assert sim.step_count == 100
    assert sim.visited_nodes_total == 100 * 16 * 16 * 8
    with pytest.raises(RuntimeError, match="observer failed at step 102"):
        sim.run(5, observers=[(3, lambda *a: (_ for _ in ()).throw(KeyError("x")))])


def test_mass_conservation_closed_box_f64():
    rng = np.random.default_rng(8)
    geom = lb.build_cavity(24, 24, 24, 0.1)
    d = geom.descriptors
    d.type_tag[d.type_tag == lb.NodeType.VELOCITY_BC] = lb.NodeType.BOUNCE_BACK_WALL
    d.bc_index[:] = -1
    d.orientation[:] = 0
    params = lb.FlowParams.from_viscosity(U=0.1, L=23, nu=0.05)
    sim = lb.Simulation(geom, params)
    shape = d.type_tag.shape
    sim.initialize(1.0 + 0.02 * (rng.random(shape) - 0.5),
                   tuple(0.04 * (rng.random(shape) - 0.5) for _ in range(3)))
    m0 = sim.total_mass()
    sim.step(1000)
    assert abs(sim.total_mass() - m0) / m0 < 1e-11


def test_cavity_c1_f32_vs_f64_and_oracle():
    """Config C1 (64^3 cavity, Re 100) for 1000 steps: f32 bitwise equal to
    the f32 oracle; f32 within 1e-4 of f64 (t/test_kernel.py:248-255)."""
    geom = lb.build_cavity(64, 64, 64, 0.1)
    params = lb.FlowParams.from_reynolds(U=0.1, L=63, Re=100)
    d = geom.descriptors
    kinds, vel, rho = geom.boundary_values.as_arrays()
    c = dict(types=d.type_tag, orient=d.orientation, bc_index=d.bc_index, bc_kind=kinds,
             bc_vel=vel, bc_rho=rho, periodic=d.periodic)
    res = {}
    for dt in (np.float32, np.float64):
        sim = lb.Simulation(geom, params, scalar=dt)
        sim.initialize(1.0)
        sim.step(1000)
        res[dt] = sim.canonical_state().astype(np.float64)
    assert np.abs(res[np.float32] - res[np.float64]).max() < 1e-4
    ref = oracle_sim(c, params.omega, np.float32)
    ref.initialize(1.0)
    ref.step(1000)
    assert np.array_equal(res[np.float32], ref.pre.astype(np.float64))


def test_ghia_re100_physics():
    """Lid-driven cavity Re 100, 128^2 extruded one node with periodic z
    (2-D flow), 12000 steps: the reference's CLI thresholds MSE <= 5e-4 and
    max |err| <= 0.03 against Ghia 1982 (pkg/cli.py:54-55)."""
    n = 128
    g2 = lb.build_cavity(n, n, 8, 0.1)
    d = g2.descriptors
    # one z-plane, periodic span: a 2-D cavity in a 3-D kernel
    t = np.ascontiguousarray(d.type_tag[3:4])
    geom = lb.from_arrays("cavity", t, g2.boundary_values, d.bc_index[3:4], d.orientation[3:4],
                          params=g2.provenance.params, periodic=(False, False, True))
    params = lb.FlowParams.from_reynolds(U=0.1, L=n - 1, Re=100)
    sim = lb.Simulation(geom, params, scalar=np.float64)
    sim.initialize(1.0)
    sim.step(12000)
    prof = lb.centerline_profiles(sim, z=0)
    table = load_golden("ghia_re100")
    cmp = lb.compare_to_ghia(prof, table)
    assert cmp.mse <= 5e-4 and cmp.max_abs_err <= 0.03, cmp


def test_channel_poiseuille_profile():
    """Pressure-driven channel reaches a parabolic profile (reference CLI
    validate for chan, pkg/cli.py:312-321; 1 - R^2 <= 1e-3)."""
    geom = lb.build_channel(96, 24, 4, lb.PressureInlet(1.01))
    params = lb.FlowParams.from_viscosity(U=0.05, L=23, nu=0.25)
    sim = lb.Simulation(geom, params, scalar=np.float64)
    sim.initialize(rho0=1.005)
    sim.step(6000)
    rho, vx, vy, vz = sim.macroscopic_fields()
    fit = lb.poiseuille_fit(vx[2, :, 60])
    assert fit.residual <= 1e-3
    assert fit.v_max > 0


@pytest.mark.parametrize("layout,scheme", [("dense", "ab"), ("pointer_tile", "ab"), ("dense", "aa"),
                                           ("pointer_tile", "aa")])
def test_macroscopic_box_probe_matches_full_readback(layout, scheme):
    """Device-side probes (lines, planes, boxes) equal the slices of the full
    readback, in both AA phases."""
    c = random_mixed_geometry3(6, n=(21, 13, 11))
    sim = lb.Simulation(to_geometry(c), params_for(1.2), layout=layout, scalar=np.float64,
                        scheme=scheme)
    sim.initialize(1.0)
    for n in (3, 2):
        sim.step(n)
        full = sim.macroscopic_fields()
        for box, sl in (((5, None, 4), np.s_[4:5, :, 5:6]), ((None, 7, 10), np.s_[10:11, 7:8, :]),
                        (((2, 19), (1, 12), (3, 9)), np.s_[3:9, 1:12, 2:19])):
            got = sim.macroscopic_box(*box)
            for a, b in zip(got, full):
                assert np.array_equal(a, b[sl])
    with pytest.raises(ValueError):
        sim.macroscopic_box(x=(4, 40))


def _open_box(n):
    types = np.full((n, n, n), lb.NodeType.FLUID, dtype=np.uint8)
    return lb.from_arrays("open", types)


@pytest.mark.parametrize("v0", [(0.05, 0.0, 0.0), (0.03, -0.02, 0.01)])
def test_uniform_motion_interior_node_unchanged_by_one_step(v0):
    """3-D analogue of t/test_kernel.py:69-82: a uniform field advected onto
    itself; interior nodes see identical neighbours."""
    sim = lb.Simulation(_open_box(12), lb.FlowParams.from_viscosity(U=0.05, L=11, nu=0.1),
                        scalar=np.float64)
    sim.initialize(rho0=1.0, v0=v0)
    before = sim.canonical_state()
    sim.step()
    after = sim.canonical_state()
    np.testing.assert_allclose(after[:, 2:-2, 2:-2, 2:-2], before[:, 2:-2, 2:-2, 2:-2], rtol=0, atol=1e-15)


def test_single_perturbed_node_matches_plain_loop_step():
    """3-D analogue of t/test_kernel.py:85-103 against the plain-loop oracle
    (oracle/scalar19.py, the t/reference_lbm.py transcription)."""
    from oracle import scalar19 as S
    n = 5
    geom = _open_box(n)
    params = lb.FlowParams.from_viscosity(U=0.05, L=4, nu=0.2)
    rho0 = np.ones((n, n, n))
    rho0[2, 2, 2] = 1.1
    vx0 = np.zeros((n, n, n))
    vx0[2, 2, 2] = 0.03
    vz0 = np.zeros((n, n, n))
    vz0[2, 2, 2] = -0.02
    sim = lb.Simulation(geom, params, scalar=np.float64)
    sim.initialize(rho0=rho0, v0=(vx0, 0.0, vz0))
    d = geom.descriptors
    f = S.ref_initialize(d.type_tag, np.zeros((1, 3)), np.zeros(1), d.bc_index, rho0=1.0)
    f[:, 2, 2, 2] = S.ref_equilibrium(1.1, (0.03, 0.0, -0.02))
    for _ in range(2):
        sim.step()
        f = S.ref_step(f, d.type_tag, d.orientation, np.zeros((1, 3)), np.zeros(1), d.bc_index,
                       params.omega)
        np.testing.assert_allclose(sim.canonical_state(), f, rtol=0, atol=1e-15)


def test_launch_configuration_does_not_change_results(monkeypatch):
    """Analogue of t/test_kernel.py:143-156 (worker count): every tile kernel
    (warp work list, CTA per tile, TMA-staged), every tile shape, the AB and
    A-A schemes and the CUDA-graph replay reproduce the ORACLE bitwise."""
    from oracle.step19 import OracleSim
    geom = lb.build_porous_random(40, 0.45, seed=5, radius_range=(3, 7), dims=(40, 32, 24))
    params = lb.FlowParams.from_viscosity(U=0.05, L=31, nu=0.2)
    d = geom.descriptors
    kinds, vel, rho = geom.boundary_values.as_arrays()
    oracle = OracleSim(d.type_tag, d.orientation, d.bc_index, kinds, vel, rho, params.omega,
                       dtype=np.float32, periodic=d.periodic)
    oracle.initialize(1.005)
    oracle.step(37)

    def run(layout, tile=(8, 8, 8), scheme="ab", **env):
        for k in ("LBM_STEP_VARIANT", "LBM_GRAPH"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        sim = lb.Simulation(geom, params, layout=layout, scalar=np.float32, tile=tile, scheme=scheme)
        sim.initialize(1.005)
        sim.step(37)
        return sim.canonical_state()

    assert np.array_equal(run("dense", LBM_GRAPH="0"), oracle.pre)
    assert np.array_equal(run("dense"), oracle.pre)
    for scheme in ("ab", "aa"):
        for v in ("7", "8", "9"):   # CTA per tile, warp work list, TMA-staged tiles
            for tile in ((8, 8, 8), (4, 8, 16)):
                got = run("pointer_tile", tile=tile, scheme=scheme, LBM_STEP_VARIANT=v)
                assert np.array_equal(got, oracle.pre), (scheme, v, tile)
    for tile in ((16, 4, 8), (8, 4, 1), (32, 2, 4)):
        assert np.array_equal(run("pointer_tile", tile=tile), oracle.pre), tile
        assert np.array_equal(run("tile", tile=tile), oracle.pre), tile


def test_square_duct_profile_matches_analytic():
    """3-D physics at full path (config C5's geometry): velocity inlet on the
    BOTTOM face, pressure outlet on TOP, bounce-back duct walls.  Downstream
    the axial profile is the fully developed square-duct solution
    u ~ sum_{n odd} (-1)^((n-1)/2) / n^3 [1 - cosh(n pi y/a) / cosh(n pi/2)] cos(n pi x/a)
    with the halfway bounce-back wall half a spacing outside the wall nodes."""
    n, nz = 17, 72
    geom = lb.build_duct_z(n, n, nz, u_in=0.02)
    params = lb.FlowParams.from_viscosity(U=0.02, L=n, nu=0.1)
    sim = lb.Simulation(geom, params, scalar=np.float64)
    sim.initialize(1.0)
    sim.step(9000)
    _, _, _, uz = sim.macroscopic_box(z=48)
    a = float(n)
    xs = np.arange(n) + 0.5 - a / 2          # node centres, walls at +-a/2
    X, Y = np.meshgrid(xs, xs, indexing="xy")

    def analytic(x, y):
        s = np.zeros_like(x)
        for k in range(0, 40):
            m = 2 * k + 1
            s += (-1) ** k / m ** 3 * (1 - np.cosh(m * np.pi * y / a) / np.cosh(m * np.pi / 2)) * np.cos(m * np.pi * x / a)
        return s

    sim_p = uz[0]
    ana = analytic(X, Y)
    scale = float((sim_p * ana).sum() / (ana * ana).sum())
    err = np.abs(sim_p - scale * ana).max() / np.abs(sim_p).max()
    assert err < 0.03, err
    # mass flux through the section equals the inflow (incompressible, steady)
    assert abs(sim_p.sum() - 0.02 * n * n) / (0.02 * n * n) < 0.05


def test_porosity_sweep_reports(tmp_path):
    """Reference porosity_sweep (metrics.py:159-203) over the device path:
    a dense reference per layout plus one report per cell, eta_P filled,
    regular placements below 0.3 skipped; CSV with the documented columns."""
    cfg = lb.SweepConfig(n=64, warmup_steps=3, timed_steps=10, radius_range=(3, 8))
    reps = lb.porosity_sweep(["dense", "pointer_tile"], [0.2, 0.5], config=cfg)
    assert len(reps) == 2 * (1 + 1 + 2)
    for r in reps:
        assert r.p_lups > 0 and r.eta_p is not None and r.consistent()
    assert [r.placement for r in reps[:4]] == ["dense", "regular", "random", "random"]
    path = tmp_path / "sweep.csv"
    lb.write_report_csv(reps, path, config_hash="abc")
    lines = path.read_text().splitlines()
    assert lines[0] == "# config_hash abc" and len(lines) == 2 + len(reps)


def test_copy_bandwidth_survey_on_device():
    """Reference copy micro-benchmark (layouts.py:473-524) on the device:
    every layout pattern copies a verified block; dense is a real HBM rate."""
    res = lb.copy_bandwidth_survey(256 << 20, repetitions=5)
    assert set(res) == set(lb.LayoutKind)
    assert all(v > 1e11 for v in res.values())
    assert res[lb.LayoutKind.DENSE] > 2e12


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("scheme", ["ab", "aa"])
def test_all_solid_domain_is_a_no_op(layout, scheme):
    """Empty input: no non-solid node, no kept tile; stepping, readbacks,
    mass and the finite check still work and report zeros."""
    types = np.zeros((6, 9, 13), dtype=np.uint8)
    sim = lb.Simulation(lb.from_arrays("solid", types), params_for(1.1), layout=layout,
                        scalar=np.float32, scheme=scheme)
    sim.initialize(1.0)
    sim.step(5)
    assert sim.active_node_count == 0
    assert not sim.canonical_state().any()
    assert all(not a.any() for a in sim.macroscopic_fields())
    assert sim.total_mass() == 0.0
    sim.check_finite()


def test_boundary_table_limit_and_bad_descriptors():
    """At most 255 boundary-table entries fit the flag word (bc index bits
    24-31); out-of-range types / missing bc indices are rejected."""
    types = np.full((4, 8, 8), lb.NodeType.FLUID, dtype=np.uint8)
    big = lb.BoundaryValueTable()
    for k in range(256):
        big.add_velocity(0.001 * k, 0.0, 0.0)
    geom = lb.from_arrays("box", types, big)
    with pytest.raises(ValueError, match="255"):
        lb.Simulation(geom, params_for(1.1), scalar=np.float32)
    g2 = lb.from_arrays("box", types)
    g2.descriptors.type_tag[1, 2, 3] = 7          # corrupt after validation
    with pytest.raises(ValueError, match="out of range"):
        lb.Simulation(g2, params_for(1.1), scalar=np.float32)


@pytest.mark.parametrize("phi", [0.15, 0.5, 0.95, 1.0])
def test_default_tile_kernel_choice_is_bitwise(phi):
    """The tile kernel is picked from the live-brick fraction of the kept
    tiles (warp work list + select below 0.99, speculative CTA per tile for
    (almost) fully live tiles); every choice reproduces the oracle bitwise."""
    from oracle.step19 import OracleSim
    geom = lb.build_porous_random(64, phi, seed=2, radius_range=(3, 9), dims=(64, 48, 32))
    params = lb.FlowParams.from_viscosity(U=0.05, L=47, nu=0.2)
    sim = lb.Simulation(geom, params, layout="pointer_tile", scalar=np.float32)   # the default tile
    assert sim.tile == lb.default_tile(geom.descriptors.type_tag, "pointer_tile")
    assert sim.tile == ((4, 4, 4) if phi <= 0.5 else (4, 4, 8))
    # live-brick fraction of the kept tiles (2x2x2 bricks), as the library computes it
    ex, ey, ez = sim.tile
    ns = geom.descriptors.type_tag != lb.NodeType.SOLID
    nz, ny, nx = ns.shape
    b = ns.reshape(nz // 2, 2, ny // 2, 2, nx // 2, 2).any(axis=(1, 3, 5))
    bx, by, bz = ex // 2, ey // 2, ez // 2
    bt = b.reshape(nz // ez, bz, ny // ey, by, nx // ex, bx).sum(axis=(1, 3, 5))
    kept = bt > 0
    live_frac = bt[kept].sum() / (kept.sum() * bx * by * bz)
    assert bool(sim.stats().tile_work_list) == (live_frac < 0.99)
    sim.initialize(1.004)
    sim.step(9)
    d = geom.descriptors
    kinds, vel, rho = geom.boundary_values.as_arrays()
    ref = OracleSim(d.type_tag, d.orientation, d.bc_index, kinds, vel, rho, params.omega,
                    dtype=np.float32, periodic=d.periodic)
    ref.initialize(1.004)
    ref.step(9)
    assert np.array_equal(sim.canonical_state(), ref.pre)
