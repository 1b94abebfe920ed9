"""CPU-side checks: the C-ABI library loads and exports every symbol the
header declares; the host copies of the per-node math are bitwise equal to
the oracle; host-side API semantics (parameters, layouts, geometry
builders) follow the reference."""

import os
import re

import numpy as np
import pytest

import paper_2108_13241_b200 as lb
from paper_2108_13241_b200 import _lib
from oracle import lattice19 as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "lbm19.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lbm\w*)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert {s for s, _, _ in _lib.SIGNATURES} == set(syms)
    assert lib.lbm_abi_version() == _lib.ABI_VERSION == 2


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors of lbm_desc / lbm_stats have the C layout
    (sizeof and every offsetof, from a gcc build against include/lbm19.h)."""
    import ctypes as C
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lines = []
    for cname, py in (("lbm_desc", _lib.LbmDesc), ("lbm_stats", _lib.LbmStats)):
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    src = ("#include <stdio.h>\n#include <stddef.h>\n#include \"lbm19.h\"\nint main(void){\n"
           + "\n".join(lines) + "\nreturn 0;}\n")
    (tmp_path / "layout.c").write_text(src)
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(tmp_path / "layout.c"), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {(a, b): int(c) for a, b, c in (l.split() for l in out if l)}
    for cname, py in (("lbm_desc", _lib.LbmDesc), ("lbm_stats", _lib.LbmStats)):
        assert got[(cname, "sizeof")] == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)


def test_scheme_argument_validation():
    from paper_2108_13241_b200.kernel import _desc
    d = _desc((8, 8, 8), (False,) * 3, np.float32, lb.LayoutKind.DENSE, (8, 8, 8), 0, 1.0, scheme="aa")
    assert d.scheme == 1
    with pytest.raises(ValueError):
        _desc((8, 8, 8), (False,) * 3, np.float32, lb.LayoutKind.DENSE, (8, 8, 8), 0, 1.0, scheme="abc")


def test_error_codes_without_device():
    lib = _lib.load()
    assert lib.lbm_create(None, None) == _lib.LBM_EINVAL
    assert "NULL" in _lib.last_error()


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_host_math_bitwise_equals_oracle(dt):
    rng = np.random.default_rng(11)
    ops = L.node_ops(dt)
    for _ in range(300):
        f = (rng.random(19) * 0.1 + 0.02).astype(dt)
        o = int(rng.integers(1, 7))
        u = (rng.random(3) * 0.1 - 0.05).astype(dt)
        a = f.copy()
        ops.zou_he_velocity19(a, o, u[0], u[1], u[2])
        b = lb.zou_he_velocity(f.astype(np.float64), o, u.astype(np.float64), dtype=dt).f
        assert np.array_equal(a.astype(np.float64), b)
        a = f.copy()
        ops.zou_he_pressure19(a, o, dt(1.01))
        b = lb.zou_he_pressure(f.astype(np.float64), o, float(dt(1.01)), dtype=dt).f
        assert np.array_equal(a.astype(np.float64), b)
        a = f.copy()
        m = [dt(v) for v in ops.moments19(a)]
        e = np.empty(19, dt)
        ops.collide19(a, *m, dt(1.3), e)
        assert np.array_equal(a.astype(np.float64),
                              lb.bgk_collide(f.astype(np.float64), float(dt(1.3)), dtype=dt))


def test_equilibrium_known_answers():
    e = lb.equilibrium(1.0, (0.1, 0.0, 0.0))
    for i, v in {0: 197 / 600, 1: 133 / 1800, 3: 73 / 1800, 2: 197 / 3600, 9: 197 / 3600,
                 5: 133 / 3600, 11: 133 / 3600, 6: 73 / 3600, 13: 73 / 3600}.items():
        assert e[i] == pytest.approx(v, rel=1e-15)
    assert sum(e) == pytest.approx(1.0, rel=1e-15)
    w = lb.equilibrium(1.0, (0, 0, 0), dtype=np.float32)
    assert np.array_equal(w, lb.W.astype(np.float32).astype(np.float64))
    with pytest.raises(ValueError):
        lb.equilibrium(1.0, (1.0, 0.0, 0.0))


def test_zou_he_reconstructs_equilibrium():
    """Known populations from an equilibrium give back that equilibrium
    (t/test_boundaries.py:53-61)."""
    for o in (lb.Orientation.WEST, lb.Orientation.EAST, lb.Orientation.NORTH,
              lb.Orientation.SOUTH, lb.Orientation.TOP, lb.Orientation.BOTTOM):
        feq = lb.equilibrium(1.02, (0.03, -0.01, 0.02))
        out = lb.zou_he_velocity(feq, o, (0.03, -0.01, 0.02))
        assert np.allclose(out.f, feq, rtol=0, atol=1e-15)
        assert out.rho == pytest.approx(1.02, rel=1e-14)


def test_flow_params_and_layout_parsing():
    p = lb.FlowParams.from_reynolds(U=0.1, L=63, Re=100)
    assert p.nu == pytest.approx(0.063)
    assert p.omega == pytest.approx(1 / (3 * 0.063 + 0.5))
    with pytest.raises(ValueError):
        lb.FlowParams(U=0.1, L=1, Re=1, nu=0.1, omega=1.0)
    assert lb.LayoutKind.parse("tile_sparse") is lb.LayoutKind.POINTER_TILE
    assert lb.LayoutKind.parse("Bitmask-Node") is lb.LayoutKind.BITMASK_NODE
    with pytest.raises(ValueError):
        lb.LayoutKind.parse("nope")


def test_geometry_builders():
    g = lb.build_cavity(16, 12, 10, 0.1)
    d = g.descriptors
    assert d.type_tag.shape == (10, 12, 16)
    assert d.count(lb.NodeType.VELOCITY_BC) == 16 * 10       # lid owns its edges
    assert g.porosity == 1.0
    c = lb.build_channel(32, 12, 8, lb.VelocityInlet((0.05, 0)))
    assert c.periodic == (False, False, True)
    assert c.descriptors.count(lb.NodeType.VELOCITY_BC) == 12 * 8
    assert c.descriptors.count(lb.NodeType.PRESSURE_BC) == 12 * 8
    p1 = lb.build_porous_random(40, 0.5, seed=4, radius_range=(3, 8))
    p2 = lb.build_porous_random(40, 0.5, seed=4, radius_range=(3, 8))
    assert p1.descriptors == p2.descriptors
    assert abs(p1.porosity - 0.5) <= 0.02 + 1e-12
    t = p1.descriptors.type_tag
    solid = t == lb.NodeType.SOLID
    # no FLUID node touches SOLID (26-neighbourhood)
    assert not np.any(lb.dilate26(solid) & (t == lb.NodeType.FLUID))
    v = lb.build_vascular(48, seed=1, fluid_fraction=0.05)
    assert 0.03 < v.porosity < 0.2
    vt = v.descriptors.type_tag
    assert not np.any(lb.dilate26(vt == lb.NodeType.SOLID) & (vt == lb.NodeType.FLUID))
    with pytest.raises(lb.GeometryError):
        lb.from_arrays("bad", np.full((4, 4, 4), 3, np.uint8))


def test_perf_report_arithmetic():
    r = lb.PerfReport.from_primaries("c", "dense", 4, 100, 100, 10, 1.0, 1e9)
    assert r.b_node_bytes == 152
    assert r.p_lups == 1000.0
    assert r.consistent()


def test_build_porous_regular_hits_porosity():
    """3-D analogue of the reference's regular array (geometry.py:315-370):
    bisection on the sphere radius reaches the target within 0.02; below 0.3
    is refused like the reference."""
    for phi in (0.3, 0.45, 0.6, 0.9, 1.0):
        g = lb.build_porous_regular(64, phi)
        assert abs(g.porosity - phi) <= 0.02 + 1e-12, (phi, g.porosity)
        t = g.descriptors.type_tag
        # walls win: no solid node on the domain faces, solids wrapped in walls
        assert not (t[:, :, 0] == lb.NodeType.SOLID).any()
    with pytest.raises(lb.GeometryError):
        lb.build_porous_regular(64, 0.2)
    with pytest.raises(lb.GeometryError):
        lb.build_porous_regular(32, 0.5)


def test_copy_bandwidth_argument_errors_without_device():
    with pytest.raises(ValueError):
        lb.copy_bandwidth_bench("dense", 1024)          # below 64 KiB (reference bound)
    with pytest.raises(ValueError):
        lb.copy_bandwidth_bench("dense", 1 << 20, repetitions=0)


@pytest.mark.parametrize("kw,msg", [
    (dict(layout="pointer_tile", tile=(3, 8, 8)), "powers of two"),
    (dict(layout="pointer_tile", tile=(2, 2, 2)), "32..512"),
    (dict(layout="tile", tile=(16, 16, 16)), "32..512"),
    (dict(scheme="bogus"), "scheme"),
])
def test_create_argument_validation_without_device(kw, msg):
    """lbm_create validates the descriptor before it touches a device, so the
    reference's ValueError contract (kernel.py:201-206, layouts.py:370-379)
    holds on any host."""
    from paper_2108_13241_b200.distributed import slab_geometry
    geom = lb.build_channel(16, 8, 8, lb.VelocityInlet((0.01, 0.0, 0.0)))
    params = lb.FlowParams.from_viscosity(U=0.01, L=7, nu=0.1)
    kw = dict(kw)
    if kw.pop("slab", False):
        geom, kw["slab"] = slab_geometry(geom, 0, 4)
    with pytest.raises(ValueError, match=msg):
        lb.Simulation(geom, params, scalar=np.float32, **kw)


def test_periodic_axis_must_divide_tile_without_device():
    types = np.full((8, 8, 12), lb.NodeType.FLUID, dtype=np.uint8)
    geom = lb.from_arrays("box", types, periodic=(True, False, False))
    params = lb.FlowParams.from_viscosity(U=0.01, L=7, nu=0.1)
    with pytest.raises(ValueError, match="periodic axis"):
        lb.Simulation(geom, params, layout="pointer_tile", tile=(8, 4, 4))
    with pytest.raises(ValueError, match="scalar"):
        lb.Simulation(geom, params, layout="dense", scalar=np.float16)


def test_kept_tile_fill_matches_brute_force():
    """The word-view fill count behind the default tile choice equals a
    plain reshape count of kept tiles, for 4 x {2,4} x {4,8} tiles."""
    rng = np.random.default_rng(5)
    for p in (0.02, 0.3, 0.9):
        t = (rng.random((16, 12, 20)) < p).astype(np.uint8) * rng.integers(1, 5, (16, 12, 20), dtype=np.uint8)
        live = t != lb.NodeType.SOLID
        for tile in ((4, 4, 8), (4, 4, 4), (4, 2, 4), (4, 4, 16)):
            ex, ey, ez = tile
            nz, ny, nx = t.shape
            got = lb.kept_tile_fill(t, tile)
            if nz % ez or ny % ey:
                assert got is None
                continue
            k = live.reshape(nz // ez, ez, ny // ey, ey, nx // ex, ex).any(axis=(1, 3, 5))
            assert got == pytest.approx(live.sum() / (k.sum() * ex * ey * ez), rel=1e-12)
    assert lb.kept_tile_fill(np.zeros((8, 4, 4), np.uint8)) is None           # no kept tile
    assert lb.kept_tile_fill(np.ones((8, 4, 6), np.uint8)) is None            # x not a multiple of 4


def test_default_tile_rule():
    """4x4x4 for the compacted tile list under AB when the kept 4x4x8 tiles are
    < 70 % non-solid; 4x4x8 otherwise (A-A, other layouts, dense media)."""
    sparse = lb.build_porous_random(64, 0.1, seed=0, radius_range=(3, 9)).descriptors.type_tag
    dense = lb.build_porous_random(64, 0.9, seed=0, radius_range=(3, 9)).descriptors.type_tag
    assert lb.kept_tile_fill(sparse) < 0.70 < lb.kept_tile_fill(dense)
    assert lb.default_tile(sparse, "pointer_tile") == (4, 4, 4)
    assert lb.default_tile(sparse, "pointer_tile", scheme="aa") == (4, 4, 8)
    assert lb.default_tile(sparse, "tile") == (4, 4, 8)
    assert lb.default_tile(dense, "pointer_tile") == (4, 4, 8)
