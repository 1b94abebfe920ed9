"""The reference's OWN Simulation (sparselbm, installed unmodified in
baseline/_ref) driven through the reference-side binding
(paper_2108_13241_b200/reference_binding.py), so that its step / run
observers / check_finite / macroscopic_fields / field.pre / total_mass /
benchmark calls run on liblbm19.  Checked against the golden outputs the
unpatched reference produced (tests/golden/*.npz, make_golden.py) at the
projection-bridge tolerances (f64 1e-12, f32 2e-6)."""

import os
import sys

import numpy as np
import pytest

from helpers import load_golden

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
CASES = ["mixed_s1", "mixed_s2", "mixed_s3", "cavity48_f64", "cavity48_f32", "chan_v",
         "chan_p", "porous64", "box_perturbed"]


@pytest.fixture(scope="module")
def slb():
    if not os.path.isdir(os.path.join(REF, "sparselbm")):
        pytest.skip("reference not installed in baseline/_ref (see DESIGN.md, reference install)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")
    sys.path.insert(0, REF)
    import sparselbm
    from paper_2108_13241_b200 import reference_binding
    reference_binding.install(sparselbm)
    yield sparselbm
    reference_binding.uninstall(sparselbm)


def _geometry(slb, g, name):
    table = slb.BoundaryValueTable()
    for k, v, r in zip(g["bc_kind"], g["bc_vel"], g["bc_rho"]):
        if int(k) == table.KIND_VELOCITY:
            table.add_velocity(float(v[0]), float(v[1]))
        else:
            table.add_pressure(float(r))
    return slb.from_arrays(name, g["types"], table, g["bc_index"], g["orient"])


def _params(slb, omega):
    nu = (1.0 / omega - 0.5) / 3.0
    U, L = 0.1, 10.0
    return slb.FlowParams(U=U, L=L, Re=U * L / nu, nu=nu, omega=slb.lattice.omega_from_viscosity(nu))


def _canonical(sim):
    n_x, n_y = sim.geometry.dims
    out = np.zeros((9, n_y, n_x), dtype=sim.dtype)
    slots = sim.field.slot_of
    ok = slots >= 0
    for i in range(9):
        out[i][ok] = sim.field.pre[i][slots[ok]]
    return out


@pytest.mark.parametrize("layout", ["dense", "pointer_tile"])
@pytest.mark.parametrize("name", CASES)
def test_reference_simulation_on_liblbm19(slb, name, layout):
    g = load_golden(name)
    dtype = np.dtype(str(g["dtype"]))
    tol = 1e-12 if dtype == np.float64 else 2e-6
    sim = slb.Simulation(_geometry(slb, g, name), _params(slb, float(g["omega"])),
                         layout=layout, scalar=dtype)
    rho0 = g["rho0"] if g["rho0"].ndim else float(g["rho0"])
    v0 = (g["v0x"], g["v0y"]) if g["rho0"].ndim else (float(g["v0x"]), float(g["v0y"]))
    sim.initialize(rho0=rho0, v0=v0)
    assert np.abs(_canonical(sim) - g["f_init"]).max() <= tol
    steps = int(g["steps"])
    seen = []

    def obs(step, fields, pre):
        assert not pre.flags.writeable and fields[0].shape == g["types"].shape
        seen.append((step, fields))

    every = max(1, steps // 4)
    sim.run(steps - 1, observers=[(every, obs)], check_divergence_every=every)
    sim.step()                      # the reference's single-step entry point
    assert sim.step_count == steps and sim.visited_nodes_total == steps * sim.visits_per_step
    assert [s for s, _ in seen] == list(range(every, steps, every))
    assert np.abs(_canonical(sim) - g["f_final"]).max() <= tol
    rho, vx, vy = sim.macroscopic_fields()
    assert np.abs(rho - g["rho"]).max() <= 10 * tol
    assert np.abs(vx - g["vx"]).max() <= 10 * tol
    assert np.abs(vy - g["vy"]).max() <= 10 * tol
    assert slb.total_mass(sim) == pytest.approx(float(g["mass_final"]),
                                                rel=1e-12 if dtype == np.float64 else 1e-6)
    sim.check_finite()
    assert sim._b200.launches_total >= steps   # the device did the stepping


def test_reference_benchmark_and_divergence(slb):
    g = load_golden("chan_v")
    sim = slb.Simulation(_geometry(slb, g, "chan_v"), _params(slb, float(g["omega"])),
                         layout="dense", scalar=np.float32)
    sim.initialize()
    rep = slb.benchmark(sim, warmup_steps=3, timed_steps=20)   # the reference's harness
    assert rep.steps == 20 and rep.p_lups > 0 and sim.step_count == 23
    # a non-finite value on the device surfaces as the reference's DivergenceError
    dev = sim._b200
    dev.field.write(7, 5, 0, 11, "pre", np.float32(np.nan))   # D3Q19 dir 11 -> D2Q9 dir 1
    with pytest.raises(slb.DivergenceError) as ei:
        sim.check_finite()
    assert ei.value.node == (7, 5) and ei.value.direction == 1
    with pytest.raises(RuntimeError):
        sim.field.write(1, 1, 0, "pre", 1.0)
