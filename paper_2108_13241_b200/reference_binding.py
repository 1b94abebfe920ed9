"""Reference-side binding: run the reference's own `sparselbm.Simulation`
(the 2-D D2Q9 API, pkg/src/sparselbm/kernel.py:155-311) on liblbm19.

    import sparselbm
    from paper_2108_13241_b200 import reference_binding
    reference_binding.install(sparselbm)     # every Simulation now steps on the GPU
    ...
    reference_binding.uninstall(sparselbm)

This is the executable form of the stub in INTEGRATION.md: what a maintainer
adds to the reference to make its time-stepping path call the C-ABI.  The
reference's constructor still runs (its layouts, slot maps, visit lists and
counters stay valid); install() replaces the methods on the stepping path:

  initialize(rho0, v0)      kernel.py:190-237 -> lbm_init_equilibrium on the
                            device (the reference's host initialisation runs
                            too, so its argument checks and counters hold)
  step()                    kernel.py:239-252 -> lbm_step(h, 1)
  run(n, observers, ...)    kernel.py:254-276 -> lbm_step(h, k) between
                            observer / divergence events
  check_finite()            kernel.py:278-283 -> lbm_check_finite
  macroscopic_fields()      kernel.py:285-311 -> lbm_get_macroscopic
  field.pre / field.post    layouts.py:300-306 -> lbm_get_pdf, on access

The D3Q19 kernel runs the 2-D geometry extruded to n_z = 1 with a periodic
z axis; every 2-D quantity is the projection of the 3-D state (SURVEY.md
A.5): f9_k = sum of f19_j over the D3Q19 directions j with the (c_x, c_y)
of k, rho and (u_x, u_y) as computed from f19, u_z = 0.  On such a geometry
the projection evolves as the reference's D2Q9 state; tests/
test_gpu_reference_binding.py drives the reference's Simulation through
this binding against the reference's own golden outputs (f64 <= 1e-12,
f32 <= 2e-6).  Pointer- and full-tile layouts use (16, 16, 1) tiles, the
reference's 16 x 16 tiles (layouts.py:34).

`field.pre` / `field.post` are read-only host mirrors refreshed after every
device step: writing them raises (the reference's test pokes of pre have no
unique D3Q19 lift).  There is no CPU fallback: install() loads liblbm19 and
raises if it is missing.
"""

import numpy as np

from . import _lib
from .geometry import from_arrays
from .layouts import BoundaryValueTable
from .kernel import DivergenceError as _DivergenceError3
from .kernel import Simulation as _Sim3

# D2Q9 direction k <- D3Q19 directions with the same (c_x, c_y)
PROJECTION = ((0, 9, 10), (1, 11, 14), (2, 15, 18), (3, 12, 13), (4, 16, 17),
              (5,), (6,), (7,), (8,))
D19_TO_D9 = np.empty(19, dtype=np.int64)
for _k, _js in enumerate(PROJECTION):
    D19_TO_D9[list(_js)] = _k

_PATCHED = ("initialize", "step", "run", "check_finite", "macroscopic_fields")
_saved = {}


def project(f19):
    """(19, 1, n_y, n_x) -> (9, n_y, n_x): each D2Q9 population is the sum
    of the (at most three) D3Q19 populations with its (c_x, c_y)."""
    f = np.asarray(f19)[:, 0]
    return np.stack([f[js[0]] if len(js) == 1 else
                     (f[js[0]] + f[js[1]] + f[js[2]]) for js in PROJECTION])


def _layout_name(layout):
    return getattr(layout, "value", str(layout))


def _device_sim(ref_sim):
    """The liblbm19 handle for a reference Simulation (created on first use)."""
    dev = getattr(ref_sim, "_b200", None)
    if dev is not None:
        return dev
    slb = _saved["module"]
    desc = ref_sim.geometry.descriptors
    n_x, n_y = desc.dims
    ext = lambda a: np.ascontiguousarray(np.asarray(a)[None])
    table = BoundaryValueTable()
    kinds, vel, rho = ref_sim.geometry.boundary_values.as_arrays(np.float64)
    for k, v, r in zip(kinds, vel, rho):
        if int(k) == slb.BoundaryValueTable.KIND_VELOCITY:
            table.add_velocity(float(v[0]), float(v[1]), 0.0)
        else:
            table.add_pressure(float(r))
    case = getattr(getattr(ref_sim.geometry, "provenance", None), "case", "reference")
    geom3 = from_arrays(f"{case}-z1", ext(desc.type_tag), table,
                        ext(desc.bc_index), ext(desc.orientation), periodic=(False, False, True))
    layout = _layout_name(ref_sim.layout)
    tile = (16, 16, 1)
    dev = _Sim3(geom3, ref_sim.params, layout=layout, scalar=ref_sim.dtype, tile=tile)
    ref_sim._b200 = dev
    return dev


class _MirrorField:
    """Stands in for the reference's PdfField on a bound Simulation: the
    same attributes, with pre / post downloaded (projected) from the device
    after each step and handed out read-only."""

    def __init__(self, ref_sim, field):
        self.__dict__["_sim"] = ref_sim
        self.__dict__["_field"] = field
        self.__dict__["_stale"] = True

    def __getattr__(self, name):
        return getattr(self._field, name)

    def __setattr__(self, name, value):
        setattr(self._field, name, value)

    def _refresh(self):
        if not self._stale:
            return
        f = self._field
        dev = self._sim._b200
        ok = f.slot_of >= 0
        for which in (0, 1):
            if which == 1 and not dev.initialized:
                break
            f19 = dev.canonical_state("pre" if which == 0 else "post")
            p = project(f19).astype(f.dtype)
            f._buffers.setflags(write=True)
            buf = f._buffers[f.parity if which == 0 else 1 - f.parity]
            buf[:] = 0
            for k in range(9):
                buf[k, f.slot_of[ok]] = p[k][ok]
            f._buffers.setflags(write=False)
        self.__dict__["_stale"] = False

    @property
    def pre(self):
        self._refresh()
        return self._field.pre

    @property
    def post(self):
        self._refresh()
        return self._field.post

    def read(self, x, y, i, which="pre"):
        self._refresh()
        return self._field.read(x, y, i, which)

    def write(self, x, y, i, which, value):
        raise RuntimeError("a liblbm19-bound Simulation's PDF buffers live on the device; "
                           "host writes have no unique D3Q19 lift (use initialize(rho0, v0))")

    def swap_buffers(self):
        self._field.swap_buffers()
        self.__dict__["_stale"] = True


def _mirror(ref_sim):
    if not isinstance(ref_sim.field, _MirrorField):
        ref_sim.field = _MirrorField(ref_sim, ref_sim.field)
    return ref_sim.field


def _initialize(self, rho0=1.0, v0=(0.0, 0.0)):
    if isinstance(self.field, _MirrorField):
        self.field = self.field._field         # the reference's own PdfField again
    self.field._buffers.setflags(write=True)
    _saved["initialize"](self, rho0, v0)       # host-side checks, counters, slot maps
    dev = _device_sim(self)
    n_x, n_y = self.geometry.descriptors.dims
    lift = lambda a: np.asarray(a, dtype=np.float64) if np.ndim(a) == 0 else \
        np.broadcast_to(np.asarray(a, dtype=np.float64), (n_y, n_x))[None]
    dev.initialize(lift(rho0), (lift(v0[0]), lift(v0[1]), 0.0))
    m = _mirror(self)
    m.__dict__["_stale"] = True


def _step(self):
    if not self.initialized:
        raise RuntimeError("initialize() must run before stepping")
    self._b200.step(1)
    m = _mirror(self)
    m.swap_buffers()
    self.step_count += 1
    self.visited_nodes_total += self.visits_per_step


def _advance(self, n):
    if n <= 0:
        return
    self._b200.step(int(n))
    m = _mirror(self)
    for _ in range(int(n) & 1):
        m._field.swap_buffers()
    m.__dict__["_stale"] = True
    self.step_count += int(n)
    self.visited_nodes_total += int(n) * self.visits_per_step


def _run(self, n_steps, observers=(), check_divergence_every=None):
    if n_steps < 0:
        raise ValueError(f"n_steps must be >= 0, got {n_steps}")
    if n_steps > 0 and not self.initialized:
        raise RuntimeError("initialize() must run before stepping")
    stops = [int(k) for k, _ in observers]
    if check_divergence_every:
        stops.append(int(check_divergence_every))
    done = 0
    while done < n_steps:
        chunk = n_steps - done
        for k in stops:
            chunk = min(chunk, (self.step_count // k + 1) * k - self.step_count)
        _advance(self, chunk)
        done += chunk
        fields = None
        for every_k, callback in observers:
            if self.step_count % every_k == 0:
                if fields is None:
                    fields = self.macroscopic_fields()
                    view = self.field.pre.view()
                    view.setflags(write=False)
                try:
                    callback(self.step_count, fields, view)
                except Exception as exc:
                    raise RuntimeError(f"observer failed at step {self.step_count}") from exc
        if check_divergence_every and self.step_count % check_divergence_every == 0:
            self.check_finite()


def _check_finite(self):
    slb = _saved["module"]
    try:
        self._b200.check_finite()
    except _DivergenceError3 as exc:
        x, y, _ = exc.node
        raise slb.DivergenceError(self.step_count, (int(x), int(y)),
                                  int(D19_TO_D9[int(exc.direction)])) from exc


def _macroscopic_fields(self):
    rho, ux, uy, _ = self._b200.macroscopic_fields()
    return rho[0], ux[0], uy[0]


def install(slb):
    """Route the reference's Simulation stepping path through liblbm19."""
    if _saved:
        return
    _lib.load()   # loud failure if the CUDA library is missing
    cls = slb.kernel.Simulation
    _saved["module"] = slb
    for name in _PATCHED:
        _saved[name] = getattr(cls, name)
    cls.initialize = _initialize
    cls.step = _step
    cls.run = _run
    cls.check_finite = _check_finite
    cls.macroscopic_fields = _macroscopic_fields


def uninstall(slb):
    if not _saved:
        return
    cls = slb.kernel.Simulation
    for name in _PATCHED:
        setattr(cls, name, _saved[name])
    _saved.clear()
