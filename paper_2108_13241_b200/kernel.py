"""`Simulation`: the reference's solver API (pkg/src/sparselbm/kernel.py:155-311)
over the B200 C-ABI library.

Geometry, PDF buffers, flag words and the tile index live on the device; the
step loop runs there with no host round trip (`step(n)` is one library call).
Host-side state is limited to the geometry object and lazily downloaded
mirrors of the PDF buffers (`sim.field.pre` / `.post`), which are written
back before the next device operation so tests may poke them the way the
reference's tests do (t/test_kernel.py:203-209).
"""

import ctypes as C

import numpy as np

from . import _lib
from .lattice import Q
from .layouts import DEFAULT_TILE, LayoutKind, NodeType, default_tile

_SOLID = int(NodeType.SOLID)


class DivergenceError(RuntimeError):
    """A non-finite distribution value appeared during stepping
    (reference kernel.py:35-44)."""

    def __init__(self, step, node, direction):
        self.step = step
        self.node = node
        self.direction = direction
        super().__init__(f"non-finite distribution at node {node}, direction {direction}, "
                         f"after step {step}")


_worker_cap = None


def set_worker_count(n):
    """Kept for API compatibility (reference kernel.py:47-53): the device
    kernel's results never depend on launch configuration."""
    global _worker_cap
    _worker_cap = int(n)


def max_worker_count():
    return 1 if _worker_cap is None else _worker_cap


def _desc(dims, periodic, dtype, layout, tile, device, omega, nz_global=None, z0=0, scheme="ab"):
    nx, ny, nz = dims
    d = _lib.LbmDesc()
    d.nx, d.ny, d.nz = int(nx), int(ny), int(nz)
    d.nz_global = int(nz_global if nz_global is not None else nz)
    d.z0 = int(z0)
    for a in range(3):
        d.periodic[a] = int(bool(periodic[a]))
        d.tile[a] = int(tile[a])
    d.dtype = _lib.LBM_F32 if np.dtype(dtype) == np.float32 else _lib.LBM_F64
    d.layout = _lib.LAYOUT_CODES[layout.value]
    d.device = int(device)
    d.omega = float(omega)
    if scheme not in _lib.SCHEME_CODES:
        raise ValueError(f"scheme must be one of {sorted(_lib.SCHEME_CODES)}, got {scheme!r}")
    d.scheme = _lib.SCHEME_CODES[scheme]
    return d


class _Handle:
    """Owns one lbm_t*; destroyed with the Python object."""

    def __init__(self, desc):
        self.lib = _lib.load()
        self.h = C.c_void_p()
        _lib.check(self.lib.lbm_create(C.byref(desc), C.byref(self.h)), "lbm_create")

    def close(self):
        if self.h:
            self.lib.lbm_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stats(self):
        s = _lib.LbmStats()
        _lib.check(self.lib.lbm_get_stats(self.h, C.byref(s)))
        return s


def _upload_geometry(handle, desc_field, table, ghost_lo=None, ghost_hi=None, zslice=None):
    types = desc_field.type_tag
    orient = desc_field.orientation
    bc = desc_field.bc_index
    if zslice is not None:
        types, orient, bc = types[zslice], orient[zslice], bc[zslice]
    types = np.ascontiguousarray(types)
    orient = np.ascontiguousarray(orient)
    bc = np.ascontiguousarray(bc)
    kinds, vel, rho = table.as_arrays(np.float64)
    kinds = np.ascontiguousarray(kinds)
    vel = np.ascontiguousarray(vel)
    rho = np.ascontiguousarray(rho)
    glo = None if ghost_lo is None else np.ascontiguousarray(ghost_lo, dtype=np.uint8)
    ghi = None if ghost_hi is None else np.ascontiguousarray(ghost_hi, dtype=np.uint8)
    _lib.check(handle.lib.lbm_set_geometry(
        handle.h, _lib.ptr(types), _lib.ptr(orient), _lib.ptr(bc), _lib.ptr(glo),
        _lib.ptr(ghi), _lib.ptr(kinds), _lib.ptr(vel), _lib.ptr(rho), len(table)),
        "lbm_set_geometry")


def device_flag_words(desc_field, device=0):
    """Packed flag words of a NodeDescriptorField, computed by the device's
    mask kernel (reference layouts.py:173-188)."""
    from .layouts import BoundaryValueTable
    nx, ny, nz = desc_field.dims
    h = _Handle(_desc((nx, ny, nz), desc_field.periodic, np.float32, LayoutKind.DENSE,
                      (8, 8, 8), device, 1.0))
    try:
        # the table content is irrelevant for masks; size it to cover bc_index
        nb = int(desc_field.bc_index.max()) + 1 if desc_field.bc_index.size else 0
        table = BoundaryValueTable()
        for _ in range(max(nb, 0)):
            table.add_velocity(0.0, 0.0, 0.0)
        _upload_geometry(h, desc_field, table)
        out = np.empty((nz, ny, nx), dtype=np.uint32)
        _lib.check(h.lib.lbm_get_flags(h.h, _lib.ptr(out)))
        return out
    finally:
        h.close()


class DeviceField:
    """Host view of the device PDF storage (reference PdfField,
    layouts.py:272-360).  `pre` / `post` download the native (19,
    plane_stride) buffers on access; edits are written back before the next
    device operation."""

    def __init__(self, sim):
        self._sim = sim
        self._mirror = {}
        self._touched = False   # a writable mirror was handed out (pre/post/write)
        self._slot_of = None
        self.frozen = False

    @property
    def dims(self):
        return self._sim.geometry.dims

    @property
    def layout(self):
        return self._sim.layout

    @property
    def dtype(self):
        return self._sim.dtype

    @property
    def parity(self):
        return int(self._sim._handle.stats().parity)

    @property
    def plane_stride(self):
        return int(self._sim._handle.stats().plane_stride)

    @property
    def n_slots(self):
        return int(self._sim._handle.stats().n_slots)

    @property
    def payload_bytes(self):
        """All buffers (two for AB, one for AA), 19 planes, one slot per
        allocated node."""
        nbuf = 1 if self._sim.scheme == "aa" else 2
        return self.n_slots * Q * nbuf * self.dtype.itemsize

    @property
    def allocated_tiles(self):
        return int(self._sim._handle.stats().n_tiles)

    def _tiled(self):
        return self.layout in (LayoutKind.TILE, LayoutKind.POINTER_TILE)

    def _get(self, which):
        """(19, n_slots) host view of buffer `which`.  Tile layouts are stored
        AoSoA (tile, direction, node) on the device; the view is transposed
        to the reference's (direction, slot) indexing and written back by
        flush()."""
        if which not in self._mirror:
            raw = np.empty(Q * self.plane_stride, dtype=self.dtype)
            _lib.check(self._sim._handle.lib.lbm_get_field(self._sim._handle.h, which,
                                                           _lib.ptr(raw)))
            if self._tiled():
                tn = int(np.prod(self._sim.tile))
                T = self.plane_stride // tn
                view = np.ascontiguousarray(raw.reshape(T, Q, tn).transpose(1, 0, 2)).reshape(Q, T * tn)
            else:
                view = raw.reshape(Q, self.plane_stride)
            self._mirror[which] = view
        return self._mirror[which]

    @property
    def pre(self):
        self._touched = True
        return self._get(0)

    @property
    def post(self):
        if self._sim.scheme == "aa":
            raise AttributeError("the AA scheme updates one buffer in place: there is no post buffer")
        self._touched = True
        return self._get(1)

    @property
    def slot_of(self):
        if self._slot_of is None:
            nx, ny, nz = self.dims
            out = np.empty((nz, ny, nx), dtype=np.int32)
            _lib.check(self._sim._handle.lib.lbm_get_slot_of(self._sim._handle.h, _lib.ptr(out)))
            self._slot_of = out
        return self._slot_of

    def flush(self):
        """Write mirrored host edits back to the device and drop the mirrors.
        Mirrors only downloaded for a read-only view (run() observers) are
        dropped without an upload."""
        if not self._touched:
            self._mirror = {}
        if not self._mirror:
            return
        h = self._sim._handle
        for which, view in self._mirror.items():
            if self._tiled():
                tn = int(np.prod(self._sim.tile))
                T = view.shape[1] // tn
                raw = np.ascontiguousarray(view.reshape(Q, T, tn).transpose(1, 0, 2))
            else:
                raw = np.ascontiguousarray(view)
            _lib.check(h.lib.lbm_set_field(h.h, which, _lib.ptr(raw)))
        self._mirror = {}
        self._touched = False

    def invalidate(self):
        self._mirror = {}
        self._touched = False

    def _slot_checked(self, x, y, z, i):
        nx, ny, nz = self.dims
        if not (0 <= x < nx and 0 <= y < ny and 0 <= z < nz):
            raise ValueError(f"node ({x}, {y}, {z}) outside domain {nx}x{ny}x{nz}")
        if not 0 <= i < Q:
            raise ValueError(f"direction index out of range: {i}")
        return int(self.slot_of[z, y, x])

    def read(self, x, y, z, i, which="pre"):
        s = self._slot_checked(x, y, z, i)
        if s < 0:
            return self.dtype.type(0.0)
        if which != "pre" and self._sim.scheme == "aa":
            raise AttributeError("the AA scheme updates one buffer in place: there is no post buffer")
        return self._get(0 if which == "pre" else 1)[i, s]  # read: no upload needed

    def write(self, x, y, z, i, which, value):
        s = self._slot_checked(x, y, z, i)
        if s < 0:
            raise RuntimeError(f"write to unallocated storage at ({x}, {y}, {z})")
        (self.pre if which == "pre" else self.post)[i, s] = value


class Simulation:
    """Geometry + device PDF storage + flow parameters, ready to step
    (reference kernel.py:155-311)."""

    def __init__(self, geometry, params, layout=LayoutKind.DENSE, scalar=np.float64,
                 device=0, tile=None, slab=None, scheme="ab"):
        self.geometry = geometry
        self.params = params
        self.layout = LayoutKind.parse(layout)
        self.dtype = np.dtype(scalar)
        if self.dtype not in (np.dtype(np.float32), np.dtype(np.float64)):
            raise ValueError(f"scalar must be float32 or float64, got {scalar}")
        self.device = int(device)
        # "ab": two buffers swapped every step (the reference's PdfField);
        # "aa": one buffer updated in place (half the memory, same results)
        self.scheme = str(scheme).lower()
        desc = geometry.descriptors
        if tile is None:
            # z-slabs cut on tile planes: every rank keeps the fixed default
            tile = DEFAULT_TILE if slab is not None else default_tile(desc.type_tag, self.layout, self.scheme)
        self.tile = tuple(int(t) for t in tile)
        self.slab = slab
        nzg, z0, glo, ghi = (None, 0, None, None) if slab is None else \
            (slab.nz_global, slab.z0, slab.ghost_lo, slab.ghost_hi)
        self._handle = _Handle(_desc(desc.dims, desc.periodic, self.dtype, self.layout,
                                     self.tile, self.device, params.omega, nz_global=nzg, z0=z0,
                                     scheme=self.scheme))
        _upload_geometry(self._handle, desc, geometry.boundary_values, ghost_lo=glo, ghost_hi=ghi)
        self.field = DeviceField(self)
        self.initialized = False

    # -- counters (reference kernel.py:180-188) ---------------------------
    @property
    def visits_per_step(self):
        return int(self._handle.stats().visits_per_step)

    @property
    def active_node_count(self):
        return int(self._handle.stats().n_nonsolid)

    @property
    def step_count(self):
        return int(self._handle.stats().step_count)

    @property
    def visited_nodes_total(self):
        return int(self._handle.stats().visited_nodes_total)

    @property
    def last_step_ms(self):
        """Device time of the last step(n) call (CUDA events on the solver stream)."""
        return float(self._handle.stats().last_step_ms)

    @property
    def launches_total(self):
        return int(self._handle.stats().launches_total)

    def stats(self):
        return self._handle.stats()

    def close(self):
        self._handle.close()

    # -- initialisation ---------------------------------------------------
    def initialize(self, rho0=1.0, v0=(0.0, 0.0, 0.0)):
        """Every non-solid node's pre buffer = equilibrium(rho0, v0) in float64,
        cast to the storage type; velocity nodes start at their imposed
        velocity, pressure nodes at their imposed density; post is zeroed
        (reference kernel.py:190-237)."""
        nx, ny, nz = self.geometry.dims
        shape = (nz, ny, nx)
        v0 = tuple(v0) + (0.0,) * (3 - len(v0))

        def field(v):
            a = np.asarray(v, dtype=np.float64)
            if a.ndim == 0:
                return None, float(a)
            return np.ascontiguousarray(np.broadcast_to(a, shape)), 0.0

        (r, r0), (a, a0), (b, b0), (c, c0) = (field(rho0), field(v0[0]), field(v0[1]),
                                              field(v0[2]))
        self.field.invalidate()
        h = self._handle
        _lib.check(h.lib.lbm_init_equilibrium(h.h, _lib.ptr(r), _lib.ptr(a), _lib.ptr(b),
                                              _lib.ptr(c), r0, a0, b0, c0), "initialize")
        self.initialized = True
        self.field.frozen = True

    # -- stepping ---------------------------------------------------------
    def step(self, n=1, block=True):
        """Advance n time steps on the device (reference kernel.py:239-252,
        n = 1).  Returns after the device finished unless block=False (then
        call synchronize(); used to drive several slabs from one thread)."""
        if not self.initialized:
            raise RuntimeError("initialize() must run before stepping")
        self.field.flush()
        h = self._handle
        if block:
            _lib.check(h.lib.lbm_step(h.h, int(n)), "step")
        else:
            _lib.check(h.lib.lbm_step_async(h.h, int(n)), "step")

    def synchronize(self):
        _lib.check(self._handle.lib.lbm_synchronize(self._handle.h), "synchronize")

    def run(self, n_steps, observers=(), check_divergence_every=None):
        """Advance n_steps, firing each (every_k, callback) observer at steps
        divisible by k with (step index, macroscopic fields, pre buffer)
        (reference kernel.py:254-276).  Steps between observer / divergence
        events run as one device call."""
        if n_steps < 0:
            raise ValueError(f"n_steps must be >= 0, got {n_steps}")
        if not self.initialized and n_steps > 0:
            raise RuntimeError("initialize() must run before stepping")
        stops = [int(k) for k, _ in observers]
        if check_divergence_every:
            stops.append(int(check_divergence_every))
        done = 0
        while done < n_steps:
            cur = self.step_count
            chunk = n_steps - done
            for k in stops:
                nxt = (cur // k + 1) * k - cur
                chunk = min(chunk, nxt)
            self.step(chunk)
            done += chunk
            sc = self.step_count
            fields = None
            for every_k, callback in observers:
                if sc % every_k == 0:
                    if fields is None:
                        fields = self.macroscopic_fields()
                        view = self.field._get(0).view()  # read-only: no upload after
                        view.setflags(write=False)
                    try:
                        callback(sc, fields, view)
                    except Exception as exc:
                        raise RuntimeError(f"observer failed at step {sc}") from exc
            if check_divergence_every and sc % check_divergence_every == 0:
                self.check_finite()

    def check_finite(self):
        """Raise DivergenceError if the pre buffer holds a non-finite value
        (reference kernel.py:278-283)."""
        self.field.flush()
        h = self._handle
        d = C.c_int32(-1)
        node = (C.c_int32 * 3)()
        rc = h.lib.lbm_check_finite(h.h, C.byref(d), node)
        if rc == _lib.LBM_EDIVERGED:
            raise DivergenceError(self.step_count, (int(node[0]), int(node[1]), int(node[2])),
                                  int(d.value))
        _lib.check(rc, "check_finite")

    # -- readback ---------------------------------------------------------
    def macroscopic_fields(self):
        """Per-node (rho, v_x, v_y, v_z), float64 (n_z, n_y, n_x); solid nodes
        report 0 (reference kernel.py:285-311)."""
        self.field.flush()
        nx, ny, nz = self.geometry.dims
        out = [np.empty((nz, ny, nx)) for _ in range(4)]
        h = self._handle
        _lib.check(h.lib.lbm_get_macroscopic(h.h, *[_lib.ptr(a) for a in out]))
        return tuple(out)

    def macroscopic_box(self, x=None, y=None, z=None):
        """(rho, v_x, v_y, v_z) on the sub-box x=(x0, x1), y=..., z=...
        (half-open, default whole axis), computed on the device; arrays
        shaped (z1-z0, y1-y0, x1-x0).  Observers use it to probe lines and
        planes without downloading the domain."""
        self.field.flush()
        dims = self.geometry.dims
        lo, hi = [], []
        for a, r in enumerate((x, y, z)):
            r = (0, dims[a]) if r is None else ((int(r), int(r) + 1) if np.isscalar(r) else r)
            lo.append(int(r[0]))
            hi.append(int(r[1]))
        shape = (hi[2] - lo[2], hi[1] - lo[1], hi[0] - lo[0])
        if min(shape) <= 0:
            raise ValueError(f"empty box {lo} .. {hi}")
        out = [np.empty(shape) for _ in range(4)]
        lo_a = np.asarray(lo, dtype=np.int32)
        hi_a = np.asarray(hi, dtype=np.int32)
        h = self._handle
        _lib.check(h.lib.lbm_get_macroscopic_box(h.h, _lib.ptr(lo_a), _lib.ptr(hi_a),
                                                 *[_lib.ptr(a) for a in out]), "macroscopic_box")
        return tuple(out)

    def density_field(self):
        """Per-node rho only, float64 (n_z, n_y, n_x) -- a quarter of the
        macroscopic_fields() readback, for domains near the host-memory limit."""
        self.field.flush()
        nx, ny, nz = self.geometry.dims
        rho = np.empty((nz, ny, nx))
        h = self._handle
        _lib.check(h.lib.lbm_get_macroscopic(h.h, _lib.ptr(rho), None, None, None))
        return rho

    def total_mass(self):
        self.field.flush()
        m = C.c_double(0.0)
        _lib.check(self._handle.lib.lbm_total_mass(self._handle.h, C.byref(m)))
        return float(m.value)

    def canonical_state(self, which="pre"):
        """(19, n_z, n_y, n_x) copy of a buffer; nodes without storage read 0
        (the reference tests' canonical_state, t/conftest.py:7-17)."""
        self.field.flush()
        nx, ny, nz = self.geometry.dims
        out = np.empty((Q, nz, ny, nx), dtype=self.dtype)
        _lib.check(self._handle.lib.lbm_get_pdf(self._handle.h, 0 if which == "pre" else 1,
                                                _lib.ptr(out)))
        return out

    def set_state(self, f, which="pre"):
        self.field.invalidate()
        f = np.ascontiguousarray(f, dtype=self.dtype)
        nx, ny, nz = self.geometry.dims
        if f.shape != (Q, nz, ny, nx):
            raise ValueError(f"state must have shape {(Q, nz, ny, nx)}, got {f.shape}")
        _lib.check(self._handle.lib.lbm_set_pdf(self._handle.h, 0 if which == "pre" else 1,
                                                _lib.ptr(f)))

    # -- z-slab halo ---------------------------------------------------------
    def halo_blob(self):
        """Opaque bytes describing this slab's PDF buffers for its neighbours
        (CUDA IPC handles + device pointers), see lbm_halo_export."""
        buf = (C.c_char * _lib.HALO_BLOB_BYTES)()
        n = C.c_size_t(0)
        _lib.check(self._handle.lib.lbm_halo_export(self._handle.h, buf, C.byref(n)))
        return bytes(buf)[:n.value]

    def connect_halo(self, lo_blob=None, hi_blob=None):
        """Attach the lower / upper neighbour slab (None: no neighbour)."""
        lo = None if lo_blob is None else C.create_string_buffer(lo_blob, len(lo_blob))
        hi = None if hi_blob is None else C.create_string_buffer(hi_blob, len(hi_blob))
        _lib.check(self._handle.lib.lbm_halo_connect(self._handle.h, lo, hi), "halo connect")

    def flag_words(self):
        nx, ny, nz = self.geometry.dims
        out = np.empty((nz, ny, nx), dtype=np.uint32)
        _lib.check(self._handle.lib.lbm_get_flags(self._handle.h, _lib.ptr(out)))
        return out

    def tile_index(self):
        """(tiles (T, 3) as (tx, ty, tz), nbr27 (T, 27)) of a tile layout."""
        h = self._handle
        T = C.c_int64(0)
        _lib.check(h.lib.lbm_get_tile_index(h.h, None, None, C.byref(T)))
        tiles = np.empty((T.value, 3), dtype=np.int32)
        nbr = np.empty((T.value, 27), dtype=np.int32)
        _lib.check(h.lib.lbm_get_tile_index(h.h, _lib.ptr(tiles), _lib.ptr(nbr), C.byref(T)))
        return tiles, nbr
