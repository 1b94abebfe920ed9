"""Node descriptors, boundary-value table and storage-layout names (3-D).

Mirrors pkg/src/sparselbm/layouts.py: `NodeType` and `Orientation` keep the
reference codes (layouts.py:55-70) and add the two z faces; the
`BoundaryValueTable` stores 3-vectors (layouts.py:73-132); the
`NodeDescriptorField` holds (nz, ny, nx) arrays indexed [z, y, x].

The per-node neighbour masks, flag words and the sparse tile index are built
ON THE DEVICE by the library (lbm_set_geometry); `NodeDescriptorField.
neighbor_mask` downloads them.  Storage layouts:

* dense         SoA (19, plane_stride), x fastest, row pitch padded to 128 B,
                one ghost plane above/below; visits every node
* bitmask_node  dense storage, counts visits over non-solid nodes only
* tile          every Tx*Ty*Tz tile allocated (default 8^3)
* pointer_tile  compacted list of tiles holding >= 1 non-solid node plus a
                27-entry neighbour table (the sparse layout); alias
                "tile_sparse" / "sparse"
"""

import enum

import numpy as np

from . import _lib


class LayoutKind(enum.Enum):
    DENSE = "dense"
    TILE = "tile"
    BITMASK_NODE = "bitmask_node"
    POINTER_TILE = "pointer_tile"

    @classmethod
    def parse(cls, name):
        if isinstance(name, cls):
            return name
        key = str(name).strip().lower().replace("-", "_")
        key = {"tile_sparse": "pointer_tile", "sparse": "pointer_tile"}.get(key, key)
        for kind in cls:
            if kind.value == key:
                return kind
        raise ValueError(f"unknown layout {name!r}; expected one of "
                         f"{[k.value for k in cls]}")


class NodeType(enum.IntEnum):
    SOLID = 0
    FLUID = 1
    BOUNCE_BACK_WALL = 2
    VELOCITY_BC = 3
    PRESSURE_BC = 4


class Orientation(enum.IntEnum):
    """Domain face a boundary node sits on (Zou-He closure selector)."""

    NONE = 0
    NORTH = 1    # y = n_y - 1
    SOUTH = 2    # y = 0
    EAST = 3     # x = n_x - 1
    WEST = 4     # x = 0
    TOP = 5      # z = n_z - 1
    BOTTOM = 6   # z = 0


class BoundaryValueTable:
    """Imposed values referenced by a node's bc_index: a velocity 3-vector or a
    density (reference layouts.py:73-132)."""

    KIND_VELOCITY = 0
    KIND_PRESSURE = 1

    def __init__(self):
        self._kinds = []
        self._vel = []
        self._rho = []

    def add_velocity(self, vx, vy, vz=0.0):
        self._kinds.append(self.KIND_VELOCITY)
        self._vel.append((float(vx), float(vy), float(vz)))
        self._rho.append(0.0)
        return len(self._kinds) - 1

    def add_pressure(self, rho):
        if rho <= 0:
            raise ValueError(f"imposed density must be positive, got {rho}")
        self._kinds.append(self.KIND_PRESSURE)
        self._vel.append((0.0, 0.0, 0.0))
        self._rho.append(float(rho))
        return len(self._kinds) - 1

    def kind(self, idx):
        return self._kinds[idx]

    def velocity(self, idx):
        if self._kinds[idx] != self.KIND_VELOCITY:
            raise ValueError(f"entry {idx} is not a velocity entry")
        return np.array(self._vel[idx])

    def pressure(self, idx):
        if self._kinds[idx] != self.KIND_PRESSURE:
            raise ValueError(f"entry {idx} is not a pressure entry")
        return self._rho[idx]

    def as_arrays(self, dtype=np.float64):
        """(kinds u8, velocities (n, 3), densities (n,)); n >= 1 rows."""
        n = len(self._kinds)
        kinds = np.array(self._kinds, dtype=np.uint8)
        vel = np.zeros((max(n, 1), 3), dtype=dtype)
        rho = np.zeros(max(n, 1), dtype=dtype)
        for i in range(n):
            vel[i] = self._vel[i]
            rho[i] = self._rho[i]
        return kinds, vel, rho

    def __len__(self):
        return len(self._kinds)

    def __eq__(self, other):
        if not isinstance(other, BoundaryValueTable):
            return NotImplemented
        return (self._kinds == other._kinds and self._vel == other._vel
                and self._rho == other._rho)


class NodeDescriptorField:
    """Per-node type tags, orientations and boundary indices, (nz, ny, nx).

    `periodic` marks axes (x, y, z) that wrap; the reference has none, the
    channel cases need a periodic span.
    """

    def __init__(self, type_tag, bc_index=None, orientation=None,
                 periodic=(False, False, False)):
        type_tag = np.ascontiguousarray(type_tag, dtype=np.uint8)
        if type_tag.ndim != 3:
            raise ValueError("type_tag must be a 3-D (n_z, n_y, n_x) array")
        shape = type_tag.shape
        self.type_tag = type_tag
        self.bc_index = (np.full(shape, -1, dtype=np.int32) if bc_index is None else
                         np.ascontiguousarray(np.asarray(bc_index, dtype=np.int32).reshape(shape)))
        self.orientation = (np.zeros(shape, dtype=np.uint8) if orientation is None else
                            np.ascontiguousarray(np.asarray(orientation, dtype=np.uint8).reshape(shape)))
        self.periodic = tuple(bool(p) for p in periodic)
        if len(self.periodic) != 3:
            raise ValueError("periodic needs one flag per axis (x, y, z)")
        self._mask = None

    @property
    def dims(self):
        n_z, n_y, n_x = self.type_tag.shape
        return (n_x, n_y, n_z)

    @property
    def flag_words(self):
        """Packed u32 flag words computed by the device (bits 0-17 mask,
        18-20 type, 21-23 orientation, 24-31 bc_index)."""
        from .kernel import device_flag_words
        return device_flag_words(self)

    @property
    def neighbor_mask(self):
        """18-bit neighbour-presence masks (bit j-1 <-> direction j), computed
        on the device (reference layouts.py:173-188)."""
        if self._mask is None:
            self._mask = (self.flag_words & np.uint32(0x3FFFF)).astype(np.uint32)
        return self._mask

    def recompute_neighbor_masks(self):
        self._mask = None

    def non_solid_count(self):
        return int(np.count_nonzero(self.type_tag != NodeType.SOLID))

    def count(self, node_type):
        return int(np.count_nonzero(self.type_tag == node_type))

    def copy(self):
        return NodeDescriptorField(self.type_tag.copy(), self.bc_index.copy(),
                                   self.orientation.copy(), self.periodic)

    def __eq__(self, other):
        if not isinstance(other, NodeDescriptorField):
            return NotImplemented
        return (np.array_equal(self.type_tag, other.type_tag)
                and np.array_equal(self.bc_index, other.bc_index)
                and np.array_equal(self.orientation, other.orientation)
                and self.periodic == other.periodic)


# ---------------------------------------------------------------------------
# default tile shape (the reference takes one fixed tile edge per layout,
# layouts.py:389-401; here the facade picks between two measured shapes)

DEFAULT_TILE = (4, 4, 8)
SPARSE_TILE = (4, 4, 4)
# node fill of the kept 4x4x8 tiles below which 4x4x4 tiles step faster with
# the AB scheme (profiles/ab_tile_fill_r02al.txt: +4 % at fill 0.49, +2.5 % at
# 0.59, +0.5 % at 0.67-0.68, -2.4 % at 0.79, -2.5 % at 0.89; level under A-A)
SPARSE_TILE_FILL = 0.70


def kept_tile_fill(type_tag, tile=DEFAULT_TILE):
    """Non-solid nodes / nodes of the kept tiles (tiles holding at least one
    non-solid node) for `type_tag` (z, y, x) cut into `tile` = (x, y, z)
    edges, or None when the extents are not multiples of the edges.  The
    x-any uses word views (4 bytes = 4 x-neighbours), 0.3 s for 1024^3."""
    t = np.ascontiguousarray(type_tag, dtype=np.uint8)
    ex, ey, ez = (int(e) for e in tile)
    nz, ny, nx = t.shape
    if ex != 4 or ny % ey or nz % ez or nx % 4:
        return None
    x = t.view(np.uint32)                                  # (nz, ny, nx / 4)
    y = x.reshape(nz, ny // ey, ey, nx // 4)
    acc = y[:, :, 0].copy()
    for j in range(1, ey):
        acc |= y[:, :, j]
    z = acc.reshape(nz // ez, ez, ny // ey, nx // 4)
    kept = z[:, 0].copy()
    for j in range(1, ez):
        kept |= z[:, j]
    n_kept = int(np.count_nonzero(kept))
    if n_kept == 0:
        return None
    live = t.size - int(np.count_nonzero(t == NodeType.SOLID))
    return live / (n_kept * ex * ey * ez)


def default_tile(type_tag, layout, scheme="ab"):
    """Tile shape used when the caller names none: 4x4x8, or 4x4x4 for the
    compacted tile list under the AB scheme when the kept 4x4x8 tiles are
    less than SPARSE_TILE_FILL non-solid (low-porosity media, where smaller
    tiles hug the solid and the step streams faster)."""
    if LayoutKind.parse(layout) is not LayoutKind.POINTER_TILE or str(scheme).lower() != "ab":
        return DEFAULT_TILE
    fill = kept_tile_fill(type_tag, DEFAULT_TILE)
    return SPARSE_TILE if fill is not None and fill < SPARSE_TILE_FILL else DEFAULT_TILE


# ---------------------------------------------------------------------------
# copy micro-benchmark (reference layouts.py:439-524), on the device


def copy_bandwidth_bench(layout, block_bytes, repetitions=100, warmup=5, device=0):
    """Achieved device copy bandwidth (bytes/s, read + write) for one
    layout's access pattern: a flat f64 block of `block_bytes` copied
    `repetitions` times after `warmup` untimed copies (CUDA events), the
    destination verified (reference layouts.py:473-510)."""
    import ctypes as C

    from . import _lib
    layout = LayoutKind.parse(layout) if not isinstance(layout, LayoutKind) else layout
    out = C.c_double(0.0)
    lib = _lib.load()
    _lib.check(lib.lbm_copy_bandwidth(int(device), _lib.LAYOUT_CODES[layout.value], int(block_bytes),
                                      int(repetitions), int(warmup), C.byref(out)), "copy_bandwidth_bench")
    return float(out.value)


def copy_bandwidth_survey(block_bytes, repetitions=20, device=0):
    """Bandwidth per layout plus a logged (never asserted) ordering check
    (reference layouts.py:513-524)."""
    import logging
    results = {k: copy_bandwidth_bench(k, block_bytes, repetitions, device=device) for k in LayoutKind}
    dense, bitmask, pointer = (results[LayoutKind.DENSE], results[LayoutKind.BITMASK_NODE],
                               results[LayoutKind.POINTER_TILE])
    if not dense >= bitmask >= pointer:
        logging.getLogger(__name__).info(
            "copy-bandwidth ordering dense >= bitmask >= pointer not observed: %s",
            {k.value: f"{v / 1e9:.2f} GB/s" for k, v in results.items()})
    return results

