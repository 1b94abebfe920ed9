"""ORACLE (test infrastructure only) -- node descriptors, neighbour masks,
packed flag words and the sparse tile index, restated on the CPU in numpy.

* `neighbor_masks` follows NodeDescriptorField.recompute_neighbor_masks
  (reference pkg/src/sparselbm/layouts.py:173-188): bit (j - 1) is set iff the
  neighbour in direction j lies in the domain (or wraps across a periodic
  axis -- the reference has no periodic axes) and is not
  SOLID; solid nodes keep mask 0.  D3Q19 has 18 bits.
* `flag_words` packs the GPU flag word: bits 0-17 mask,
  18-20 node type, 21-23 orientation, 24-31 bc_index (0 when < 0).
* `tile_index` restates the pointer-tile compaction of layouts.py:263-269 and
  389-401 in 3-D: a tile is kept iff it holds >= 1 in-domain non-solid node,
  kept tiles are ranked row-major in (tz, ty, tx) order, and `nbr27` records
  the rank of the 26 neighbouring tiles (-1 when outside a non-periodic
  domain or not kept), SURVEY.md A.6.
* `mask_is_symmetric` restates layouts.py:205-226 (vectorised).
"""

import numpy as np

from .lattice19 import CX, CY, CZ, OPP, SOLID, Q


def _shift_present(nonsolid, dx, dy, dz, periodic):
    """present[z, y, x] = nonsolid[z + dz, y + dy, x + dx] (wrapping on the
    periodic axes, False outside the domain on the others)."""
    out = nonsolid
    for axis, d in ((2, dx), (1, dy), (0, dz)):
        if d == 0:
            continue
        rolled = np.roll(out, -d, axis=axis)
        if not periodic[2 - axis]:
            sl = [slice(None)] * 3
            n = out.shape[axis]
            sl[axis] = slice(n - d, n) if d > 0 else slice(0, -d)
            rolled = rolled.copy()
            rolled[tuple(sl)] = False
        out = rolled
    return out


def neighbor_masks(types, periodic=(False, False, False)):
    """(nz, ny, nx) uint32 neighbour-presence masks."""
    types = np.asarray(types, dtype=np.uint8)
    nonsolid = types != SOLID
    mask = np.zeros(types.shape, dtype=np.uint32)
    for j in range(1, Q):
        present = _shift_present(nonsolid, int(CX[j]), int(CY[j]), int(CZ[j]),
                                 periodic)
        mask |= present.astype(np.uint32) << np.uint32(j - 1)
    mask[~nonsolid] = 0
    return mask


def flag_words(types, orient, bc_index, periodic=(False, False, False)):
    types = np.asarray(types, dtype=np.uint8)
    orient = np.asarray(orient, dtype=np.uint8)
    bc_index = np.asarray(bc_index, dtype=np.int32)
    m = neighbor_masks(types, periodic)
    b = np.where(bc_index < 0, 0, bc_index).astype(np.uint32) & np.uint32(0xFF)
    w = (m | (types.astype(np.uint32) << np.uint32(18))
         | (orient.astype(np.uint32) << np.uint32(21)) | (b << np.uint32(24)))
    return w.astype(np.uint32)


def mask_is_symmetric(types, masks, periodic=(False, False, False)):
    types = np.asarray(types, dtype=np.uint8)
    nonsolid = types != SOLID
    for j in range(1, Q):
        bit = ((masks >> np.uint32(j - 1)) & 1).astype(bool)
        present = _shift_present(nonsolid, int(CX[j]), int(CY[j]), int(CZ[j]),
                                 periodic)
        if np.any(bit[nonsolid] != present[nonsolid]):
            return False
        # neighbour must see us through the opposite bit
        ob = ((masks >> np.uint32(int(OPP[j]) - 1)) & 1).astype(bool)
        back = _shift_present(ob, int(CX[j]), int(CY[j]), int(CZ[j]), periodic)
        if np.any(bit & ~back):
            return False
    return True


def tile_grid(dims, tile):
    nx, ny, nz = dims
    tx, ty, tz = tile
    return (-(-nx // tx), -(-ny // ty), -(-nz // tz))


def tile_index(types, tile=(8, 8, 8), periodic=(False, False, False),
               keep_all=False):
    """Return (tiles (T, 3) int32 as (tx, ty, tz), nbr27 (T, 27) int32,
    rank grid (gz, gy, gx) int32 with -1 for dropped tiles)."""
    types = np.asarray(types, dtype=np.uint8)
    nz, ny, nx = types.shape
    ex, ey, ez = tile
    gx, gy, gz = tile_grid((nx, ny, nz), tile)
    padded = np.zeros((gz * ez, gy * ey, gx * ex), dtype=bool)
    padded[:nz, :ny, :nx] = types != SOLID
    keep = padded.reshape(gz, ez, gy, ey, gx, ex).any(axis=(1, 3, 5))
    if keep_all:
        keep[:] = True
    rank = np.full((gz, gy, gx), -1, dtype=np.int32)
    rank[keep] = np.arange(int(keep.sum()), dtype=np.int32)
    kz, ky, kx = np.nonzero(keep)            # row-major (tz, ty, tx) order
    tiles = np.stack([kx, ky, kz], axis=1).astype(np.int32)
    T = tiles.shape[0]
    nbr = np.full((T, 27), -1, dtype=np.int32)
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                col = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1)
                qx, qy, qz = kx + dx, ky + dy, kz + dz
                ok = np.ones(T, dtype=bool)
                for q, g, per in ((qx, gx, periodic[0]), (qy, gy, periodic[1]),
                                  (qz, gz, periodic[2])):
                    if per:
                        q %= g
                    else:
                        ok &= (q >= 0) & (q < g)
                vals = np.full(T, -1, dtype=np.int32)
                vals[ok] = rank[qz[ok], qy[ok], qx[ok]]
                nbr[:, col] = vals
    return tiles, nbr, rank
