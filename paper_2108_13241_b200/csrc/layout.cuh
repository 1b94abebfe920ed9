// Device-side layout: the Geo parameter block, the in-tile brick order, slot
// maps and the A-A decoder (where the reference's pre_i(x) lives).
// Part of liblbm19 (included once, in order, by lbm19.cu).
#pragma once

// ------------------------------------------------------------- device params
struct Geo {
  int nx, ny, nz, nxp;     // extents; nxp = padded row pitch (dense)
  long long plane;         // ny * nxp (dense)
  long long ps;            // elements between direction planes
  int px, py, pzw;         // periodic x, y; wrap z inside this handle
  int tiled;               // tile layout?
  int ex, ey, ez, lex, ley, lez;  // tile edges and their log2
  int lbx, lby, lbz;       // log2 of the in-tile brick (one 32-B sector: 2x2x2 fp32, 2x2x1 fp64)
  int gx, gy, gz;          // tile grid
  int tn;                  // nodes per tile
  int ltn;                 // log2(tn)
  int zero_fill;           // complete mixed sectors with zeros (full-sector stores)
  int aa;                  // LBM_SCHEME_AA: one buffer updated in place
  int aph;                 // AA state phase (step_count mod 2), set per readback launch
};

// In-tile slot order: the tile is cut into bricks of one 32-byte sector
// (2x2x2 fp32 / 2x2x1 fp64 nodes), bricks x-fastest, nodes x-fastest inside
// a brick.  A sector then holds a compact brick instead of an 8-node x-row,
// which raises the live fraction of fetched sectors on sparse geometries.
// The order is separable: loc = bx(lx) + by(ly) + bz(lz) (disjoint bits).
__host__ __device__ __forceinline__ int brick_x(const Geo& g, int lx) {
  return ((lx >> g.lbx) << (g.lbx + g.lby + g.lbz)) | (lx & ((1 << g.lbx) - 1));
}
__host__ __device__ __forceinline__ int brick_y(const Geo& g, int ly) {
  return ((ly >> g.lby) << (g.lex - g.lbx + g.lbx + g.lby + g.lbz)) | ((ly & ((1 << g.lby) - 1)) << g.lbx);
}
__host__ __device__ __forceinline__ int brick_z(const Geo& g, int lz) {
  return ((lz >> g.lbz) << (g.lex - g.lbx + g.ley - g.lby + g.lbx + g.lby + g.lbz)) |
         ((lz & ((1 << g.lbz) - 1)) << (g.lbx + g.lby));
}
__host__ __device__ __forceinline__ void brick_inv(const Geo& g, int l, int& lx, int& ly, int& lz) {
  const int lb = g.lbx + g.lby + g.lbz;
  const int r = l & ((1 << lb) - 1), q = l >> lb;
  const int nbx = g.lex - g.lbx, nby = g.ley - g.lby;
  lx = ((q & ((1 << nbx) - 1)) << g.lbx) | (r & ((1 << g.lbx) - 1));
  ly = (((q >> nbx) & ((1 << nby) - 1)) << g.lby) | ((r >> g.lbx) & ((1 << g.lby) - 1));
  lz = ((q >> (nbx + nby)) << g.lbz) | (r >> (g.lbx + g.lby));
}

// element index of (direction i, slot s): dense SoA i*ps + s; tiles AoSoA
// f[tile][i][node], i.e. each tile's 19 direction blocks are contiguous
__host__ __device__ __forceinline__ long long fidx(const Geo& g, int i, long long s) {
  if (!g.tiled) return (long long)i * g.ps + s;
  return ((s >> g.ltn) * Q + i) << g.ltn | (s & (g.tn - 1));
}

struct SlotMap {
  const int* rank;  // tile rank grid (gz, gy, gx), -1 = not allocated (tile layouts)
  __device__ __forceinline__ long long slot(const Geo& g, int x, int y, int z) const {
    if (!g.tiled) return ((long long)(z + 1) * g.ny + y) * g.nxp + x;
    const int tx = x >> g.lex, ty = y >> g.ley, tz = z >> g.lez;
    const int r = rank[((long long)tz * g.gy + ty) * g.gx + tx];
    if (r < 0) return -1;
    const int l = brick_x(g, x & (g.ex - 1)) + brick_y(g, y & (g.ey - 1)) + brick_z(g, z & (g.ez - 1));
    return (long long)r * g.tn + l;
  }
  // flag-array index of a slot (dense flags carry no ghost planes)
  __device__ __forceinline__ long long flag_index(const Geo& g, long long s) const {
    return g.tiled ? s : s - g.plane;
  }
  // slot of the neighbour x + c_i of a node whose link i is present (so the
  // neighbour is inside the domain or across a periodic face)
  __device__ __forceinline__ long long nbr_slot(const Geo& g, int x, int y, int z, int i) const {
    x += cx(i);
    y += cy(i);
    z += cz(i);
    if (x < 0) x += g.nx; else if (x >= g.nx) x -= g.nx;
    if (y < 0) y += g.ny; else if (y >= g.ny) y -= g.ny;
    if (g.pzw) { if (z < 0) z += g.nz; else if (z >= g.nz) z -= g.nz; }
    return slot(g, x, y, z);
  }
};

// Where pre_i(x) of the reference lives (element index into the buffer).
// AB: the pre buffer itself.  AA (one buffer F, in place):
//   phase 0 (even step count): pre_i(x) = F[opp(i)][x]
//   phase 1 (odd):             pre_i(x) = F[i][x + c_i] if link i of x is
//                              present, else F[opp(i)][x]
// (see k_step_dense_aa for the two steps that produce these states).
// Tile A-A z-slabs: a present link across the cut has x + c_i in the
// neighbouring slab; the neighbour step mirrored that push into the region
// appended to this slab's buffer (offset Q * ps, step_tiles.cuh TileAAHalo).
__device__ __forceinline__ long long pre_index(const Geo& g, const SlotMap& sm, int i, long long s,
                                               uint32_t w, int x, int y, int z) {
  if (!g.aa || i == 0) return fidx(g, i, s);
  if (g.aph && ((w >> (i - 1)) & 1u)) {
    const int zz = z + cz(i);
    if (g.tiled && !g.pzw && (zz < 0 || zz >= g.nz)) {
      int xx = x + cx(i), yy = y + cy(i);
      if (xx < 0) xx += g.nx; else if (xx >= g.nx) xx -= g.nx;
      if (yy < 0) yy += g.ny; else if (yy >= g.ny) yy -= g.ny;
      const long long pn = (long long)g.nx * g.ny;
      const int j = zz < 0 ? (i - 10) / 2 : 5 + (i - 9) / 2;  // kZm(j) -> j, kZp(j) -> 5 + j
      return (long long)Q * g.ps + j * pn + (long long)yy * g.nx + xx;
    }
    return fidx(g, i, sm.nbr_slot(g, x, y, z, i));
  }
  return fidx(g, opp(i), s);
}
