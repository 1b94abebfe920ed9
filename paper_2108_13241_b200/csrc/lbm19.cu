// liblbm19 -- B200-native D3Q19 fused pull stream + BGK collide (sm_100a).
//
// Drop-in replacement for the reference's compiled step operator
// (pkg/src/sparselbm/kernel.py:56-141) and the Simulation plumbing around it;
// the C-ABI is declared in include/lbm19.h.  Kernels:
//
//   k_flags        node descriptors -> packed u32 flag word per slot (mask,
//                  type, orientation, bc index); layouts.py:173-188 on device
//   k_tile_keep / k_tile_compact
//                  sparse tile index: kept-tile flags, exclusive scan (CUB),
//                  compacted (tx,ty,tz) list and the 27-entry neighbour table
//                  (layouts.py:263-269, 389-401 generalised)
//   k_init         float64 equilibrium, cast to the storage type (kernel.py:190-237)
//   k_step_dense   ONE fused pass per step: pull gather with link-wise bounce-back,
//                  Zou-He closures, moments, BGK, node-local store (kernel.py:72-141)
//   k_step_tile    the same over the compacted tile list + nbr27
//   k_macro / k_mass / k_nonfinite / k_get_pdf / k_set_pdf   readbacks
//
// Storage (HBM): two buffers, each (19, plane_stride) in the storage type.
//   dense: slot(x,y,z) = ((z+1)*ny + y)*nxp + x, nxp = nx rounded up to 32,
//          one ghost plane below and above (z-slab halos / periodic wrap);
//   tile:  slot = rank*TN + ((lz*ey + ly)*ex + lx), each (tile, direction)
//          block contiguous (8^3 fp32 -> 2 KB).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <unistd.h>
#include <string>
#include <thread>
#include <vector>

#include "d3q19.cuh"
#include "lbm19.h"

using namespace lbm;

// ------------------------------------------------------------ error plumbing
static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      if (e_ == cudaErrorMemoryAllocation) {                                          \
        cudaGetLastError();                                                           \
        return fail(LBM_ENOMEM, "%s: %s", #call, cudaGetErrorString(e_));             \
      }                                                                               \
      return fail(LBM_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                          \
    }                                                                                 \
  } while (0)

#define CKL() CK(cudaGetLastError())

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
__device__ __forceinline__ long long fidx(const Geo& g, int i, long long s) {
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
__device__ __forceinline__ long long pre_index(const Geo& g, const SlotMap& sm, int i, long long s,
                                               uint32_t w, int x, int y, int z) {
  if (!g.aa || i == 0) return fidx(g, i, s);
  if (g.aph && ((w >> (i - 1)) & 1u)) return fidx(g, i, sm.nbr_slot(g, x, y, z, i));
  return fidx(g, opp(i), s);
}

// --------------------------------------------------------------- geometry
__device__ __forceinline__ uint32_t type_at(const uint8_t* __restrict__ type,
                                            const uint8_t* __restrict__ glo,
                                            const uint8_t* __restrict__ ghi, const Geo& g, int x,
                                            int y, int z) {
  // returns 0 (SOLID / absent) outside the domain on non-periodic axes
  if (x < 0 || x >= g.nx) {
    if (!g.px) return SOLID;
    x = x < 0 ? x + g.nx : x - g.nx;
  }
  if (y < 0 || y >= g.ny) {
    if (!g.py) return SOLID;
    y = y < 0 ? y + g.ny : y - g.ny;
  }
  if (z < 0) return glo ? glo[(long long)y * g.nx + x] : SOLID;
  if (z >= g.nz) return ghi ? ghi[(long long)y * g.nx + x] : SOLID;
  return type[((long long)z * g.ny + y) * g.nx + x];
}

__device__ __forceinline__ uint32_t node_flag(const uint8_t* __restrict__ type,
                                              const uint8_t* __restrict__ orient,
                                              const int* __restrict__ bcidx,
                                              const uint8_t* __restrict__ glo,
                                              const uint8_t* __restrict__ ghi, const Geo& g,
                                              int x, int y, int z, int nb, int* err) {
  const long long n = ((long long)z * g.ny + y) * g.nx + x;
  const uint32_t t = type[n];
  const uint32_t o = orient[n];
  const int b = bcidx[n];
  if (t > PRESSURE_BC || o > O_BOTTOM) atomicOr(err, 1);
  if ((t == VELOCITY_BC || t == PRESSURE_BC) && (b < 0 || b >= nb || o == O_NONE)) atomicOr(err, 2);
  uint32_t m = 0;
  if (t != SOLID) {
#pragma unroll
    for (int j = 1; j < Q; ++j)
      if (type_at(type, glo, ghi, g, x + cx(j), y + cy(j), z + cz(j)) != SOLID) m |= 1u << (j - 1);
  }
  return make_flag(m, t, o, b < 0 ? 0u : (uint32_t)b);
}

// dense: one thread per (padded) flag entry
__global__ void k_flags_dense(uint32_t* __restrict__ flags, const uint8_t* __restrict__ type,
                              const uint8_t* __restrict__ orient, const int* __restrict__ bcidx,
                              const uint8_t* __restrict__ glo, const uint8_t* __restrict__ ghi,
                              Geo g, int nb, int* err, unsigned long long* nonsolid) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= g.nxp) return;
  uint32_t w = 0;
  if (x < g.nx) w = node_flag(type, orient, bcidx, glo, ghi, g, x, y, z, nb, err);
  flags[((long long)z * g.ny + y) * g.nxp + x] = w;
  const unsigned c = __popc(__ballot_sync(0xffffffffu, flag_type(w) != SOLID));
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(nonsolid, (unsigned long long)c);
}

// tiles: one warp per tile of the full tile grid -> keep flag
__global__ void k_tile_keep(int* __restrict__ keep, const uint8_t* __restrict__ type, Geo g,
                            int keep_all, long long ntiles) {
  const long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= ntiles) return;
  int any = 0;
  if (keep_all) {
    any = 1;
  } else {
    const int tx = (int)(t % g.gx), ty = (int)((t / g.gx) % g.gy), tz = (int)(t / ((long long)g.gx * g.gy));
    for (int l = lane; l < g.tn && !any; l += 32) {
      const int lx = l & (g.ex - 1), ly = (l >> g.lex) & (g.ey - 1), lz = l >> (g.lex + g.ley);
      const int x = tx * g.ex + lx, y = ty * g.ey + ly, z = tz * g.ez + lz;
      if (x < g.nx && y < g.ny && z < g.nz && type[((long long)z * g.ny + y) * g.nx + x] != SOLID) any = 1;
    }
    any = __any_sync(0xffffffffu, any);
  }
  if (lane == 0) keep[t] = any;
}

__global__ void k_tile_compact(int* __restrict__ rank, const int* __restrict__ keep,
                               const int* __restrict__ scan, int* __restrict__ tiles, Geo g,
                               long long ntiles) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  if (keep[t]) {
    const int r = scan[t];
    rank[t] = r;
    tiles[3LL * r + 0] = (int)(t % g.gx);
    tiles[3LL * r + 1] = (int)((t / g.gx) % g.gy);
    tiles[3LL * r + 2] = (int)(t / ((long long)g.gx * g.gy));
  } else {
    rank[t] = -1;
  }
}

__global__ void k_tile_nbr(int* __restrict__ nbr, const int* __restrict__ tiles,
                           const int* __restrict__ rank, Geo g, long long T) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= T * 27) return;
  const long long t = k / 27;
  const int c = (int)(k % 27);
  const int dx = c % 3 - 1, dy = (c / 3) % 3 - 1, dz = c / 9 - 1;
  int qx = tiles[3 * t] + dx, qy = tiles[3 * t + 1] + dy, qz = tiles[3 * t + 2] + dz;
  int v = -1;
  bool ok = true;
  if (qx < 0 || qx >= g.gx) { if (g.px) qx = (qx + g.gx) % g.gx; else ok = false; }
  if (qy < 0 || qy >= g.gy) { if (g.py) qy = (qy + g.gy) % g.gy; else ok = false; }
  if (qz < 0 || qz >= g.gz) { if (g.pzw) qz = (qz + g.gz) % g.gz; else ok = false; }
  if (ok) v = rank[((long long)qz * g.gy + qy) * g.gx + qx];
  nbr[k] = v;
}

// Morton key of each kept tile (x, y, z bits interleaved), sorted to a launch
// order: 3-D neighbours of a tile then run close in time, so the sectors they
// share (pulled across tile faces, or pushed by the AA neighbour step) are
// still in L2 when the second CTA touches them.  The rank order itself --
// the reference's row-major pointer-tile order -- is unchanged.
__device__ __forceinline__ unsigned long long spread3(unsigned v) {
  unsigned long long x = v & 0x1fffffu;
  x = (x | x << 32) & 0x1f00000000ffffULL;
  x = (x | x << 16) & 0x1f0000ff0000ffULL;
  x = (x | x << 8) & 0x100f00f00f00f00fULL;
  x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
  x = (x | x << 2) & 0x1249249249249249ULL;
  return x;
}
// mode 1: Morton; mode 2: y-pencils of B tile rows -- (y block, z, y, x) with
// x fastest, so a tile's z neighbour runs gx*B tiles later instead of gx*gy
__global__ void k_tile_order_key(unsigned long long* __restrict__ key, int* __restrict__ val,
                                 const int* __restrict__ tiles, long long T, int mode, int B, Geo g) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= T) return;
  const unsigned tx = tiles[3 * r], ty = tiles[3 * r + 1], tz = tiles[3 * r + 2];
  if (mode == 1)
    key[r] = spread3(tx) | spread3(ty) << 1 | spread3(tz) << 2;
  else if (mode == 2)
    key[r] = ((((unsigned long long)(ty / B) * g.gz + tz) * B + ty % B) * g.gx) + tx;
  else  // mode 3: z-groups of B tile layers interleaved, (tz / B, ty, tx, tz % B)
    key[r] = ((((unsigned long long)(tz / B) * g.gy + ty) * g.gx + tx) * B) + tz % B;
  val[r] = (int)r;
}

// tiles: one thread per slot of the kept tiles
__global__ void k_flags_tile(uint32_t* __restrict__ flags, const int* __restrict__ tiles,
                             const uint8_t* __restrict__ type, const uint8_t* __restrict__ orient,
                             const int* __restrict__ bcidx, const uint8_t* __restrict__ glo,
                             const uint8_t* __restrict__ ghi, Geo g, long long nslots, int nb,
                             int* err, unsigned long long* nonsolid) {
  const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t w = 0;
  if (s < nslots) {
    const long long t = s / g.tn;
    const int l = (int)(s - t * g.tn);
    int lx, ly, lz;
    brick_inv(g, l, lx, ly, lz);
    const int x = tiles[3 * t] * g.ex + lx;
    const int y = tiles[3 * t + 1] * g.ey + ly;
    const int z = tiles[3 * t + 2] * g.ez + lz;
    if (x < g.nx && y < g.ny && z < g.nz) w = node_flag(type, orient, bcidx, glo, ghi, g, x, y, z, nb, err);
    flags[s] = w;
  }
  const unsigned c = __popc(__ballot_sync(0xffffffffu, s < nslots && flag_type(w) != SOLID));
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(nonsolid, (unsigned long long)c);
}

// dense: bit c of the uniform-chunk bitmap is set iff the 32 nodes of warp
// chunk c (flag index 32c .. 32c + 31) are all FLUID / BOUNCE_BACK_WALL with
// a full neighbour mask -- such warps skip the per-node flag load
__global__ void k_uniform_bits(uint32_t* __restrict__ ubits, const uint32_t* __restrict__ flags,
                               long long nflags) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t w = k < nflags ? flags[k] : 0u;
  const uint32_t t = flag_type(w);
  const bool simple = k < nflags && (w & kMaskBits) == kMaskBits && (t == FLUID || t == BOUNCE_BACK_WALL);
  const unsigned all = __ballot_sync(0xffffffffu, simple);
  if ((threadIdx.x & 31) == 0 && all == 0xffffffffu) atomicOr(ubits + (k >> 10), 1u << ((k >> 5) & 31));
}

// live-brick masks: bit b of tile t is set iff brick b holds a non-solid node
// words 0-3 of a tile: live bricks; words 4-7: uniform bricks (every node
// FLUID / BOUNCE_BACK_WALL with a full mask: the step skips their flag words)
__global__ void k_brick_mask(uint32_t* __restrict__ bmask, const uint32_t* __restrict__ flags, Geo g,
                             long long nbricks) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nbricks) return;
  const int lbn = g.lbx + g.lby + g.lbz;
  const long long t = k >> (g.ltn - lbn);
  const int b = (int)(k & ((g.tn >> lbn) - 1));
  bool live = false, uni = true;
  for (int r = 0; r < (1 << lbn); ++r) {
    const uint32_t w = flags[(k << lbn) + r];
    const uint32_t ty = flag_type(w);
    live |= ty != SOLID;
    uni &= (w & kMaskBits) == kMaskBits && (ty == FLUID || ty == BOUNCE_BACK_WALL);
  }
  if (live) atomicOr(bmask + 8 * t + (b >> 5), 1u << (b & 31));
  if (uni) atomicOr(bmask + 8 * t + 4 + (b >> 5), 1u << (b & 31));
}

// ------------------------------------------------------------ init / readback
template <typename T>
__global__ void k_init(T* __restrict__ pre, const uint32_t* __restrict__ flags, SlotMap sm, Geo g,
                       const double* __restrict__ rho, const double* __restrict__ ux,
                       const double* __restrict__ uy, const double* __restrict__ uz, double rho0,
                       double ux0, double uy0, double uz0, const uint8_t* __restrict__ bckind,
                       const double* __restrict__ bcv, const double* __restrict__ bcr, int nb) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= g.nx) return;
  const long long s = sm.slot(g, x, y, z);
  if (s < 0) return;
  const uint32_t w = flags[sm.flag_index(g, s)];
  const uint32_t t = flag_type(w);
  if (t == SOLID) return;
  const long long n = ((long long)z * g.ny + y) * g.nx + x;
  double r = rho ? rho[n] : rho0, vx = ux ? ux[n] : ux0, vy = uy ? uy[n] : uy0, vz = uz ? uz[n] : uz0;
  const int b = (int)flag_bc(w);
  if (t == VELOCITY_BC && b < nb && bckind[b] == 0) {
    vx = bcv[3 * b];
    vy = bcv[3 * b + 1];
    vz = bcv[3 * b + 2];
  } else if (t == PRESSURE_BC && b < nb && bckind[b] == 1) {
    r = bcr[b];
  }
  // AA starts in phase 0: pre_i(x) sits at F[opp(i)][x]
#pragma unroll
  for (int i = 0; i < Q; ++i) pre[fidx(g, g.aa ? opp(i) : i, s)] = (T)init_eq(i, r, vx, vy, vz);
}

template <typename T>
__global__ void k_macro(const T* __restrict__ pre, const uint32_t* __restrict__ flags, SlotMap sm,
                        Geo g, int z0, double* __restrict__ rho, double* __restrict__ ux,
                        double* __restrict__ uy, double* __restrict__ uz, int bx0 = 0, int by0 = 0,
                        int bnx = -1) {
  // box [bx0, bx0 + bnx) x [by0, by0 + gridDim.y) x [z0, z0 + gridDim.z) into
  // a staging chunk (the whole x/y extent by default)
  if (bnx < 0) bnx = g.nx;
  const int lx = blockIdx.x * blockDim.x + threadIdx.x;
  if (lx >= bnx) return;
  const int x = bx0 + lx, y = by0 + blockIdx.y, z = blockIdx.z + z0;
  const long long n = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * bnx + lx;
  const long long s = sm.slot(g, x, y, z);
  double r = 0, vx = 0, vy = 0, vz = 0;
  const uint32_t w = s >= 0 ? flags[sm.flag_index(g, s)] : 0u;
  if (s >= 0 && flag_type(w) != SOLID) {
    double f[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) f[i] = (double)pre[pre_index(g, sm, i, s, w, x, y, z)];
    using A = ar<double>;
    r = density19(f);
    if (r != 0.0) {
      double mx, my, mz;
      momentum19(f, mx, my, mz);
      vx = A::div(mx, r);
      vy = A::div(my, r);
      vz = A::div(mz, r);
    }
  }
  if (rho) rho[n] = r;
  if (ux) ux[n] = vx;
  if (uy) uy[n] = vy;
  if (uz) uz[n] = vz;
}

template <typename T>
__global__ void k_get_pdf(const T* __restrict__ buf, const uint32_t* __restrict__ flags, SlotMap sm, Geo g,
                          int z0, T* __restrict__ out) {
  // planes z0 .. z0 + gridDim.z - 1 into a (19, chunk nodes) staging block
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z + z0;
  if (x >= g.nx) return;
  const long long N = (long long)g.nx * g.ny * gridDim.z;
  const long long n = ((long long)blockIdx.z * g.ny + y) * g.nx + x;
  const long long s = sm.slot(g, x, y, z);
  if (s < 0) {
#pragma unroll
    for (int i = 0; i < Q; ++i) out[i * N + n] = (T)0;
    return;
  }
  const uint32_t w = flags[sm.flag_index(g, s)];
  // AA holds only non-solid nodes' values; solid storage reads 0 either way
  const bool live = !g.aa || flag_type(w) != SOLID;
#pragma unroll
  for (int i = 0; i < Q; ++i) out[i * N + n] = live ? buf[pre_index(g, sm, i, s, w, x, y, z)] : (T)0;
}

template <typename T>
__global__ void k_set_pdf(T* __restrict__ buf, const uint32_t* __restrict__ flags, SlotMap sm, Geo g,
                          int z0, const T* __restrict__ in) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z + z0;
  if (x >= g.nx) return;
  const long long N = (long long)g.nx * g.ny * gridDim.z;
  const long long n = ((long long)blockIdx.z * g.ny + y) * g.nx + x;
  const long long s = sm.slot(g, x, y, z);
  if (s < 0) return;
  const uint32_t w = flags[sm.flag_index(g, s)];
  if (g.aa && flag_type(w) == SOLID) return;  // AA: solid storage is never written
#pragma unroll
  for (int i = 0; i < Q; ++i) buf[pre_index(g, sm, i, s, w, x, y, z)] = in[i * N + n];
}

// AA: decoded pre buffer in the native slot order (lbm_get_field / set_field)
template <typename T, bool GET>
__global__ void k_field_aa(T* __restrict__ buf, const uint32_t* __restrict__ flags, SlotMap sm, Geo g,
                           T* __restrict__ io) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= g.nx) return;
  const long long s = sm.slot(g, x, y, z);
  if (s < 0) return;
  const uint32_t w = flags[sm.flag_index(g, s)];
  if (flag_type(w) == SOLID) return;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const long long k = pre_index(g, sm, i, s, w, x, y, z);
    if (GET)
      io[fidx(g, i, s)] = buf[k];
    else
      buf[k] = io[fidx(g, i, s)];
  }
}

__global__ void k_slot_of(SlotMap sm, Geo g, int* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= g.nx) return;
  out[((long long)z * g.ny + y) * g.nx + x] = (int)sm.slot(g, x, y, z);
}

__global__ void k_get_flags(const uint32_t* __restrict__ flags, SlotMap sm, Geo g,
                            uint32_t* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= g.nx) return;
  const long long s = sm.slot(g, x, y, z);
  out[((long long)z * g.ny + y) * g.nx + x] = s >= 0 ? flags[sm.flag_index(g, s)] : 0u;
}

// first non-finite value of `pre` in (direction, visit order); visit order is
// canonical for dense layouts and tile-major for tile layouts
template <typename T>
__global__ void k_nonfinite(const T* __restrict__ pre, const uint32_t* __restrict__ flags, SlotMap sm,
                            Geo g, long long V, unsigned long long* best) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= g.nx) return;
  const long long s = sm.slot(g, x, y, z);
  if (s < 0) return;
  const uint32_t w = flags[sm.flag_index(g, s)];
  if (flag_type(w) == SOLID) return;
  const long long v = g.tiled ? s : ((long long)z * g.ny + y) * g.nx + x;
  for (int i = 0; i < Q; ++i) {
    const T val = pre[pre_index(g, sm, i, s, w, x, y, z)];
    if (!isfinite((double)val)) {
      atomicMin(best, (unsigned long long)(i * V + v));
      return;
    }
  }
}

// deterministic two-pass mass reduction: per-block partial sums, then one block
template <typename T>
__global__ void k_mass_partial(const T* __restrict__ pre, const uint32_t* __restrict__ flags, SlotMap sm,
                               const int* __restrict__ tiles, Geo g, long long nflags,
                               double* __restrict__ partial) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < nflags;
       k += (long long)gridDim.x * blockDim.x) {
    const uint32_t w = flags[k];
    if (flag_type(w) == SOLID) continue;
    const long long s = g.tiled ? k : k + g.plane;
    int x = 0, y = 0, z = 0;  // node coordinates (AA phase 1 reads neighbours)
    if (g.aa && g.aph) {
      if (g.tiled) {
        const long long t = k >> g.ltn;
        brick_inv(g, (int)(k & (g.tn - 1)), x, y, z);
        x += tiles[3 * t] * g.ex;
        y += tiles[3 * t + 1] * g.ey;
        z += tiles[3 * t + 2] * g.ez;
      } else {
        z = (int)(k / g.plane);
        const long long r = k - (long long)z * g.plane;
        y = (int)(r / g.nxp);
        x = (int)(r - (long long)y * g.nxp);
      }
    }
    double a = 0.0;
    for (int i = 0; i < Q; ++i) a += (double)pre[pre_index(g, sm, i, s, w, x, y, z)];
    acc += a;
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void k_mass_final(const double* __restrict__ partial, int n, double* out) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) acc += partial[k];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// ------------------------------------------------------------------ steps
// Solid lanes complete the 32-B sectors of their non-solid neighbours with
// zeros (the values they already hold), so every store is a full sector.
template <typename T>
__device__ __forceinline__ bool sector_needs_zero(bool nonsolid) {
  constexpr int SEC = 32 / (int)sizeof(T);
  const unsigned act = __ballot_sync(0xffffffffu, nonsolid);
  const int lane = threadIdx.x & 31;
  const unsigned grp = ((1u << SEC) - 1u) << (lane & ~(SEC - 1));
  return (act & grp) != 0u;
}

// z-slab halo, fused into the step: the outgoing populations of the two
// boundary planes (c_z = -1 from z = 0, c_z = +1 from z = nz - 1) are stored
// straight into the neighbouring slab's ghost plane (peer memory over
// NVLink / IPC), next to the node-local store.  Null pointers: no neighbour.
__host__ __device__ constexpr int kZm(int j) { return 10 + 2 * j; }  // c_z = -1: 10 12 14 16 18
__host__ __device__ constexpr int kZp(int j) { return 9 + 2 * j; }   // c_z = +1: 9 11 13 15 17
template <typename T>
struct Halo {
  T* lo[5];  // lower neighbour's upper ghost plane, directions kZm
  T* hi[5];  // upper neighbour's lower ghost plane, directions kZp
};

__global__ void k_halo_wait(const unsigned long long* sync, int need_lo, int need_hi,
                            unsigned long long target, int* err) {
  const long long t0 = clock64();
  const volatile unsigned long long* vs = sync;
  while ((need_lo && vs[0] < target) || (need_hi && vs[1] < target)) {
    __nanosleep(200);
    if (clock64() - t0 > 60LL * 2000000000LL) {  // ~1 min at 2 GHz: a neighbour is gone
      atomicOr(err, 1);
      return;
    }
  }
  __threadfence_system();
}

__global__ void k_halo_signal(unsigned long long* lo_slot, unsigned long long* hi_slot,
                              unsigned long long value) {
  __threadfence_system();
  if (lo_slot) *(volatile unsigned long long*)lo_slot = value;
  if (hi_slot) *(volatile unsigned long long*)hi_slot = value;
  __threadfence_system();
}

// initial ghost fill (after initialize / set_pdf): boundary planes of `pre`
template <typename T>
__global__ void k_halo_push(const T* __restrict__ pre, Halo<T> H, Geo g) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= g.nxp) return;
  const int row = y * g.nxp + x;
  const int s0 = (int)g.plane + row, s1 = g.nz * (int)g.plane + row;
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    if (H.lo[0]) H.lo[j][row] = pre[(long long)kZm(j) * g.ps + s0];
    if (H.hi[0]) H.hi[j][row] = pre[(long long)kZp(j) * g.ps + s1];
  }
  __threadfence_system();
}

// 19 direction planes of one buffer, resolved on the host once per launch, so
// every access is a 32-bit slot offset from a per-direction base pointer
template <typename T>
struct Planes {
  const T* pre[Q];
  T* post[Q];
};

template <typename T>
__device__ __forceinline__ void bc_collide(T (&f)[Q], uint32_t w, const T* __restrict__ bcv,
                                           const T* __restrict__ bcr, T om) {
  const uint32_t t = flag_type(w);
  if (t == VELOCITY_BC) {
    const uint32_t b = flag_bc(w);
    zou_he_velocity19<T>(f, flag_orient(w), bcv[3 * b], bcv[3 * b + 1], bcv[3 * b + 2]);
  } else if (t == PRESSURE_BC) {
    zou_he_pressure19<T>(f, flag_orient(w), bcr[flag_bc(w)]);
  }
  T rho, vx, vy, vz;
  moments19(f, rho, vx, vy, vz);
  collide19(f, rho, vx, vy, vz, om);
}

template <typename T>
__device__ __forceinline__ void bc_collide_store(T (&f)[Q], uint32_t w, const T* __restrict__ bcv,
                                                 const T* __restrict__ bcr, T om,
                                                 const Planes<T>& P, unsigned s) {
  bc_collide<T>(f, w, bcv, bcr, om);
#pragma unroll
  for (int i = 0; i < Q; ++i) P.post[i][s] = f[i];
}

// Link-wise bounce-back fix-up: every f_i was loaded speculatively from the
// upstream slot (always a valid address); where the mask bit of opp(i) is
// clear the node reflects its own f_opp(i) instead (reference kernel.py:84-116).
template <typename T>
__device__ __forceinline__ void bounce_back_fixup(T (&f)[Q], uint32_t miss, const Planes<T>& P, unsigned s) {
  if (miss) {
#pragma unroll
    for (int i = 1; i < Q; ++i)
      if ((miss >> (opp(i) - 1)) & 1u) f[i] = __ldg(P.pre[opp(i)] + s);
  }
}

// Gather of the 18 moving populations.  MODE 0: speculative pull of every
// upstream slot, then the fix-up for masked links.  MODE 1: warps whose live
// nodes all have full masks pull unconditionally, the others select per link
// so no byte is fetched for a masked link.
template <typename T, int MODE, typename Up>
__device__ __forceinline__ void gather(T (&f)[Q], uint32_t miss, bool fast, const Planes<T>& P, unsigned s,
                                       Up up) {
  if (MODE == 0 || fast) {
#pragma unroll
    for (int i = 1; i < Q; ++i) f[i] = __ldg(P.pre[i] + up(i));
    if (MODE == 0) bounce_back_fixup(f, miss, P, s);
  } else {
#pragma unroll
    for (int i = 1; i < Q; ++i)
      f[i] = ((miss >> (opp(i) - 1)) & 1u) ? __ldg(P.pre[opp(i)] + s) : __ldg(P.pre[i] + up(i));
  }
}

template <typename T>
__device__ __forceinline__ void zero_fill(const Planes<T>& P, unsigned s) {
#pragma unroll
  for (int i = 0; i < Q; ++i) P.post[i][s] = (T)0;
}

// dense: offsets from slot s to the upstream node x - c_i, per axis (wrap on
// periodic axes; on closed axes the edge offset is 0 and the link is masked,
// so the speculative address stays valid)
struct UpOffsets {
  unsigned xm, xp, ym, yp, zm, zp;
  __device__ __forceinline__ UpOffsets(const Geo& g, int x, int y, int z) {
    xm = x == 0 ? (g.px ? g.nx - 1 : 0) : -1;
    xp = x == g.nx - 1 ? (g.px ? -(g.nx - 1) : 0) : 1;
    ym = y == 0 ? (g.py ? (unsigned)(g.ny - 1) * g.nxp : 0u) : (unsigned)-g.nxp;
    yp = y == g.ny - 1 ? (g.py ? (unsigned)-((g.ny - 1) * g.nxp) : 0u) : (unsigned)g.nxp;
    const unsigned pl = (unsigned)g.plane;
    zm = (z == 0 && g.pzw) ? (unsigned)(g.nz - 1) * pl : 0u - pl;
    zp = (z == g.nz - 1 && g.pzw) ? 0u - (unsigned)(g.nz - 1) * pl : pl;
  }
  // slot of x - c_i
  __device__ __forceinline__ unsigned up(unsigned s, int i) const {
    return s + (cx(i) == 1 ? xm : (cx(i) == -1 ? xp : 0u)) + (cy(i) == 1 ? ym : (cy(i) == -1 ? yp : 0u)) +
           (cz(i) == 1 ? zm : (cz(i) == -1 ? zp : 0u));
  }
};

template <typename T, int MODE, int MINB>
__global__ void __launch_bounds__(128, MINB) k_step_dense(const Planes<T> P, const uint32_t* __restrict__ flags,
                                                   const uint32_t* __restrict__ ubits,
                                                   const T* __restrict__ bcv,
                                                   const T* __restrict__ bcr, Geo g, T om,
                                                   const Halo<T> H) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= g.nxp) return;  // whole warps (nxp % 32 == 0)
  // 32-bit unsigned slot arithmetic (slabs up to 2^32 slots; negative
  // offsets wrap modulo 2^32 and land on the right slot)
  const unsigned fi = ((unsigned)z * g.ny + y) * g.nxp + x;
  const unsigned s = fi + (unsigned)g.plane;
  const uint32_t ub = __ldg(ubits + (fi >> 10));
  const uint32_t w = ((ub >> ((fi >> 5) & 31)) & 1u) ? make_flag(kMaskBits, FLUID, 0, 0) : __ldg(flags + fi);
  const bool live = flag_type(w) != SOLID;
  const bool zfill = sector_needs_zero<T>(live) && g.zero_fill;
  const uint32_t miss = ~w & kMaskBits;
  // warps whose live nodes all have full masks pull unconditionally; the
  // rest select per link, so no byte is fetched for a masked link
  const bool fast = MODE == 1 && __all_sync(0xffffffffu, !live || miss == 0u);
  if (!live) {
    if (zfill) zero_fill(P, s);
    return;
  }
  // offsets to the upstream node x - c_i along each axis (wrap on periodic
  // axes; on closed axes the edge offset is 0 and the link is masked)
  const UpOffsets o(g, x, y, z);
  auto up = [&](int i) { return o.up(s, i); };
  T f[Q];
  f[0] = __ldg(P.pre[0] + s);
  gather<T, MODE>(f, miss, fast, P, s, up);
  bc_collide_store<T>(f, w, bcv, bcr, om, P, s);
  if ((z == 0 && H.lo[0]) || (z == g.nz - 1 && H.hi[0])) {
    const int row = y * g.nxp + x;
    if (z == 0 && H.lo[0]) {
#pragma unroll
      for (int j = 0; j < 5; ++j) H.lo[j][row] = f[kZm(j)];
    }
    if (z == g.nz - 1 && H.hi[0]) {
#pragma unroll
      for (int j = 0; j < 5; ++j) H.hi[j][row] = f[kZp(j)];
    }
    __threadfence_system();
  }
}

// A-A in place (LBM_SCHEME_AA): one buffer F, two alternating kernels, each
// node reading and writing only locations no other node touches in the same
// launch, so no second buffer is needed.  Per reference step (pull gather of
// the previous post-collision values, then collide; kernel.py:72-141):
//   NB = 1 (state phase 0 -> 1), F[opp(i)][x] holds pre_i(x):
//      f_i = F[opp(i)][x - c_i]  if link opp(i) of x is present (pre_i(x - c_i))
//          = F[i][x]             otherwise (bounce-back: pre_opp(i)(x))
//      store f*_i to F[i][x + c_i] if link i is present, else F[opp(i)][x]
//   NB = 0 (phase 1 -> 0): f_i = F[i][x]; store f*_i to F[opp(i)][x]
// F[i][x + c_i] is read (as f_opp(i)) and written by node x alone, so the
// update is race-free; the arithmetic is the AB kernel's, bit for bit.
template <typename T>
struct Planes1 {
  T* f[Q];
};

// AA loads may take the read-only (non-coherent) path: every location is
// read and then written by one thread only, so no cached copy can be stale
template <typename T>
__device__ __forceinline__ T LDA(const T* p) {
  return __ldg(p);
}

// hides a value from the optimiser: the neighbour step's store addresses are
// the load addresses of the opposite directions, and letting the compiler
// keep those 18 addresses live across the collision costs spills; an opaque
// copy makes it recompute them from a handful of offsets instead
__device__ __forceinline__ unsigned opaque(unsigned v) {
  asm volatile("" : "+r"(v));
  return v;
}
__device__ __forceinline__ int opaque(int v) {
  asm volatile("" : "+r"(v));
  return v;
}

template <typename T, int NB, int MINB>
__global__ void __launch_bounds__(128, MINB) k_step_dense_aa(const Planes1<T> P, const uint32_t* __restrict__ flags,
                                                      const uint32_t* __restrict__ ubits,
                                                      const T* __restrict__ bcv, const T* __restrict__ bcr,
                                                      Geo g, T om) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= g.nxp) return;
  const unsigned fi = ((unsigned)z * g.ny + y) * g.nxp + x;
  const unsigned s = fi + (unsigned)g.plane;
  const uint32_t ub = __ldg(ubits + (fi >> 10));
  const uint32_t w = ((ub >> ((fi >> 5) & 31)) & 1u) ? make_flag(kMaskBits, FLUID, 0, 0) : __ldg(flags + fi);
  // no zero-fill of solid lanes here (unlike the AB kernel): every sector
  // this step writes was read by the same step, so it sits in L2 whole and a
  // partial store needs no DRAM read-for-merge; zero stores from solid lanes
  // would instead race ahead of the live lanes' loads of the same sectors
  if (flag_type(w) == SOLID) return;
  const uint32_t miss = ~w & kMaskBits;
  T f[Q];
  f[0] = LDA(P.f[0] + s);
  if (NB) {
    const UpOffsets o(g, x, y, z);
#pragma unroll
    for (int i = 1; i < Q; ++i) f[i] = LDA(P.f[opp(i)] + o.up(s, i));  // speculative, always a valid slot
    if (miss) {
#pragma unroll
      for (int i = 1; i < Q; ++i)
        if ((miss >> (opp(i) - 1)) & 1u) f[i] = LDA(P.f[i] + s);
    }
    bc_collide<T>(f, w, bcv, bcr, om);
    // recompute the store addresses from opaque copies (measured: keeping the
    // 18 load addresses live at 64 registers is no faster)
    const unsigned s2 = opaque(s);
    const UpOffsets o2(g, opaque(x), opaque(y), opaque(z));
    P.f[0][s2] = f[0];
#pragma unroll
    for (int i = 1; i < Q; ++i) {
      T* dst = ((miss >> (i - 1)) & 1u) ? P.f[opp(i)] + s2 : P.f[i] + o2.up(s2, opp(i));
      *dst = f[i];
    }
  } else {
#pragma unroll
    for (int i = 1; i < Q; ++i) f[i] = LDA(P.f[i] + s);
    bc_collide<T>(f, w, bcv, bcr, om);
#pragma unroll
    for (int i = 0; i < Q; ++i) P.f[opp(i)][s] = f[i];
  }
}

// Sparse tiles, AoSoA storage f[tile][i][TN]: one CTA per kept tile.  All
// addresses are 32-bit element offsets from the CTA's own tile block; the
// upstream slot of direction i is separable per axis (tile code
// (dx+1) + 3(dy+1) + 9(dz+1), relative tile offset from shared memory, and
// in-tile offset lx' + ex ly' + ex ey lz'), and every own-tile access
// (bounce-back, stores) has a compile-time offset i*TN.

// Live-brick work list of one tile (MODE 2): threads cover only the tile's
// live bricks (sector-sized bricks holding >= 1 non-solid node, a 128-bit
// mask per tile), so a sparse tile costs lanes in proportion to its live
// sectors, not its TN slots.  Words 4-7 of the mask mark uniform bricks
// (all FLUID / wall with full masks) whose flag words the step skips.
struct TileBricks {
  uint32_t m[4], u[4];
  int pre_cnt[4];
  int work, lbn, bn;
  bool dense_tile;
  __device__ __forceinline__ TileBricks(const uint32_t* __restrict__ bmask, long long t, const Geo& g, int tn,
                                        bool compact) {
    lbn = g.lbx + g.lby + g.lbz;
    bn = 1 << lbn;
    int acc = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      u[q] = __ldg(bmask + 8LL * t + 4 + q);
      m[q] = compact ? __ldg(bmask + 8LL * t + q) : 0u;
      pre_cnt[q] = acc;
      acc += __popc(m[q]);
    }
    work = compact ? ((acc << lbn) + 31) & ~31 : tn;  // whole warps; lanes past acc*bn idle
    dense_tile = !compact || acc == (tn >> lbn);       // every brick live: identity mapping
  }
  // in-tile slot of work item k; `in` false for idle lanes past the last live brick
  __device__ __forceinline__ int slot(int k, bool& in) const {
    in = true;
    if (dense_tile) return k;
    const int j = k >> lbn;  // live-brick ordinal
    in = j < pre_cnt[3] + __popc(m[3]);
    int q = 3;
    if (j < pre_cnt[3]) q = 2;
    if (j < pre_cnt[2]) q = 1;
    if (j < pre_cnt[1]) q = 0;
    const uint32_t mq = q == 0 ? m[0] : (q == 1 ? m[1] : (q == 2 ? m[2] : m[3]));
    const int pq = q == 0 ? 0 : (q == 1 ? pre_cnt[1] : (q == 2 ? pre_cnt[2] : pre_cnt[3]));
    const uint32_t pos = __fns(mq, 0, j - pq + 1);
    const int b = in ? q * 32 + (int)pos : 0;
    return (b << lbn) | (k & (bn - 1));
  }
  // flag word of in-tile slot l (uniform bricks skip the load)
  __device__ __forceinline__ uint32_t flag(const uint32_t* __restrict__ flags, long long t, int tn, int l,
                                           bool in) const {
    const int bb = l >> lbn;
    const uint32_t uq = bb < 32 ? u[0] : (bb < 64 ? u[1] : (bb < 96 ? u[2] : u[3]));
    const bool uniform = in && ((uq >> (bb & 31)) & 1u);
    return uniform ? make_flag(kMaskBits, FLUID, 0, 0) : (in ? __ldg(flags + (size_t)t * tn + l) : 0u);
  }
};

// offset (from the own tile's block, excluding the direction plane) of the
// node x - c_i: neighbour tile from the shared relative-offset table,
// in-tile position from the separable brick order
struct TileUp {
  int cxm, lxm, cxp, lxp, cym, lym, cyp, lyp, czm, lzm, czp, lzp, lx0, ly0, lz0;
  __device__ __forceinline__ TileUp(const Geo& g, int l) {
    int lx, ly, lz;
    brick_inv(g, l, lx, ly, lz);
    // c = +1 pulls from l - 1, c = -1 from l + 1: (tile-code delta, in-tile offset)
    cxm = lx == 0 ? -1 : 0, lxm = brick_x(g, lx == 0 ? g.ex - 1 : lx - 1);
    cxp = lx == g.ex - 1 ? 1 : 0, lxp = brick_x(g, lx == g.ex - 1 ? 0 : lx + 1);
    cym = ly == 0 ? -3 : 0, lym = brick_y(g, ly == 0 ? g.ey - 1 : ly - 1);
    cyp = ly == g.ey - 1 ? 3 : 0, lyp = brick_y(g, ly == g.ey - 1 ? 0 : ly + 1);
    czm = lz == 0 ? -9 : 0, lzm = brick_z(g, lz == 0 ? g.ez - 1 : lz - 1);
    czp = lz == g.ez - 1 ? 9 : 0, lzp = brick_z(g, lz == g.ez - 1 ? 0 : lz + 1);
    lx0 = brick_x(g, lx), ly0 = brick_y(g, ly), lz0 = brick_z(g, lz);
  }
  __device__ __forceinline__ int code(int i) const {
    return 13 + (cx(i) == 1 ? cxm : (cx(i) == -1 ? cxp : 0)) + (cy(i) == 1 ? cym : (cy(i) == -1 ? cyp : 0)) +
           (cz(i) == 1 ? czm : (cz(i) == -1 ? czp : 0));
  }
  __device__ __forceinline__ int loc(int i) const {
    return (cx(i) == 1 ? lxm : (cx(i) == -1 ? lxp : lx0)) + (cy(i) == 1 ? lym : (cy(i) == -1 ? lyp : ly0)) +
           (cz(i) == 1 ? lzm : (cz(i) == -1 ? lzp : lz0));
  }
  __device__ __forceinline__ int at(const int* srel, int i) const { return srel[code(i)] + loc(i); }
};

// stage the 27 neighbour ranks as relative element offsets (absent: 0, i.e.
// the own tile -- such links are masked)
template <int TN>
__device__ __forceinline__ void stage_nbr(int* srel, const int* __restrict__ nbr27, int t) {
  if (threadIdx.x < 27) {
    const int v = __ldg(nbr27 + 27LL * t + threadIdx.x);
    srel[threadIdx.x] = v < 0 ? 0 : (v - t) * (Q * TN);
  }
}

// z-slab halo for tile layouts: ghost planes (5 populations x ny x nx, row
// pitch nx) per buffer.  pre_lo / pre_hi: this slab's ghosts of the pre
// buffer (filled by the neighbours' previous step); push_lo / push_hi: the
// neighbours' ghosts of the post buffer (peer memory), which this step fills
// with the c_z = -1 / +1 populations of its bottom / top plane.
template <typename T>
struct TileHalo {
  int on;
  const int* tiles;
  const T* pre_lo;   // kZp(j) populations of plane z = -1
  const T* pre_hi;   // kZm(j) populations of plane z = nz
  T* push_lo[5];     // lower neighbour's hi ghost (kZm)
  T* push_hi[5];     // upper neighbour's lo ghost (kZp)
};

template <typename T>
__device__ __forceinline__ long long ghost_row(const Geo& g, int x, int y) {
  if (x < 0) x += g.nx; else if (x >= g.nx) x -= g.nx;  // present links wrap only on periodic axes
  if (y < 0) y += g.ny; else if (y >= g.ny) y -= g.ny;
  return (long long)y * g.nx + x;
}

// links into the ghost planes replace the (meaningless) speculative values
template <typename T>
__device__ __forceinline__ void tile_ghost_gather(T (&f)[Q], uint32_t miss, const TileHalo<T>& TH, const Geo& g,
                                                  int x, int y, int z) {
  const long long pn = (long long)g.nx * g.ny;
  if (z == 0 && TH.pre_lo) {
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int i = kZp(j);
      if (!((miss >> (opp(i) - 1)) & 1u)) f[i] = __ldg(TH.pre_lo + j * pn + ghost_row<T>(g, x - cx(i), y - cy(i)));
    }
  }
  if (z == g.nz - 1 && TH.pre_hi) {
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int i = kZm(j);
      if (!((miss >> (opp(i) - 1)) & 1u)) f[i] = __ldg(TH.pre_hi + j * pn + ghost_row<T>(g, x - cx(i), y - cy(i)));
    }
  }
}

template <typename T>
__device__ __forceinline__ void tile_ghost_push(const T (&f)[Q], const TileHalo<T>& TH, const Geo& g, int x, int y,
                                                int z) {
  const long long r = (long long)y * g.nx + x;
  if (z == 0 && TH.push_lo[0]) {
#pragma unroll
    for (int j = 0; j < 5; ++j) TH.push_lo[j][r] = f[kZm(j)];
    __threadfence_system();
  }
  if (z == g.nz - 1 && TH.push_hi[0]) {
#pragma unroll
    for (int j = 0; j < 5; ++j) TH.push_hi[j][r] = f[kZp(j)];
    __threadfence_system();
  }
}

// initial ghost fill for tile layouts: boundary planes of `pre`
template <typename T>
__global__ void k_tile_halo_push(const T* __restrict__ pre, SlotMap sm, Geo g, TileHalo<T> TH) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= g.nx) return;
  const long long r = (long long)y * g.nx + x;
  const long long s0 = sm.slot(g, x, y, 0), s1 = sm.slot(g, x, y, g.nz - 1);
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    if (TH.push_lo[0]) TH.push_lo[j][r] = s0 >= 0 ? pre[fidx(g, kZm(j), s0)] : (T)0;
    if (TH.push_hi[0]) TH.push_hi[j][r] = s1 >= 0 ? pre[fidx(g, kZp(j), s1)] : (T)0;
  }
  __threadfence_system();
}

// MODE 0: speculative pull + fix-up over all TN slots; MODE 1: select per
// link (no masked link fetches a byte); MODE 2: MODE 0 over live bricks only;
// MODE 3: MODE 1 over live bricks; MODE 4: live bricks, warps whose live
// nodes all have full masks pull unconditionally, the others select per link.
template <typename T, int TN, int MODE, int MINB, bool CUT = false>
__global__ void __launch_bounds__(TN < 256 ? TN : 256, MINB)
k_step_tiles(const T* __restrict__ pre, T* __restrict__ post, const uint32_t* __restrict__ flags,
             const int* __restrict__ nbr27, const T* __restrict__ bcv, const T* __restrict__ bcr, Geo g, T om,
             const uint32_t* __restrict__ bmask, const int* __restrict__ order, const TileHalo<T> TH) {
  constexpr int BT = TN < 256 ? TN : 256;
  __shared__ int srel[27];
  const int t = order ? __ldg(order + blockIdx.x) : (int)blockIdx.x;
  stage_nbr<TN>(srel, nbr27, t);
  // z-slab cut: tiles on the first / last tile plane exchange their boundary
  // nodes' c_z populations through ghost planes (uniform per CTA)
  int tz0 = 0, tx0 = 0, ty0 = 0;
  bool cut = false;
  if (CUT) {
    tx0 = __ldg(TH.tiles + 3 * t) * g.ex;
    ty0 = __ldg(TH.tiles + 3 * t + 1) * g.ey;
    tz0 = __ldg(TH.tiles + 3 * t + 2) * g.ez;
    cut = tz0 == 0 || tz0 + g.ez >= g.nz;
  }
  const T* __restrict__ tb = pre + (size_t)t * (Q * TN);
  T* __restrict__ tp = post + (size_t)t * (Q * TN);
  constexpr bool kCompact = MODE >= 2;
  constexpr bool kSelect = MODE == 1 || MODE == 3;
  const TileBricks tw(bmask, t, g, TN, kCompact);
  __syncthreads();
#pragma unroll 1
  for (int k = threadIdx.x; k < tw.work; k += BT) {
    bool in;
    const int l = tw.slot(k, in);
    const uint32_t w = tw.flag(flags, t, TN, l, in);
    const bool live = flag_type(w) != SOLID;
    const bool zfill = sector_needs_zero<T>(live) && g.zero_fill;
    const uint32_t miss = ~w & kMaskBits;
    const bool fast = MODE == 4 ? __all_sync(0xffffffffu, !live || miss == 0u) : !kSelect;
    if (!live) {
      if (zfill && in) {
#pragma unroll
        for (int i = 0; i < Q; ++i) tp[i * TN + l] = (T)0;
      }
      continue;
    }
    const TileUp up(g, l);
    T f[Q];
    f[0] = __ldg(tb + l);
    if (fast) {
#pragma unroll
      for (int i = 1; i < Q; ++i) f[i] = __ldg(tb + i * TN + up.at(srel, i));
      if (miss) {
#pragma unroll
        for (int i = 1; i < Q; ++i)
          if ((miss >> (opp(i) - 1)) & 1u) f[i] = __ldg(tb + opp(i) * TN + l);
      }
    } else {
#pragma unroll
      for (int i = 1; i < Q; ++i)
        f[i] = __ldg(tb + (((miss >> (opp(i) - 1)) & 1u) ? opp(i) * TN + l : i * TN + up.at(srel, i)));
    }
    int x = 0, y = 0, z = -1;
    if (CUT && cut) {
      brick_inv(g, l, x, y, z);
      x += tx0;
      y += ty0;
      z += tz0;
      tile_ghost_gather<T>(f, miss, TH, g, x, y, z);
    }
    bc_collide<T>(f, w, bcv, bcr, om);
#pragma unroll
    for (int i = 0; i < Q; ++i) tp[i * TN + l] = f[i];
    if (CUT && cut) tile_ghost_push<T>(f, TH, g, x, y, z);
  }
}

// Shared-memory tile staging (MODE 6): pass 1 stages the tile's live bricks
// (each thread its own nodes' 19 values, coalesced) in shared memory; after
// one barrier, pass 2 gathers in-tile upstream values from shared memory and
// only face links from global memory (the neighbour tiles, mostly L2 hits).
// This cuts the L1 -> L2 sector traffic of the brick-shifted gathers, which
// is 2-3x the DRAM traffic in the direct kernel.
template <typename T, int TN, int MINB>
__global__ void __launch_bounds__(TN < 256 ? TN : 256, MINB)
k_step_tiles_s(const T* __restrict__ pre, T* __restrict__ post, const uint32_t* __restrict__ flags,
               const int* __restrict__ nbr27, const T* __restrict__ bcv, const T* __restrict__ bcr, Geo g, T om,
               const uint32_t* __restrict__ bmask) {
  constexpr int BT = TN < 256 ? TN : 256;
  constexpr int IT = TN / BT;  // passes per thread
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sf = reinterpret_cast<T*>(smem_raw);  // [Q][TN], same order as the tile block
  __shared__ int srel[27];
  const int t = blockIdx.x;
  stage_nbr<TN>(srel, nbr27, t);
  const T* __restrict__ tb = pre + (size_t)t * (Q * TN);
  T* __restrict__ tp = post + (size_t)t * (Q * TN);
  const TileBricks tw(bmask, t, g, TN, true);
  int ls[IT];
  uint32_t ws[IT];
  bool ins[IT];
#pragma unroll
  for (int p = 0; p < IT; ++p) {
    const int k = threadIdx.x + p * BT;
    ins[p] = false;
    ls[p] = 0;
    ws[p] = 0u;
    if (k < tw.work) {
      bool in;
      const int l = tw.slot(k, in);
      ls[p] = l;
      ins[p] = in;
      ws[p] = tw.flag(flags, t, TN, l, in);
      if (in) {
#pragma unroll
        for (int i = 0; i < Q; ++i) sf[i * TN + l] = __ldg(tb + i * TN + l);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int p = 0; p < IT; ++p) {
    const int k = threadIdx.x + p * BT;
    if (k >= tw.work) break;  // whole warps (work is a multiple of 32)
    const int l = ls[p];
    const uint32_t w = ws[p];
    const bool live = flag_type(w) != SOLID;
    const bool zfill = sector_needs_zero<T>(live) && g.zero_fill;
    if (!live) {
      if (zfill && ins[p]) {
#pragma unroll
        for (int i = 0; i < Q; ++i) tp[i * TN + l] = (T)0;
      }
      continue;
    }
    const uint32_t miss = ~w & kMaskBits;
    const TileUp up(g, l);
    T f[Q];
    f[0] = sf[l];
#pragma unroll
    for (int i = 1; i < Q; ++i) {
      const int c = up.code(i);
      // in-tile upstream (code 13) from shared memory, face links from global
      f[i] = c == 13 ? sf[i * TN + up.loc(i)] : __ldg(tb + srel[c] + i * TN + up.loc(i));
    }
    if (miss) {
#pragma unroll
      for (int i = 1; i < Q; ++i)
        if ((miss >> (opp(i) - 1)) & 1u) f[i] = sf[opp(i) * TN + l];
    }
    bc_collide<T>(f, w, bcv, bcr, om);
#pragma unroll
    for (int i = 0; i < Q; ++i) tp[i * TN + l] = f[i];
  }
}

// Warp work list (MODE 5): one warp per group of live bricks of one tile
// (32 lanes = 4 fp32 bricks), items t * 16 + g from a precomputed list, so no
// lane idles for a tile's dead bricks or its last partial pass and no CTA
// slot is held by a nearly empty tile.  The 27 neighbour offsets live in
// lanes 0-26 and are fetched with shuffles.
template <typename T, int TN, int MINB>
__global__ void __launch_bounds__(256, MINB)
k_step_tiles_w(const T* __restrict__ pre, T* __restrict__ post, const uint32_t* __restrict__ flags,
               const int* __restrict__ nbr27, const T* __restrict__ bcv, const T* __restrict__ bcr, Geo g, T om,
               const uint32_t* __restrict__ bmask, const int* __restrict__ items, int n_items) {
  const int wid = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (wid >= n_items) return;  // whole warps
  const int item = __ldg(items + wid);
  const int t = item >> 4, grp = item & 15;
  int srel = 0;
  if (lane < 27) {
    const int v = __ldg(nbr27 + 27LL * t + lane);
    srel = v < 0 ? 0 : (v - t) * (Q * TN);
  }
  const int lbn = g.lbx + g.lby + g.lbz, bn = 1 << lbn;
  // live-brick ordinal of this lane -> brick index (128-bit mask, words 0-3)
  uint32_t m[4];
  int pre_cnt[4], acc = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    m[q] = __ldg(bmask + 8LL * t + q);
    pre_cnt[q] = acc;
    acc += __popc(m[q]);
  }
  const int j = (grp << (5 - lbn)) + (lane >> lbn);
  const bool in = j < acc;
  int q = 3;
  if (j < pre_cnt[3]) q = 2;
  if (j < pre_cnt[2]) q = 1;
  if (j < pre_cnt[1]) q = 0;
  const uint32_t mq = q == 0 ? m[0] : (q == 1 ? m[1] : (q == 2 ? m[2] : m[3]));
  const int pq = q == 0 ? 0 : (q == 1 ? pre_cnt[1] : (q == 2 ? pre_cnt[2] : pre_cnt[3]));
  const int b = in ? q * 32 + (int)__fns(mq, 0, j - pq + 1) : 0;
  const int l = (b << lbn) | (lane & (bn - 1));
  const uint32_t uq = __ldg(bmask + 8LL * t + 4 + (b >> 5));
  const bool uniform = in && ((uq >> (b & 31)) & 1u);
  const uint32_t w = uniform ? make_flag(kMaskBits, FLUID, 0, 0) : (in ? __ldg(flags + (size_t)t * TN + l) : 0u);
  const bool live = flag_type(w) != SOLID;
  const bool zfill = sector_needs_zero<T>(live) && g.zero_fill;
  const T* __restrict__ tb = pre + (size_t)t * (Q * TN);
  T* __restrict__ tp = post + (size_t)t * (Q * TN);
  // every lane must take part in the shuffles: dead lanes compute garbage
  // addresses they never use
  const TileUp up(g, l);
  int off[Q];
#pragma unroll
  for (int i = 1; i < Q; ++i) off[i] = __shfl_sync(0xffffffffu, srel, up.code(i)) + up.loc(i);
  if (!live) {
    if (zfill && in) {
#pragma unroll
      for (int i = 0; i < Q; ++i) tp[i * TN + l] = (T)0;
    }
    return;
  }
  const uint32_t miss = ~w & kMaskBits;
  T f[Q];
  f[0] = __ldg(tb + l);
#pragma unroll
  for (int i = 1; i < Q; ++i) f[i] = __ldg(tb + i * TN + off[i]);
  if (miss) {
#pragma unroll
    for (int i = 1; i < Q; ++i)
      if ((miss >> (opp(i) - 1)) & 1u) f[i] = __ldg(tb + opp(i) * TN + l);
  }
  bc_collide<T>(f, w, bcv, bcr, om);
#pragma unroll
  for (int i = 0; i < Q; ++i) tp[i * TN + l] = f[i];
}

// A-A in place over the tile list (see k_step_dense_aa for the scheme):
// NB = 1 pulls F[opp(i)] at x - c_i and pushes to F[i] at x + c_i through
// the neighbour table; NB = 0 is node-local.
template <typename T, int TN, int NB, int MINB>
__global__ void __launch_bounds__(TN < 256 ? TN : 256, MINB)
k_step_tiles_aa(T* __restrict__ F, const uint32_t* __restrict__ flags, const int* __restrict__ nbr27,
                const T* __restrict__ bcv, const T* __restrict__ bcr, Geo g, T om,
                const uint32_t* __restrict__ bmask, const int* __restrict__ order) {
  constexpr int BT = TN < 256 ? TN : 256;
  __shared__ int srel[27];
  const int t = order ? __ldg(order + blockIdx.x) : (int)blockIdx.x;
  if (NB) stage_nbr<TN>(srel, nbr27, t);
  T* __restrict__ tb = F + (size_t)t * (Q * TN);
  const TileBricks tw(bmask, t, g, TN, true);
  if (NB) __syncthreads();
#pragma unroll 1
  for (int k = threadIdx.x; k < tw.work; k += BT) {
    bool in;
    const int l = tw.slot(k, in);
    const uint32_t w = tw.flag(flags, t, TN, l, in);
    if (flag_type(w) == SOLID) continue;  // no zero-fill under AA (see k_step_dense_aa)
    const uint32_t miss = ~w & kMaskBits;
    T f[Q];
    f[0] = LDA(tb + l);
    if (NB) {
      const TileUp up(g, l);
#pragma unroll
      for (int i = 1; i < Q; ++i) f[i] = LDA(tb + opp(i) * TN + up.at(srel, i));
      if (miss) {
#pragma unroll
        for (int i = 1; i < Q; ++i)
          if ((miss >> (opp(i) - 1)) & 1u) f[i] = LDA(tb + i * TN + l);
      }
      bc_collide<T>(f, w, bcv, bcr, om);
      const int l2 = opaque(l);
      const TileUp up2(g, l2);
      tb[l2] = f[0];
#pragma unroll
      for (int i = 1; i < Q; ++i)
        tb[((miss >> (i - 1)) & 1u) ? opp(i) * TN + l2 : i * TN + up2.at(srel, opp(i))] = f[i];
    } else {
#pragma unroll
      for (int i = 1; i < Q; ++i) f[i] = LDA(tb + i * TN + l);
      bc_collide<T>(f, w, bcv, bcr, om);
#pragma unroll
      for (int i = 0; i < Q; ++i) tb[opp(i) * TN + l] = f[i];
    }
  }
}

// ----------------------------------------------------------------- handle
struct lbm_handle {
  lbm_desc d{};
  int esize = 4;
  Geo g{};
  SlotMap sm{nullptr};
  long long n_nodes = 0, n_slots = 0, nflags = 0;
  long long n_tiles = 0, ntiles_grid = 0;
  long long n_nonsolid = 0;
  void* f[2] = {nullptr, nullptr};
  uint32_t* flags = nullptr;
  int* rank = nullptr;    // tile rank grid
  int* tiles = nullptr;   // (T, 3)
  int* nbr27 = nullptr;   // (T, 27)
  int* order = nullptr;   // (T) CTA -> tile rank launch order (Morton), or null (rank order)
  void* gh[2] = {nullptr, nullptr};  // tile slabs: ghost planes per buffer, [lo | hi] x 5 x ny x nx
  int* items = nullptr;   // warp work list (tile << 4 | live-brick group), MODE 5
  int n_items = 0;
  bool has_glo = false, has_ghi = false;  // tile slabs: links cross z = -1 / z = nz
  int order_mode = 0;     // 0 rank order, 1 Morton, 2 y-pencils of `pencil` tile rows, 3 z-groups of `pencil` layers
  int pencil = 4;
  uint32_t* bmask = nullptr;  // (T, 4) live-brick bit masks
  uint32_t* ubits = nullptr;  // dense: uniform-chunk bitmap (1 bit per 32 nodes)
  bool use_ubits = true;
  long long meta_bytes = 0;   // flag / index bytes one step reads
  void* bcv = nullptr;    // (nb, 3) storage type
  void* bcr = nullptr;    // (nb) storage type
  uint8_t* bckind64 = nullptr;
  double* bcv64 = nullptr;
  double* bcr64 = nullptr;
  int nb = 0;
  int parity = 0;
  int variant = 0;  // step-kernel variant (LBM_STEP_VARIANT), see launch_step
  bool geometry = false, initialized = false;
  long long step_count = 0, visited_total = 0, launches = 0;
  long long device_bytes = 0;
  double last_ms = 0.0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  void* pin[2] = {nullptr, nullptr};   // pinned host staging for pipelined readbacks
  size_t pin_bytes = 0;
  cudaEvent_t evc[2] = {nullptr, nullptr};
  double* scratch = nullptr;   // reductions
  unsigned long long* uscratch = nullptr;
  // z-slab halo (fused peer stores); see k_step_dense and lbm_halo_connect
  struct Peer {
    bool on = false, ipc = false;
    void* f[2] = {nullptr, nullptr};
    unsigned long long* sync = nullptr;
    long long ps = 0;
    int nz = 0;
  } lo, hi;
  unsigned long long* sync = nullptr;  // [0] written by the lower, [1] by the upper neighbour
  int* herr = nullptr;
  unsigned long long epoch = 0;        // halo pushes done by this handle
  bool halo_dirty = true;
  bool pending = false;                // lbm_step_async issued, not yet synchronised
  cudaGraphExec_t graph[2] = {nullptr, nullptr};  // kGraphSteps steps from parity 0 / 1
  bool use_graph = true;
};

constexpr int kGraphSteps = 32;

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int ilog2(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  return l;
}

template <typename P>
int dev_alloc(lbm_handle* h, P** p, size_t bytes) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, bytes ? bytes : 16);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? LBM_ENOMEM : LBM_ECUDA,
                "cudaMalloc(%zu bytes): %s", bytes, cudaGetErrorString(e));
  }
  h->device_bytes += (long long)bytes;
  *p = (P*)q;
  return 0;
}

void dev_free(void* p) {
  if (p) cudaFree(p);
}

void drop_graphs(lbm_handle* h) {
  for (int p = 0; p < 2; ++p)
    if (h->graph[p]) {
      cudaGraphExecDestroy(h->graph[p]);
      h->graph[p] = nullptr;
    }
}

void free_geometry(lbm_handle* h) {
  drop_graphs(h);
  dev_free(h->f[0]);
  dev_free(h->f[1]);
  dev_free(h->flags);
  dev_free(h->rank);
  dev_free(h->tiles);
  dev_free(h->nbr27);
  dev_free(h->order);
  dev_free(h->items);
  h->items = nullptr;
  h->n_items = 0;
  dev_free(h->gh[0]);
  dev_free(h->gh[1]);
  h->gh[0] = h->gh[1] = nullptr;
  dev_free(h->bmask);
  dev_free(h->ubits);
  dev_free(h->bcv);
  dev_free(h->bcr);
  dev_free(h->bckind64);
  dev_free(h->bcv64);
  dev_free(h->bcr64);
  h->f[0] = h->f[1] = nullptr;
  h->flags = nullptr;
  h->rank = h->tiles = h->nbr27 = h->order = nullptr;
  h->bmask = nullptr;
  h->ubits = nullptr;
  h->bcv = h->bcr = nullptr;
  h->bckind64 = nullptr;
  h->bcv64 = h->bcr64 = nullptr;
  h->device_bytes = 0;
  h->geometry = h->initialized = false;
}

bool is_tiled(int layout) { return layout == LBM_LAYOUT_TILE || layout == LBM_LAYOUT_POINTER_TILE; }

dim3 node_grid(const Geo& g, int bx) { return dim3((g.nx + bx - 1) / bx, g.ny, g.nz); }

// peer ghost planes of buffer q (lockstep: every slab is at the same parity)
template <typename T>
Halo<T> make_halo(const lbm_handle* h, int q) {
  Halo<T> H;
  for (int j = 0; j < 5; ++j) {
    H.lo[j] = h->lo.on ? (T*)h->lo.f[q] + (size_t)kZm(j) * h->lo.ps + (size_t)(h->lo.nz + 1) * h->g.plane
                       : nullptr;
    H.hi[j] = h->hi.on ? (T*)h->hi.f[q] + (size_t)kZp(j) * h->hi.ps : nullptr;
  }
  return H;
}

template <typename T>
TileHalo<T> make_tile_halo(const lbm_handle* h, int q_pre, int q_post) {
  TileHalo<T> TH{};
  TH.on = h->g.tiled && h->gh[0] != nullptr;
  if (!TH.on) return TH;
  const size_t pn = (size_t)h->g.nx * h->g.ny;
  TH.tiles = h->tiles;
  TH.pre_lo = h->has_glo ? (const T*)h->gh[q_pre] : nullptr;
  TH.pre_hi = h->has_ghi ? (const T*)h->gh[q_pre] + 5 * pn : nullptr;
  for (int j = 0; j < 5; ++j) {
    TH.push_lo[j] = h->lo.on ? (T*)h->lo.f[q_post] + (5 + j) * pn : nullptr;
    TH.push_hi[j] = h->hi.on ? (T*)h->hi.f[q_post] + j * pn : nullptr;
  }
  return TH;
}

bool halo_on(const lbm_handle* h) { return h->lo.on || h->hi.on; }

// buffer holding the reference's `pre` (AA: the single in-place buffer)
void* pre_buf(const lbm_handle* h) { return h->g.aa ? h->f[0] : h->f[h->parity]; }

// Geo for readback launches: carries the AA state phase
Geo rb_geo(const lbm_handle* h) {
  Geo g = h->g;
  g.aph = h->g.aa ? h->parity : 0;
  return g;
}

long long visits_per_step(const lbm_handle* h) {
  return (h->d.layout == LBM_LAYOUT_DENSE) ? h->n_nodes
         : (h->d.layout == LBM_LAYOUT_BITMASK_NODE) ? h->n_nonsolid
                                                     : h->n_slots;
}

void halo_signal(lbm_handle* h) {
  h->epoch += 1;
  h->launches += 1;
  k_halo_signal<<<1, 1, 0, h->stream>>>(h->lo.on ? h->lo.sync + 1 : nullptr,
                                         h->hi.on ? h->hi.sync + 0 : nullptr, h->epoch);
}

void halo_wait(lbm_handle* h) {
  h->launches += 1;
  k_halo_wait<<<1, 1, 0, h->stream>>>(h->sync, h->lo.on, h->hi.on, h->epoch, h->herr);
}

template <typename T>
void halo_push(lbm_handle* h) {
  if (h->g.tiled) {
    const TileHalo<T> TH = make_tile_halo<T>(h, h->parity, h->parity);
    h->launches += 1;
    k_tile_halo_push<T><<<dim3((h->g.nx + 127) / 128, h->g.ny), 128, 0, h->stream>>>((const T*)h->f[h->parity], h->sm,
                                                                                     h->g, TH);
    return;
  }
  const Halo<T> H = make_halo<T>(h, h->parity);
  h->launches += 1;
  dim3 grid((h->g.nxp + 127) / 128, h->g.ny);
  k_halo_push<T><<<grid, 128, 0, h->stream>>>((const T*)h->f[h->parity], H, h->g);
}

template <typename T, int TN>
void launch_tiles(lbm_handle* h, const T* pre, T* post, int var) {
  constexpr int BT = TN < 256 ? TN : 256;
  const TileHalo<T> TH = make_tile_halo<T>(h, h->parity, 1 - h->parity);
  constexpr int M = sizeof(T) == 4 ? (1536 / BT > 32 ? 32 : 1536 / BT) : (768 / BT);
  const unsigned nt = (unsigned)h->n_tiles;
  const T* bv = (const T*)h->bcv;
  const T* br = (const T*)h->bcr;
  const T om = (T)h->d.omega;
  if (TH.on) {  // z-slab: the live-brick kernel with the ghost-plane exchange
    k_step_tiles<T, TN, 2, (M * 5 / 6 > 0 ? M * 5 / 6 : 1), true><<<nt, BT, 0, h->stream>>>(
        pre, post, h->flags, h->nbr27, bv, br, h->g, om,
                                                               h->bmask, h->order, TH);
    return;
  }
  // the select variants need more registers than the speculative gather
  constexpr int MS = M * 5 / 6 > 0 ? M * 5 / 6 : 1;
  if (var == 6) {
    constexpr int SMEM = Q * TN * (int)sizeof(T);
    constexpr int MSM = (200 * 1024) / (SMEM + 512) > 0 ? (200 * 1024) / (SMEM + 512) : 1;
    constexpr int MB = MSM < M ? MSM : M;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_step_tiles_s<T, TN, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
      attr = true;
    }
    k_step_tiles_s<T, TN, MB><<<nt, BT, SMEM, h->stream>>>(pre, post, h->flags, h->nbr27, bv, br, h->g, om, h->bmask);
    return;
  }
  if (var == 5) {
    constexpr int MW = sizeof(T) == 4 ? 6 : 3;
    if (h->n_items)
      k_step_tiles_w<T, TN, MW><<<(unsigned)((h->n_items + 7) / 8), 256, 0, h->stream>>>(
          pre, post, h->flags, h->nbr27, bv, br, h->g, om, h->bmask, h->items, h->n_items);
    return;
  }
  if (var == 3)
    k_step_tiles<T, TN, 3, MS><<<nt, BT, 0, h->stream>>>(pre, post, h->flags, h->nbr27, bv, br, h->g, om, h->bmask, h->order, TH);
  else if (var == 4)
    k_step_tiles<T, TN, 4, MS><<<nt, BT, 0, h->stream>>>(pre, post, h->flags, h->nbr27, bv, br, h->g, om, h->bmask, h->order, TH);
  else if (var == 1)
    k_step_tiles<T, TN, 1, M><<<nt, BT, 0, h->stream>>>(pre, post, h->flags, h->nbr27, bv, br, h->g, om, h->bmask, h->order, TH);
  else if (var == 2)
    k_step_tiles<T, TN, 0, M><<<nt, BT, 0, h->stream>>>(pre, post, h->flags, h->nbr27, bv, br, h->g, om, h->bmask, h->order, TH);
  else
    k_step_tiles<T, TN, 2, M><<<nt, BT, 0, h->stream>>>(pre, post, h->flags, h->nbr27, bv, br, h->g, om, h->bmask, h->order, TH);
}

template <typename T, int TN>
void launch_tiles_aa(lbm_handle* h, T* F) {
  constexpr int BT = TN < 256 ? TN : 256;
  constexpr int M = sizeof(T) == 4 ? (1536 / BT > 32 ? 32 : 1536 / BT) : (768 / BT);
  const unsigned nt = (unsigned)h->n_tiles;
  const T* bv = (const T*)h->bcv;
  const T* br = (const T*)h->bcr;
  const T om = (T)h->d.omega;
  constexpr int MN = M * 5 / 6 > 0 ? M * 5 / 6 : 1;  // neighbour step: looser register cap
  if (h->parity == 0)
    k_step_tiles_aa<T, TN, 1, MN><<<nt, BT, 0, h->stream>>>(F, h->flags, h->nbr27, bv, br, h->g, om, h->bmask, h->order);
  else
    k_step_tiles_aa<T, TN, 0, M><<<nt, BT, 0, h->stream>>>(F, h->flags, h->nbr27, bv, br, h->g, om, h->bmask, h->order);
}

// one step from `pre` into `post` (AB); AA updates `post` (== pre) in place
template <typename T>
int launch_step(lbm_handle* h, const void* pre, void* post) {
  const Geo& g = h->g;
  const T om = (T)h->d.omega;
  Planes<T> P;
  for (int i = 0; i < Q; ++i) {
    P.pre[i] = (const T*)pre + (size_t)i * g.ps;
    P.post[i] = (T*)post + (size_t)i * g.ps;
  }
  // variants (LBM_STEP_VARIANT): 0 speculative + fix-up, 1 warp-uniform
  // fast path else per-link select; 2 / 3 the same with a looser register cap
  const int var = h->variant;
  constexpr int D1 = sizeof(T) == 4 ? 12 : 6, D2 = sizeof(T) == 4 ? 10 : 5;
  const T* bv = (const T*)h->bcv;
  const T* br = (const T*)h->bcr;
  if (g.aa) {
    // parity = AA state phase: 0 -> neighbour step, 1 -> node-local step
    if (!g.tiled) {
      Planes1<T> F;
      for (int i = 0; i < Q; ++i) F.f[i] = (T*)post + (size_t)i * g.ps;
      dim3 grid((g.nxp + 127) / 128, g.ny, g.nz);
      if (h->parity == 0)
        k_step_dense_aa<T, 1, D1><<<grid, 128, 0, h->stream>>>(F, h->flags, h->ubits, bv, br, g, om);
      else
        k_step_dense_aa<T, 0, D1><<<grid, 128, 0, h->stream>>>(F, h->flags, h->ubits, bv, br, g, om);
    } else {
      if (h->n_tiles == 0) return 0;
      switch (g.tn) {
        case 32: launch_tiles_aa<T, 32>(h, (T*)post); break;
        case 64: launch_tiles_aa<T, 64>(h, (T*)post); break;
        case 128: launch_tiles_aa<T, 128>(h, (T*)post); break;
        case 256: launch_tiles_aa<T, 256>(h, (T*)post); break;
        default: launch_tiles_aa<T, 512>(h, (T*)post); break;
      }
    }
    h->launches += 1;
    return 0;
  }
  if (!g.tiled) {
    const int bx = 128;
    dim3 grid((g.nxp + bx - 1) / bx, g.ny, g.nz);
    const Halo<T> H = make_halo<T>(h, 1 - h->parity);
    if (var == 1)
      k_step_dense<T, 1, D1><<<grid, bx, 0, h->stream>>>(P, h->flags, h->ubits, bv, br, g, om, H);
    else if (var == 2)
      k_step_dense<T, 0, D2><<<grid, bx, 0, h->stream>>>(P, h->flags, h->ubits, bv, br, g, om, H);
    else if (var == 3)
      k_step_dense<T, 1, D2><<<grid, bx, 0, h->stream>>>(P, h->flags, h->ubits, bv, br, g, om, H);
    else
      k_step_dense<T, 0, D1><<<grid, bx, 0, h->stream>>>(P, h->flags, h->ubits, bv, br, g, om, H);
  } else {
    if (h->n_tiles == 0) return 0;
    switch (g.tn) {
      case 32: launch_tiles<T, 32>(h, (const T*)pre, (T*)post, var); break;
      case 64: launch_tiles<T, 64>(h, (const T*)pre, (T*)post, var); break;
      case 128: launch_tiles<T, 128>(h, (const T*)pre, (T*)post, var); break;
      case 256: launch_tiles<T, 256>(h, (const T*)pre, (T*)post, var); break;
      default: launch_tiles<T, 512>(h, (const T*)pre, (T*)post, var); break;
    }
  }
  h->launches += 1;
  return 0;
}

// CUDA lazy module loading loads a kernel at its first launch, and loading
// waits for the device: with a neighbour's k_halo_wait spinning, that first
// launch would stall until the wait times out.  A slab therefore loads every
// kernel its step loop can launch when it is connected, before any spins.
template <typename T, int TN>
void preload_tiles(cudaFuncAttributes* a) {
  constexpr int BT = TN < 256 ? TN : 256;
  constexpr int M = sizeof(T) == 4 ? (1536 / BT > 32 ? 32 : 1536 / BT) : (768 / BT);
  cudaFuncGetAttributes(a, k_step_tiles<T, TN, 2, (M * 5 / 6 > 0 ? M * 5 / 6 : 1), true>);
}

template <typename T>
void preload_halo_kernels(const lbm_handle* h) {
  constexpr int D1 = sizeof(T) == 4 ? 12 : 6, D2 = sizeof(T) == 4 ? 10 : 5;
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_halo_wait);
  cudaFuncGetAttributes(&a, k_halo_signal);
  if (!h->g.tiled) {
    cudaFuncGetAttributes(&a, k_halo_push<T>);
    cudaFuncGetAttributes(&a, k_step_dense<T, 0, D1>);
    cudaFuncGetAttributes(&a, k_step_dense<T, 1, D1>);
    cudaFuncGetAttributes(&a, k_step_dense<T, 0, D2>);
    cudaFuncGetAttributes(&a, k_step_dense<T, 1, D2>);
  } else {
    cudaFuncGetAttributes(&a, k_tile_halo_push<T>);
    switch (h->g.tn) {
      case 32: preload_tiles<T, 32>(&a); break;
      case 64: preload_tiles<T, 64>(&a); break;
      case 128: preload_tiles<T, 128>(&a); break;
      case 256: preload_tiles<T, 256>(&a); break;
      default: preload_tiles<T, 512>(&a); break;
    }
  }
  cudaGetLastError();
}

}  // namespace

// ================================================================= C-ABI
extern "C" {

const char* lbm_last_error(void) { return g_err.c_str(); }
int lbm_abi_version(void) { return LBM_ABI_VERSION; }

int lbm_device_count(int* n) {
  if (!n) return fail(LBM_EINVAL, "n is NULL");
  CK(cudaGetDeviceCount(n));
  return 0;
}

int lbm_create(const lbm_desc* desc, lbm_t** out) {
  if (!desc || !out) return fail(LBM_EINVAL, "desc/out is NULL");
  const lbm_desc& d = *desc;
  if (d.nx <= 0 || d.ny <= 0 || d.nz <= 0)
    return fail(LBM_EINVAL, "dims must be positive, got (%d, %d, %d)", d.nx, d.ny, d.nz);
  if (d.dtype != LBM_F32 && d.dtype != LBM_F64) return fail(LBM_EINVAL, "dtype must be LBM_F32 or LBM_F64");
  if (d.layout < 0 || d.layout > LBM_LAYOUT_POINTER_TILE) return fail(LBM_EINVAL, "unknown layout %d", d.layout);
  if (!(d.omega > 0.0 && d.omega < 2.0)) return fail(LBM_EINVAL, "omega must lie in (0, 2), got %g", d.omega);
  if (d.scheme != LBM_SCHEME_AB && d.scheme != LBM_SCHEME_AA) return fail(LBM_EINVAL, "unknown scheme %d", d.scheme);
  const int nzg = d.nz_global > 0 ? d.nz_global : d.nz;
  if (d.z0 < 0 || d.z0 + d.nz > nzg) return fail(LBM_EINVAL, "slab [%d, %d) outside nz_global %d", d.z0, d.z0 + d.nz, nzg);
  if (!is_tiled(d.layout) && (long long)(d.nz + 2) * d.ny * ((d.nx + 31) / 32 * 32) + 64 >= (1LL << 32))
    return fail(LBM_EINVAL, "dense slab of %d x %d x %d nodes exceeds 2^32 slots; split it into z-slabs", d.nx, d.ny, d.nz);
  if (is_tiled(d.layout)) {
    for (int a = 0; a < 3; ++a) {
      const int e = d.tile[a];
      if (e < 1 || (e & (e - 1))) return fail(LBM_EINVAL, "tile edges must be powers of two, got %d", e);
    }
    if (d.tile[0] * d.tile[1] * d.tile[2] > 512 || d.tile[0] * d.tile[1] * d.tile[2] < 32)
      return fail(LBM_EINVAL, "tile must hold 32..512 nodes");
    const int n3[3] = {d.nx, d.ny, d.nz};
    for (int a = 0; a < 3; ++a)
      if (d.periodic[a] && n3[a] % d.tile[a])
        return fail(LBM_EINVAL, "periodic axis %d needs extent %d divisible by the tile edge %d", a, n3[a], d.tile[a]);
  }
  if (d.scheme == LBM_SCHEME_AA && nzg != d.nz) return fail(LBM_EINVAL, "the AA scheme is single-slab in this build");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (d.device < 0 || d.device >= ndev) return fail(LBM_EINVAL, "device %d not present (%d devices)", d.device, ndev);
  DeviceGuard dg(d.device);
  lbm_handle* h = new lbm_handle();
  h->d = d;
  h->d.nz_global = nzg;
  h->esize = d.dtype == LBM_F32 ? 4 : 8;
  Geo& g = h->g;
  g.nx = d.nx;
  g.ny = d.ny;
  g.nz = d.nz;
  g.px = d.periodic[0] != 0;
  g.py = d.periodic[1] != 0;
  g.pzw = (d.periodic[2] != 0) && (nzg == d.nz);
  g.tiled = is_tiled(d.layout);
  g.aa = d.scheme == LBM_SCHEME_AA;
  {
    const char* zf = getenv("LBM_ZERO_FILL");  // A/B switch for the sector-completion stores
    g.zero_fill = (zf && zf[0] == '0') ? 0 : 1;
    const char* sv = getenv("LBM_STEP_VARIANT");
    h->variant = sv ? atoi(sv) : 0;
    const char* ub = getenv("LBM_UBITS");
    h->use_ubits = !(ub && ub[0] == '0');
    const char* to = getenv("LBM_TILE_ORDER");  // "row": launch tiles in rank order
    // "morton" | "pencil[:B]" | "row" (rank order)
    h->order_mode = !to ? 0 : to[0] == 'm' ? 1 : to[0] == 'p' ? 2 : to[0] == 'z' ? 3 : 0;
    if (to && strchr(to, ':')) h->pencil = atoi(strchr(to, ':') + 1) > 0 ? atoi(strchr(to, ':') + 1) : 4;
    const char* gv = getenv("LBM_GRAPH");
    h->use_graph = !(gv && gv[0] == '0');
  }
  h->n_nodes = (long long)d.nx * d.ny * d.nz;
  if (!g.tiled) {
    g.nxp = (d.nx + 31) / 32 * 32;
    g.plane = (long long)g.ny * g.nxp;
    h->n_slots = (long long)(g.nz + 2) * g.plane;
    g.ps = (h->n_slots + 63) / 64 * 64;
    h->nflags = (long long)g.nz * g.plane;
  } else {
    g.ex = d.tile[0];
    g.ey = d.tile[1];
    g.ez = d.tile[2];
    g.lex = ilog2(g.ex);
    g.ley = ilog2(g.ey);
    g.lez = ilog2(g.ez);
    {
      // one 32-B sector per brick: 2x2x2 fp32, 2x2x1 fp64 (LBM_BRICK=0: x-rows)
      const char* bv = getenv("LBM_BRICK");
      const bool rows = bv && bv[0] == '0';
      const int want = d.dtype == LBM_F32 ? 3 : 2;  // log2(nodes per sector)
      int b[3] = {0, 0, 0}, left = want;
      if (rows) {
        b[0] = want < g.lex ? want : g.lex;
      } else {
        for (int a = 0; left > 0 && a < 3 * 4; ++a) {
          const int ax = a % 3, lim = ax == 0 ? g.lex : (ax == 1 ? g.ley : g.lez);
          if (b[ax] < lim) { ++b[ax]; --left; }
        }
      }
      g.lbx = b[0];
      g.lby = b[1];
      g.lbz = b[2];
    }
    g.gx = (d.nx + g.ex - 1) / g.ex;
    g.gy = (d.ny + g.ey - 1) / g.ey;
    g.gz = (d.nz + g.ez - 1) / g.ez;
    g.tn = g.ex * g.ey * g.ez;
    g.ltn = ilog2(g.tn);
    g.nxp = d.nx;
    h->ntiles_grid = (long long)g.gx * g.gy * g.gz;
  }
  cudaError_t e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&h->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&h->ev1);
  if (e == cudaSuccess) e = cudaMalloc(&h->scratch, 4096 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&h->uscratch, 4 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&h->sync, 2 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(h->sync, 0, 2 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&h->herr, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(h->herr, 0, sizeof(int));
  if (e != cudaSuccess) {
    lbm_destroy(h);
    return fail(LBM_ECUDA, "stream/event setup: %s", cudaGetErrorString(e));
  }
  *out = h;
  return 0;
}

void lbm_destroy(lbm_t* h) {
  if (!h) return;
  DeviceGuard dg(h->d.device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (lbm_handle::Peer* pr : {&h->lo, &h->hi}) {
    if (pr->on && pr->ipc) {
      cudaIpcCloseMemHandle(pr->f[0]);
      cudaIpcCloseMemHandle(pr->f[1]);
      cudaIpcCloseMemHandle(pr->sync);
    }
    pr->on = false;
  }
  free_geometry(h);
  dev_free(h->scratch);
  dev_free(h->uscratch);
  dev_free(h->sync);
  dev_free(h->herr);
  for (int b = 0; b < 2; ++b) {
    if (h->pin[b]) cudaFreeHost(h->pin[b]);
    if (h->evc[b]) cudaEventDestroy(h->evc[b]);
  }
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

// LBM_TIMING=1: phase times of lbm_set_geometry on stderr (device synchronised)
struct PhaseTimer {
  bool on = false;
  cudaStream_t st = nullptr;
  std::chrono::steady_clock::time_point t0;
  explicit PhaseTimer(cudaStream_t s) : st(s) {
    const char* v = getenv("LBM_TIMING");
    on = v && v[0] == '1';
    t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[lbm timing] %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

int lbm_set_geometry(lbm_t* h, const uint8_t* type, const uint8_t* orient, const int32_t* bc_index,
                     const uint8_t* ghost_lo, const uint8_t* ghost_hi, const uint8_t* bc_kind,
                     const double* bc_vel, const double* bc_rho, int32_t nb) {
  if (!h || !type || !orient || !bc_index) return fail(LBM_EINVAL, "NULL geometry array");
  if (nb < 0 || nb > 255) return fail(LBM_EINVAL, "boundary table holds %d entries; at most 255 supported", nb);
  if (nb > 0 && (!bc_kind || !bc_vel || !bc_rho)) return fail(LBM_EINVAL, "NULL boundary table");
  DeviceGuard dg(h->d.device);
  CK(cudaStreamSynchronize(h->stream));
  free_geometry(h);
  Geo& g = h->g;
  const long long N = h->n_nodes;
  const long long plane_nodes = (long long)g.nx * g.ny;
  int rc = 0;
  uint8_t *dtype_ = nullptr, *dorient = nullptr, *dglo = nullptr, *dghi = nullptr;
  int* dbc = nullptr;
  int* derr = nullptr;
  int *keep = nullptr, *scan = nullptr;
  void* cub_tmp = nullptr;
  const int nbt = nb > 0 ? nb : 1;
  PhaseTimer pt(h->stream);
  // temporaries
  if ((rc = dev_alloc(h, &dtype_, N)) || (rc = dev_alloc(h, &dorient, N)) ||
      (rc = dev_alloc(h, &dbc, N * 4)) || (rc = dev_alloc(h, &derr, 16)))
    goto done;
  pt.mark("alloc temporaries");
  CK(cudaMemcpyAsync(dtype_, type, N, cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemcpyAsync(dorient, orient, N, cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemcpyAsync(dbc, bc_index, N * 4, cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemsetAsync(derr, 0, 16, h->stream));
  CK(cudaMemsetAsync(h->uscratch, 0, 4 * sizeof(unsigned long long), h->stream));
  if (ghost_lo) {
    if ((rc = dev_alloc(h, &dglo, plane_nodes))) goto done;
    CK(cudaMemcpyAsync(dglo, ghost_lo, plane_nodes, cudaMemcpyHostToDevice, h->stream));
  } else if (g.pzw) {
    dglo = nullptr;  // wrap handled below
  }
  if (ghost_hi) {
    if ((rc = dev_alloc(h, &dghi, plane_nodes))) goto done;
    CK(cudaMemcpyAsync(dghi, ghost_hi, plane_nodes, cudaMemcpyHostToDevice, h->stream));
  }
  {
    // whole-domain periodic z: the ghost planes are the wrapped planes
    const uint8_t* glo = dglo ? dglo : (g.pzw ? dtype_ + (long long)(g.nz - 1) * plane_nodes : nullptr);
    const uint8_t* ghi = dghi ? dghi : (g.pzw ? dtype_ : nullptr);
    // boundary tables (float64 for init, storage type for the step)
    if ((rc = dev_alloc(h, &h->bckind64, nbt)) || (rc = dev_alloc(h, &h->bcv64, nbt * 3 * 8)) ||
        (rc = dev_alloc(h, &h->bcr64, nbt * 8)) || (rc = dev_alloc(h, (char**)&h->bcv, nbt * 3 * h->esize)) ||
        (rc = dev_alloc(h, (char**)&h->bcr, nbt * h->esize)))
      goto done;
    {
      std::vector<uint8_t> kk(nbt, 0);
      std::vector<double> vv(nbt * 3, 0.0), rr(nbt, 0.0);
      for (int b = 0; b < nb; ++b) {
        kk[b] = bc_kind[b];
        for (int c = 0; c < 3; ++c) vv[3 * b + c] = bc_vel[3 * b + c];
        rr[b] = bc_rho[b];
      }
      CK(cudaMemcpy(h->bckind64, kk.data(), nbt, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(h->bcv64, vv.data(), nbt * 3 * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(h->bcr64, rr.data(), nbt * 8, cudaMemcpyHostToDevice));
      if (h->esize == 4) {
        std::vector<float> vf(nbt * 3), rf(nbt);
        for (int k = 0; k < nbt * 3; ++k) vf[k] = (float)vv[k];
        for (int k = 0; k < nbt; ++k) rf[k] = (float)rr[k];
        CK(cudaMemcpy(h->bcv, vf.data(), nbt * 3 * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->bcr, rf.data(), nbt * 4, cudaMemcpyHostToDevice));
      } else {
        CK(cudaMemcpy(h->bcv, vv.data(), nbt * 3 * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->bcr, rr.data(), nbt * 8, cudaMemcpyHostToDevice));
      }
    }
    if (!g.tiled) {
      if ((rc = dev_alloc(h, &h->flags, h->nflags * 4))) goto done;
      dim3 grid((g.nxp + 127) / 128, g.ny, g.nz);
      k_flags_dense<<<grid, 128, 0, h->stream>>>(h->flags, dtype_, dorient, dbc, glo, ghi, g, nb, derr,
                                                 h->uscratch);
      CKL();
      const long long nwords = (h->nflags + 1023) / 1024;
      if ((rc = dev_alloc(h, &h->ubits, nwords * 4))) goto done;
      CK(cudaMemsetAsync(h->ubits, 0, nwords * 4, h->stream));
      if (h->use_ubits) {
        k_uniform_bits<<<(unsigned)((h->nflags + 255) / 256), 256, 0, h->stream>>>(h->ubits, h->flags, h->nflags);
        CKL();
      }
      {
        std::vector<uint32_t> hb(nwords);
        CK(cudaMemcpyAsync(hb.data(), h->ubits, nwords * 4, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        long long uni = 0;
        for (uint32_t v : hb) uni += __builtin_popcount(v);
        // the step reads the bitmap plus the flag words of non-uniform chunks
        h->meta_bytes = nwords * 4 + (h->nflags - 32 * uni) * 4;
      }
    } else {
      const long long G = h->ntiles_grid;
      if ((rc = dev_alloc(h, &h->rank, G * 4)) || (rc = dev_alloc(h, &keep, G * 4)) ||
          (rc = dev_alloc(h, &scan, G * 4)))
        goto done;
      const int keep_all = h->d.layout == LBM_LAYOUT_TILE;
      pt.mark("upload descriptors");
      k_tile_keep<<<(unsigned)((G * 32 + 255) / 256), 256, 0, h->stream>>>(keep, dtype_, g, keep_all, G);
      CKL();
      size_t tmp_bytes = 0;
      if (G > 0x7fffffffLL) { rc = fail(LBM_EINVAL, "too many tiles"); goto done; }
      CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, keep, scan, (int)G, h->stream));
      if ((rc = dev_alloc(h, (char**)&cub_tmp, tmp_bytes))) goto done;
      CK(cub::DeviceScan::ExclusiveSum(cub_tmp, tmp_bytes, keep, scan, (int)G, h->stream));
      int last_scan = 0, last_keep = 0;
      CK(cudaMemcpyAsync(&last_scan, scan + G - 1, 4, cudaMemcpyDeviceToHost, h->stream));
      CK(cudaMemcpyAsync(&last_keep, keep + G - 1, 4, cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      const long long T = (long long)last_scan + last_keep;
      if (T * g.tn >= (1LL << 31)) { rc = fail(LBM_EINVAL, "%lld kept tiles exceed 2^31 slots", T); goto done; }
      h->n_tiles = T;
      if ((rc = dev_alloc(h, &h->tiles, (T > 0 ? T : 1) * 3 * 4)) ||
          (rc = dev_alloc(h, &h->nbr27, (T > 0 ? T : 1) * 27 * 4)))
        goto done;
      pt.mark("tile keep + scan");
      k_tile_compact<<<(unsigned)((G + 255) / 256), 256, 0, h->stream>>>(h->rank, keep, scan, h->tiles, g, G);
      CKL();
      if (T > 0) {
        k_tile_nbr<<<(unsigned)((T * 27 + 255) / 256), 256, 0, h->stream>>>(h->nbr27, h->tiles, h->rank, g, T);
        CKL();
      }
      if (T > 0 && h->order_mode) {
        unsigned long long *k0 = nullptr, *k1 = nullptr;
        int* v0 = nullptr;
        void* st = nullptr;
        size_t sb = 0;
        if ((rc = dev_alloc(h, &k0, T * 8)) || (rc = dev_alloc(h, &k1, T * 8)) || (rc = dev_alloc(h, &v0, T * 4)) ||
            (rc = dev_alloc(h, &h->order, T * 4)))
          goto done;
        k_tile_order_key<<<(unsigned)((T + 255) / 256), 256, 0, h->stream>>>(k0, v0, h->tiles, T, h->order_mode,
                                                                             h->pencil, g);
        CKL();
        CK(cub::DeviceRadixSort::SortPairs(nullptr, sb, k0, k1, v0, h->order, (int)T, 0, 63, h->stream));
        if ((rc = dev_alloc(h, (char**)&st, sb))) goto done;
        CK(cub::DeviceRadixSort::SortPairs(st, sb, k0, k1, v0, h->order, (int)T, 0, 63, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        dev_free(k0);
        dev_free(k1);
        dev_free(v0);
        dev_free(st);
      }
      h->n_slots = T * g.tn;
      g.ps = h->n_slots;  // AoSoA: 19 * ps elements = T tiles x 19 blocks
      h->nflags = h->n_slots;
      if ((rc = dev_alloc(h, &h->flags, (h->nflags > 0 ? h->nflags : 1) * 4))) goto done;
      if (h->nflags > 0) {
        pt.mark("compact + nbr27 + order");
        k_flags_tile<<<(unsigned)((h->nflags + 255) / 256), 256, 0, h->stream>>>(
            h->flags, h->tiles, dtype_, dorient, dbc, glo, ghi, g, h->nflags, nb, derr, h->uscratch);
        CKL();
      }
      if ((rc = dev_alloc(h, &h->bmask, (T > 0 ? T : 1) * 32))) goto done;
      CK(cudaMemsetAsync(h->bmask, 0, (T > 0 ? T : 1) * 32, h->stream));
      const int bn = 1 << (g.lbx + g.lby + g.lbz);
      const long long nbricks = h->nflags / bn;
      if (nbricks > 0) {
        k_brick_mask<<<(unsigned)((nbricks + 255) / 256), 256, 0, h->stream>>>(h->bmask, h->flags, g, nbricks);
        CKL();
      }
      if (!h->use_ubits) CK(cudaMemset2DAsync(h->bmask + 4, 32, 0, 16, (T > 0 ? T : 1), h->stream));
      {
        pt.mark("flags + brick masks");
        std::vector<uint32_t> hb((T > 0 ? T : 1) * 8);
        CK(cudaMemcpyAsync(hb.data(), h->bmask, hb.size() * 4, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        long long live = 0, uni = 0;
        for (size_t k = 0; k < hb.size(); ++k) (k % 8 < 4 ? live : uni) += __builtin_popcount(hb[k]);
        // warp work list: groups of (32 / bricksize) live bricks per tile
        {
          const int per = 32 / bn;
          std::vector<int> it;
          it.reserve((size_t)(live / per + T));
          for (long long t = 0; t < T; ++t) {
            int nl = 0;
            for (int q = 0; q < 4; ++q) nl += __builtin_popcount(hb[8 * t + q]);
            for (int gi = 0; gi * per < nl; ++gi) it.push_back((int)(t << 4 | gi));
          }
          pt.mark("brick masks to host + work list");
          h->n_items = (int)it.size();
          if ((rc = dev_alloc(h, &h->items, (it.size() ? it.size() : 1) * 4))) goto done;
          if (!it.empty()) CK(cudaMemcpy(h->items, it.data(), it.size() * 4, cudaMemcpyHostToDevice));
        }
        // per tile: nbr27 + brick masks; per live, non-uniform brick: its flag words
        h->meta_bytes = T * (27 * 4 + 32 + (h->order ? 4 : 0)) + (live - uni) * bn * 4;
      }
      h->sm.rank = h->rank;
      // z-slab ghost planes (tile layouts keep them outside the tile storage)
      h->has_glo = ghost_lo != nullptr;
      h->has_ghi = ghost_hi != nullptr;
      if (h->has_glo || h->has_ghi) {
        const size_t gb = (size_t)10 * plane_nodes * h->esize;
        if ((rc = dev_alloc(h, (char**)&h->gh[0], gb)) || (rc = dev_alloc(h, (char**)&h->gh[1], gb))) goto done;
        CK(cudaMemsetAsync(h->gh[0], 0, gb, h->stream));
        CK(cudaMemsetAsync(h->gh[1], 0, gb, h->stream));
      }
    }
    int herr = 0;
    unsigned long long nons = 0;
    CK(cudaMemcpyAsync(&herr, derr, 4, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(&nons, h->uscratch, 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (herr & 1) { rc = fail(LBM_EINVAL, "node type or orientation out of range"); goto done; }
    if (herr & 2) { rc = fail(LBM_EINVAL, "velocity/pressure node without a valid bc_index or orientation"); goto done; }
    h->n_nonsolid = (long long)nons;
    h->nb = nb;
    // release the descriptor temporaries before the PDF buffers claim HBM
    // (a 2^31-node domain needs every byte: 163 GB AA PDFs + 8.6 GB flags)
    for (void** p : {(void**)&dtype_, (void**)&dorient, (void**)&dbc, (void**)&dglo, (void**)&dghi,
                     (void**)&keep, (void**)&scan, (void**)&cub_tmp}) {
      dev_free(*p);
      *p = nullptr;
    }
    pt.mark("geometry done");
    // PDF buffers
    const size_t fbytes = (size_t)Q * (size_t)(g.ps > 0 ? g.ps : 64) * h->esize;
    if ((rc = dev_alloc(h, (char**)&h->f[0], fbytes))) goto done;
    if (!g.aa && (rc = dev_alloc(h, (char**)&h->f[1], fbytes))) goto done;  // AA: one buffer
    CK(cudaMemsetAsync(h->f[0], 0, fbytes, h->stream));
    if (h->f[1]) CK(cudaMemsetAsync(h->f[1], 0, fbytes, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    pt.mark("PDF buffers alloc + zero");
    h->geometry = true;
    h->parity = 0;
    h->step_count = h->visited_total = 0;
  }
done:
  {
    cudaStreamSynchronize(h->stream);
    dev_free(dtype_);
    dev_free(dorient);
    dev_free(dbc);
    dev_free(dglo);
    dev_free(dghi);
    dev_free(derr);
    dev_free(keep);
    dev_free(scan);
    dev_free(cub_tmp);
    // recompute resident bytes (temporaries released)
    if (h->geometry) {
      long long b = (h->g.aa ? 1LL : 2LL) * Q * (h->g.ps > 0 ? h->g.ps : 64) * h->esize + h->nflags * 4;
      if (h->g.tiled) b += h->ntiles_grid * 4 + h->n_tiles * (30 + 8 + (h->order ? 1 : 0)) * 4;
      if (h->gh[0]) b += 2LL * 10 * h->g.nx * h->g.ny * h->esize;
      h->device_bytes = b;
    }
  }
  if (rc) free_geometry(h);
  return rc;
}

int lbm_init_equilibrium(lbm_t* h, const double* rho, const double* ux, const double* uy,
                         const double* uz, double rho0, double ux0, double uy0, double uz0) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  if (!h->geometry) return fail(LBM_ESTATE, "lbm_set_geometry must run before lbm_init_equilibrium");
  DeviceGuard dg(h->d.device);
  const Geo& g = h->g;
  const long long N = h->n_nodes;
  const double* src[4] = {rho, ux, uy, uz};
  double* dev[4] = {nullptr, nullptr, nullptr, nullptr};
  int rc = 0;
  for (int k = 0; k < 4 && !rc; ++k) {
    if (!src[k]) continue;
    cudaError_t e = cudaMalloc(&dev[k], N * 8);
    if (e != cudaSuccess) {
      rc = fail(LBM_ENOMEM, "init field upload: %s", cudaGetErrorString(e));
      break;
    }
    e = cudaMemcpyAsync(dev[k], src[k], N * 8, cudaMemcpyHostToDevice, h->stream);
    if (e != cudaSuccess) rc = fail(LBM_ECUDA, "init upload: %s", cudaGetErrorString(e));
  }
  if (!rc) {
    const size_t fbytes = (size_t)Q * g.ps * h->esize;
    cudaMemsetAsync(h->f[0], 0, fbytes, h->stream);
    if (h->f[1]) cudaMemsetAsync(h->f[1], 0, fbytes, h->stream);
    h->parity = 0;
    const int bx = 128;
    if (h->esize == 4)
      k_init<float><<<node_grid(g, bx), bx, 0, h->stream>>>((float*)h->f[0], h->flags, h->sm, g, dev[0], dev[1],
                                                            dev[2], dev[3], rho0, ux0, uy0, uz0, h->bckind64,
                                                            h->bcv64, h->bcr64, h->nb);
    else
      k_init<double><<<node_grid(g, bx), bx, 0, h->stream>>>((double*)h->f[0], h->flags, h->sm, g, dev[0], dev[1],
                                                             dev[2], dev[3], rho0, ux0, uy0, uz0, h->bckind64,
                                                             h->bcv64, h->bcr64, h->nb);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) rc = fail(LBM_ECUDA, "k_init: %s", cudaGetErrorString(e));
  }
  for (int k = 0; k < 4; ++k) dev_free(dev[k]);
  if (rc) return rc;
  h->initialized = true;
  h->halo_dirty = true;
  h->step_count = h->visited_total = 0;
  return 0;
}

int lbm_set_omega(lbm_t* h, double omega) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  if (!(omega > 0.0 && omega < 2.0)) return fail(LBM_EINVAL, "omega must lie in (0, 2), got %g", omega);
  h->d.omega = omega;
  drop_graphs(h);
  return 0;
}

int lbm_step_async(lbm_t* h, int64_t n) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  if (n < 0) return fail(LBM_EINVAL, "n_steps must be >= 0, got %lld", (long long)n);
  if (!h->initialized) return fail(LBM_ESTATE, "initialize() must run before stepping");
  DeviceGuard dg(h->d.device);
  const bool halo = halo_on(h);
  if (halo && h->halo_dirty && n > 0) {
    // ghost planes of `pre` after initialize / set_pdf: push, then signal
    if (h->esize == 4) halo_push<float>(h); else halo_push<double>(h);
    halo_signal(h);
    h->halo_dirty = false;
  }
  CK(cudaEventRecord(h->ev0, h->stream));
  // launch-bound small domains: replay a captured CUDA graph of kGraphSteps
  // steps (an even count, so it starts and ends on the same parity)
  if (!halo && h->use_graph && n >= kGraphSteps) {
    cudaGraphExec_t& ge = h->graph[h->parity];
    if (!ge) {
      cudaGraph_t gr = nullptr;
      const int p0 = h->parity;
      const long long l0 = h->launches;
      CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
      for (int k = 0; k < kGraphSteps; ++k) {
        if (h->esize == 4)
          launch_step<float>(h, pre_buf(h), h->g.aa ? h->f[0] : h->f[1 - h->parity]);
        else
          launch_step<double>(h, pre_buf(h), h->g.aa ? h->f[0] : h->f[1 - h->parity]);
        h->parity ^= 1;
      }
      CK(cudaStreamEndCapture(h->stream, &gr));
      h->parity = p0;
      h->launches = l0;
      cudaError_t e = cudaGraphInstantiate(&ge, gr, 0);
      cudaGraphDestroy(gr);
      if (e != cudaSuccess) return fail(LBM_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(e));
    }
    while (n >= kGraphSteps) {
      CK(cudaGraphLaunch(ge, h->stream));
      h->launches += kGraphSteps;
      n -= kGraphSteps;
      h->step_count += kGraphSteps;
      h->visited_total += kGraphSteps * visits_per_step(h);
    }
  }
  for (int64_t k = 0; k < n; ++k) {
    const void* pre = pre_buf(h);
    void* post = h->g.aa ? h->f[0] : h->f[1 - h->parity];
    if (halo) halo_wait(h);   // neighbours pushed my ghosts and finished reading theirs
    if (h->esize == 4)
      launch_step<float>(h, pre, post);
    else
      launch_step<double>(h, pre, post);
    if (halo) halo_signal(h);
    h->parity ^= 1;
  }
  CKL();
  CK(cudaEventRecord(h->ev1, h->stream));
  h->pending = true;
  h->step_count += n;
  h->visited_total += n * visits_per_step(h);
  return 0;
}

int lbm_synchronize(lbm_t* h) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  DeviceGuard dg(h->d.device);
  if (!h->pending) return 0;
  h->pending = false;
  CK(cudaEventSynchronize(h->ev1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  h->last_ms = ms;
  if (halo_on(h)) {
    int herr = 0;
    CK(cudaMemcpy(&herr, h->herr, 4, cudaMemcpyDeviceToHost));
    if (herr) return fail(LBM_ENCCL, "halo wait timed out: a neighbouring slab stopped stepping");
  }
  return 0;
}

int lbm_step(lbm_t* h, int64_t n) {
  int rc = lbm_step_async(h, n);
  if (rc) return rc;
  return lbm_synchronize(h);
}

// z-planes per readback chunk: device staging bounded by kStageBytes, so
// readbacks work next to a domain that fills HBM
constexpr long long kStageBytes = 1LL << 30;
int chunk_planes(const lbm_handle* h, long long bytes_per_node) {
  const long long plane = (long long)h->g.nx * h->g.ny * bytes_per_node;
  long long c = kStageBytes / (plane > 0 ? plane : 1);
  if (c < 1) c = 1;
  if (c > h->g.nz) c = h->g.nz;
  if (c > 65535) c = 65535;  // grid z limit
  return (int)c;
}

extern "C++" {
// host copy split over threads (also spreads the page faults of fresh
// destination arrays)
static void par_copy(const std::vector<std::pair<char*, const char*>>& dst_src, const std::vector<size_t>& n) {
  size_t total = 0;
  for (size_t v : n) total += v;
  const int nt = total > (8u << 20) ? 8 : 1;
  auto work = [&](int t) {
    for (size_t k = 0; k < n.size(); ++k) {
      const size_t per = (n[k] + nt - 1) / nt, a = per * t, b = a + per < n[k] ? a + per : n[k];
      if (a < b) memcpy(dst_src[k].first + a, dst_src[k].second + a, b - a);
    }
  };
  if (nt == 1) {
    work(0);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
}

// Pipelined device -> host readback in z chunks: chunk k's kernel and D2H
// copy (into pinned staging) overlap the host copy of chunk k-1 out of the
// other pinned slot.  launch(k, z0, nzc, dev) enqueues the chunk kernel;
// consume(k, z0, nzc, pinned) copies it into the caller's arrays.
template <class Launch, class Consume>
static int pipelined_d2h(lbm_handle* h, long long bytes_per_node, Launch launch, Consume consume) {
  const long long pn = (long long)h->g.nx * h->g.ny;
  const size_t want = 64u << 20;  // per staging slot
  long long cz = (long long)want / (pn * bytes_per_node);
  if (cz < 1) cz = 1;
  if (cz > h->g.nz) cz = h->g.nz;
  if (cz > 65535) cz = 65535;
  const size_t slot = (size_t)(cz * pn * bytes_per_node);
  if (h->pin_bytes < slot) {
    for (int b = 0; b < 2; ++b) {
      if (h->pin[b]) cudaFreeHost(h->pin[b]);
      h->pin[b] = nullptr;
    }
    h->pin_bytes = 0;
    for (int b = 0; b < 2; ++b)
      if (cudaHostAlloc(&h->pin[b], slot, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return fail(LBM_ENOMEM, "pinned staging of %zu bytes failed", slot);
      }
    h->pin_bytes = slot;
  }
  for (int b = 0; b < 2; ++b)
    if (!h->evc[b]) CK(cudaEventCreateWithFlags(&h->evc[b], cudaEventDisableTiming));
  char* dev = nullptr;
  cudaError_t e = cudaMalloc(&dev, 2 * slot);
  if (e != cudaSuccess) return fail(LBM_ENOMEM, "readback staging: %s", cudaGetErrorString(e));
  const int nz = h->g.nz;
  const int nchunk = (int)((nz + cz - 1) / cz);
  for (int k = 0; k <= nchunk && e == cudaSuccess; ++k) {
    if (k < nchunk) {
      const int b = k & 1, z0 = (int)(k * cz), nzc = (int)(nz - z0 < cz ? nz - z0 : cz);
      launch(k, z0, nzc, dev + b * slot);
      e = cudaGetLastError();
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(h->pin[b], dev + b * slot, (size_t)(nzc * pn * bytes_per_node), cudaMemcpyDeviceToHost,
                            h->stream);
      if (e == cudaSuccess) e = cudaEventRecord(h->evc[b], h->stream);
    }
    if (k > 0 && e == cudaSuccess) {
      const int b = (k - 1) & 1, z0 = (int)((k - 1) * cz), nzc = (int)(nz - z0 < cz ? nz - z0 : cz);
      e = cudaEventSynchronize(h->evc[b]);
      if (e == cudaSuccess) consume(k - 1, z0, nzc, (const char*)h->pin[b]);
    }
  }
  cudaStreamSynchronize(h->stream);
  cudaFree(dev);
  if (e != cudaSuccess) return fail(LBM_ECUDA, "readback: %s", cudaGetErrorString(e));
  return 0;
}

}  // extern "C++"

int lbm_get_macroscopic(lbm_t* h, double* rho, double* ux, double* uy, double* uz) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  DeviceGuard dg(h->d.device);
  const Geo g = rb_geo(h);
  const long long pn = (long long)g.nx * g.ny;
  double* outs[4] = {rho, ux, uy, uz};
  int nf = 0, which[4];
  for (int k = 0; k < 4; ++k)
    if (outs[k]) which[nf++] = k;
  if (!nf) return 0;
  // staging chunk: the requested fields back to back, (nf, nzc * pn) doubles
  auto launch = [&](int, int z0, int nzc, char* dev) {
    double* d = (double*)dev;
    const long long C = (long long)nzc * pn;
    double* f[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int j = 0; j < nf; ++j) f[which[j]] = d + j * C;
    const dim3 grid((g.nx + 127) / 128, g.ny, nzc);
    if (h->esize == 4)
      k_macro<float><<<grid, 128, 0, h->stream>>>((const float*)pre_buf(h), h->flags, h->sm, g, z0, f[0], f[1], f[2],
                                                  f[3]);
    else
      k_macro<double><<<grid, 128, 0, h->stream>>>((const double*)pre_buf(h), h->flags, h->sm, g, z0, f[0], f[1],
                                                   f[2], f[3]);
  };
  auto consume = [&](int, int z0, int nzc, const char* pin) {
    const long long C = (long long)nzc * pn;
    std::vector<std::pair<char*, const char*>> ds;
    std::vector<size_t> n;
    for (int j = 0; j < nf; ++j) {
      ds.emplace_back((char*)(outs[which[j]] + z0 * pn), pin + (size_t)j * C * 8);
      n.push_back((size_t)C * 8);
    }
    par_copy(ds, n);
  };
  return pipelined_d2h(h, 8LL * nf, launch, consume);
}

int lbm_get_macroscopic_box(lbm_t* h, const int32_t* lo, const int32_t* hi, double* rho, double* ux,
                            double* uy, double* uz) {
  if (!h || !lo || !hi) return fail(LBM_EINVAL, "NULL argument");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  const int n3[3] = {h->g.nx, h->g.ny, h->g.nz};
  for (int a = 0; a < 3; ++a)
    if (lo[a] < 0 || hi[a] > n3[a] || lo[a] >= hi[a])
      return fail(LBM_EINVAL, "box [%d, %d) outside axis %d of extent %d", lo[a], hi[a], a, n3[a]);
  DeviceGuard dg(h->d.device);
  const Geo g = rb_geo(h);
  const int bx = hi[0] - lo[0], by = hi[1] - lo[1], bz = hi[2] - lo[2];
  if (by > 65535 || bz > 65535) return fail(LBM_EINVAL, "box too tall for one launch");
  const long long C = (long long)bx * by * bz;
  double* d = nullptr;
  cudaError_t e = cudaMalloc(&d, C * 8 * 4);
  if (e != cudaSuccess) return fail(LBM_ENOMEM, "box readback: %s", cudaGetErrorString(e));
  double* outs[4] = {rho, ux, uy, uz};
  double* f[4];
  for (int k = 0; k < 4; ++k) f[k] = outs[k] ? d + k * C : nullptr;
  const dim3 grid((bx + 127) / 128, by, bz);
  if (h->esize == 4)
    k_macro<float><<<grid, 128, 0, h->stream>>>((const float*)pre_buf(h), h->flags, h->sm, g, lo[2], f[0], f[1], f[2],
                                                f[3], lo[0], lo[1], bx);
  else
    k_macro<double><<<grid, 128, 0, h->stream>>>((const double*)pre_buf(h), h->flags, h->sm, g, lo[2], f[0], f[1],
                                                 f[2], f[3], lo[0], lo[1], bx);
  e = cudaGetLastError();
  for (int k = 0; k < 4 && e == cudaSuccess; ++k)
    if (outs[k]) e = cudaMemcpyAsync(outs[k], d + k * C, C * 8, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  cudaFree(d);
  if (e != cudaSuccess) return fail(LBM_ECUDA, "box readback: %s", cudaGetErrorString(e));
  return 0;
}

int lbm_check_finite(lbm_t* h, int32_t* dir, int32_t* node_xyz) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  DeviceGuard dg(h->d.device);
  const Geo g = rb_geo(h);
  const unsigned long long none = ~0ULL;
  const long long V = g.tiled ? h->n_slots : h->n_nodes;
  CK(cudaMemcpyAsync(h->uscratch, &none, 8, cudaMemcpyHostToDevice, h->stream));
  const int bx = 128;
  if (h->esize == 4)
    k_nonfinite<float><<<node_grid(g, bx), bx, 0, h->stream>>>((const float*)pre_buf(h), h->flags, h->sm, g, V, h->uscratch);
  else
    k_nonfinite<double><<<node_grid(g, bx), bx, 0, h->stream>>>((const double*)pre_buf(h), h->flags, h->sm, g, V, h->uscratch);
  CKL();
  unsigned long long best = 0;
  CK(cudaMemcpyAsync(&best, h->uscratch, 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (best == none) {
    if (dir) *dir = -1;
    return 0;
  }
  const long long i = (long long)(best / (unsigned long long)V);
  const long long v = (long long)(best % (unsigned long long)V);
  int x, y, z;
  if (!g.tiled) {
    x = (int)(v % g.nx);
    y = (int)((v / g.nx) % g.ny);
    z = (int)(v / ((long long)g.nx * g.ny));
  } else {
    const long long t = v / g.tn;
    const int l = (int)(v % g.tn);
    int tc[3];
    CK(cudaMemcpy(tc, h->tiles + 3 * t, 12, cudaMemcpyDeviceToHost));
    int lx, ly, lz;
    brick_inv(g, l, lx, ly, lz);
    x = tc[0] * g.ex + lx;
    y = tc[1] * g.ey + ly;
    z = tc[2] * g.ez + lz;
  }
  if (dir) *dir = (int32_t)i;
  if (node_xyz) {
    node_xyz[0] = x;
    node_xyz[1] = y;
    node_xyz[2] = z;
  }
  return fail(LBM_EDIVERGED, "non-finite distribution at node (%d, %d, %d), direction %lld", x, y, z, i);
}

int lbm_total_mass(lbm_t* h, double* mass) {
  if (!h || !mass) return fail(LBM_EINVAL, "NULL argument");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  DeviceGuard dg(h->d.device);
  const int nblk = 1184;  // 8 x 148 SMs; fixed so the reduction order is fixed
  if (h->esize == 4)
    k_mass_partial<float><<<nblk, 256, 0, h->stream>>>((const float*)pre_buf(h), h->flags, h->sm, h->tiles, rb_geo(h),
                                                       h->nflags, h->scratch);
  else
    k_mass_partial<double><<<nblk, 256, 0, h->stream>>>((const double*)pre_buf(h), h->flags, h->sm, h->tiles, rb_geo(h),
                                                        h->nflags, h->scratch);
  k_mass_final<<<1, 256, 0, h->stream>>>(h->scratch, nblk, h->scratch + nblk);
  CKL();
  CK(cudaMemcpyAsync(mass, h->scratch + nblk, 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return 0;
}

static int pdf_io(lbm_t* h, int which, void* host, bool get) {
  if (!h || !host) return fail(LBM_EINVAL, "NULL argument");
  if (which != 0 && which != 1) return fail(LBM_EINVAL, "which must be 0 (pre) or 1 (post)");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  if (h->g.aa && which != 0) return fail(LBM_EINVAL, "the AA scheme keeps one buffer: there is no post buffer");
  DeviceGuard dg(h->d.device);
  const Geo g = rb_geo(h);
  const long long N = h->n_nodes, pn = (long long)g.nx * g.ny;
  const int es = h->esize;
  const int cz = chunk_planes(h, (long long)Q * es);
  const long long C = pn * cz;
  char* d = nullptr;
  cudaError_t e = cudaMalloc(&d, C * Q * es);
  if (e != cudaSuccess) return fail(LBM_ENOMEM, "pdf staging: %s", cudaGetErrorString(e));
  void* buf = which == 0 ? pre_buf(h) : h->f[1 - h->parity];
  char* hb = (char*)host;
  if (get) {
    cudaFree(d);
    // pipelined: chunk = (19, nzc * pn) in the storage type
    auto launch = [&](int, int z0, int nzc, char* dev) {
      const dim3 grid((g.nx + 127) / 128, g.ny, nzc);
      if (es == 4)
        k_get_pdf<float><<<grid, 128, 0, h->stream>>>((const float*)buf, h->flags, h->sm, g, z0, (float*)dev);
      else
        k_get_pdf<double><<<grid, 128, 0, h->stream>>>((const double*)buf, h->flags, h->sm, g, z0, (double*)dev);
    };
    auto consume = [&](int, int z0, int nzc, const char* pin) {
      const long long cn = pn * nzc;
      std::vector<std::pair<char*, const char*>> ds;
      std::vector<size_t> n;
      for (int i = 0; i < Q; ++i) {
        ds.emplace_back(hb + (i * N + z0 * pn) * es, pin + (size_t)i * cn * es);
        n.push_back((size_t)cn * es);
      }
      par_copy(ds, n);
    };
    return pipelined_d2h(h, (long long)Q * es, launch, consume);
  }
  // canonical (19, nz, ny, nx): one host block per direction and z chunk
  for (int z0 = 0; z0 < g.nz && e == cudaSuccess; z0 += cz) {
    const int nzc = g.nz - z0 < cz ? g.nz - z0 : cz;
    const long long cn = pn * nzc;
    const dim3 grid((g.nx + 127) / 128, g.ny, nzc);
    if (!get) {
      for (int i = 0; i < Q && e == cudaSuccess; ++i)
        e = cudaMemcpyAsync(d + i * cn * es, hb + (i * N + z0 * pn) * es, cn * es, cudaMemcpyHostToDevice, h->stream);
      if (e != cudaSuccess) break;
      if (es == 4)
        k_set_pdf<float><<<grid, 128, 0, h->stream>>>((float*)buf, h->flags, h->sm, g, z0, (const float*)d);
      else
        k_set_pdf<double><<<grid, 128, 0, h->stream>>>((double*)buf, h->flags, h->sm, g, z0, (const double*)d);
      e = cudaGetLastError();
    } else {
      if (es == 4)
        k_get_pdf<float><<<grid, 128, 0, h->stream>>>((const float*)buf, h->flags, h->sm, g, z0, (float*)d);
      else
        k_get_pdf<double><<<grid, 128, 0, h->stream>>>((const double*)buf, h->flags, h->sm, g, z0, (double*)d);
      e = cudaGetLastError();
      for (int i = 0; i < Q && e == cudaSuccess; ++i)
        e = cudaMemcpyAsync(hb + (i * N + z0 * pn) * es, d + i * cn * es, cn * es, cudaMemcpyDeviceToHost, h->stream);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  }
  cudaFree(d);
  if (e != cudaSuccess) return fail(LBM_ECUDA, "pdf io: %s", cudaGetErrorString(e));
  return 0;
}

int lbm_get_pdf(lbm_t* h, int32_t which, void* out) { return pdf_io(h, which, out, true); }
int lbm_set_pdf(lbm_t* h, int32_t which, const void* in) {
  if (h) h->halo_dirty = true;
  return pdf_io(h, which, (void*)in, false);
}

static int field_io(lbm_t* h, int which, void* host, bool get) {
  if (!h || !host) return fail(LBM_EINVAL, "NULL argument");
  if (which != 0 && which != 1) return fail(LBM_EINVAL, "which must be 0 (pre) or 1 (post)");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  if (h->g.aa && which != 0) return fail(LBM_EINVAL, "the AA scheme keeps one buffer: there is no post buffer");
  DeviceGuard dg(h->d.device);
  const size_t bytes = (size_t)Q * h->g.ps * h->esize;
  if (h->g.aa) {
    // decoded pre buffer in the native slot order, staged on the device
    void* d = nullptr;
    cudaError_t e = cudaMalloc(&d, bytes);
    if (e != cudaSuccess) return fail(LBM_ENOMEM, "field staging: %s", cudaGetErrorString(e));
    const Geo g = rb_geo(h);
    const dim3 grid = node_grid(g, 128);
    if (get) {
      e = cudaMemsetAsync(d, 0, bytes, h->stream);
      if (e == cudaSuccess) {
        if (h->esize == 4)
          k_field_aa<float, true><<<grid, 128, 0, h->stream>>>((float*)h->f[0], h->flags, h->sm, g, (float*)d);
        else
          k_field_aa<double, true><<<grid, 128, 0, h->stream>>>((double*)h->f[0], h->flags, h->sm, g, (double*)d);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess) e = cudaMemcpyAsync(host, d, bytes, cudaMemcpyDeviceToHost, h->stream);
    } else {
      e = cudaMemcpyAsync(d, host, bytes, cudaMemcpyHostToDevice, h->stream);
      if (e == cudaSuccess) {
        if (h->esize == 4)
          k_field_aa<float, false><<<grid, 128, 0, h->stream>>>((float*)h->f[0], h->flags, h->sm, g, (float*)d);
        else
          k_field_aa<double, false><<<grid, 128, 0, h->stream>>>((double*)h->f[0], h->flags, h->sm, g, (double*)d);
        e = cudaGetLastError();
      }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    cudaFree(d);
    if (e != cudaSuccess) return fail(LBM_ECUDA, "field io: %s", cudaGetErrorString(e));
    return 0;
  }
  void* buf = h->f[which == 0 ? h->parity : 1 - h->parity];
  if (get)
    CK(cudaMemcpy(host, buf, bytes, cudaMemcpyDeviceToHost));
  else
    CK(cudaMemcpy(buf, host, bytes, cudaMemcpyHostToDevice));
  return 0;
}

int lbm_get_field(lbm_t* h, int32_t which, void* out) { return field_io(h, which, out, true); }
int lbm_set_field(lbm_t* h, int32_t which, const void* in) {
  if (h) h->halo_dirty = true;
  return field_io(h, which, (void*)in, false);
}

int lbm_get_slot_of(lbm_t* h, int32_t* out) {
  if (!h || !out) return fail(LBM_EINVAL, "NULL argument");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  DeviceGuard dg(h->d.device);
  int* d = nullptr;
  cudaError_t e = cudaMalloc(&d, h->n_nodes * 4);
  if (e != cudaSuccess) return fail(LBM_ENOMEM, "slot_of staging: %s", cudaGetErrorString(e));
  k_slot_of<<<node_grid(h->g, 128), 128, 0, h->stream>>>(h->sm, h->g, d);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, h->n_nodes * 4, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  cudaFree(d);
  if (e != cudaSuccess) return fail(LBM_ECUDA, "slot_of: %s", cudaGetErrorString(e));
  return 0;
}

int lbm_get_flags(lbm_t* h, uint32_t* out) {
  if (!h || !out) return fail(LBM_EINVAL, "NULL argument");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  DeviceGuard dg(h->d.device);
  uint32_t* d = nullptr;
  cudaError_t e = cudaMalloc(&d, h->n_nodes * 4);
  if (e != cudaSuccess) return fail(LBM_ENOMEM, "flags staging: %s", cudaGetErrorString(e));
  k_get_flags<<<node_grid(h->g, 128), 128, 0, h->stream>>>(h->flags, h->sm, h->g, d);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, h->n_nodes * 4, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  cudaFree(d);
  if (e != cudaSuccess) return fail(LBM_ECUDA, "flags: %s", cudaGetErrorString(e));
  return 0;
}

int lbm_get_tile_index(lbm_t* h, int32_t* tiles, int32_t* nbr27, int64_t* n_tiles) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  if (!h->geometry) return fail(LBM_ESTATE, "no geometry");
  if (n_tiles) *n_tiles = h->n_tiles;
  if (!h->g.tiled) return 0;
  DeviceGuard dg(h->d.device);
  if (tiles && h->n_tiles) CK(cudaMemcpy(tiles, h->tiles, h->n_tiles * 12, cudaMemcpyDeviceToHost));
  if (nbr27 && h->n_tiles) CK(cudaMemcpy(nbr27, h->nbr27, h->n_tiles * 27 * 4, cudaMemcpyDeviceToHost));
  return 0;
}

int lbm_get_stats(lbm_t* h, lbm_stats* s) {
  if (!h || !s) return fail(LBM_EINVAL, "NULL argument");
  memset(s, 0, sizeof(*s));
  s->n_nodes = h->n_nodes;
  s->n_nonsolid = h->n_nonsolid;
  s->visits_per_step = (h->d.layout == LBM_LAYOUT_DENSE) ? h->n_nodes
                       : (h->d.layout == LBM_LAYOUT_BITMASK_NODE) ? h->n_nonsolid
                                                                   : h->n_slots;
  s->n_slots = h->n_slots;
  s->plane_stride = h->g.ps;
  s->n_tiles = h->n_tiles;
  s->step_count = h->step_count;
  s->visited_nodes_total = h->visited_total;
  s->device_bytes = h->device_bytes;
  s->launches_total = h->launches;
  s->last_step_ms = h->last_ms;
  s->meta_bytes_per_step = h->meta_bytes;
  s->parity = h->parity;
  s->initialized = h->initialized ? 1 : 0;
  s->scheme = h->d.scheme;
  return 0;
}

// ------------------------------------------------------------- halo C-ABI
namespace {
struct HaloBlob {
  uint32_t magic;
  int32_t device, esize, nz, ny, nxp, tiled;
  int64_t pid, ps;
  void* f[2];
  void* sync;
  cudaIpcMemHandle_t ipc_f[2];
  cudaIpcMemHandle_t ipc_sync;
};
constexpr uint32_t kHaloMagic = 0x4C424D48u;  // "LBMH"
static_assert(sizeof(HaloBlob) <= LBM_HALO_BLOB_BYTES, "halo blob too large");

int open_peer(lbm_handle* h, const HaloBlob& b, lbm_handle::Peer& pr) {
  if (b.magic != kHaloMagic) return fail(LBM_EINVAL, "not a halo blob");
  if (b.esize != h->esize || b.ny != h->g.ny || b.nxp != h->g.nxp || b.tiled != h->g.tiled)
    return fail(LBM_EINVAL, "neighbouring slab has a different dtype, layout family or x/y extent");
  if (b.pid == (int64_t)getpid()) {
    if (b.device != h->d.device) {
      int can = 0;
      CK(cudaDeviceCanAccessPeer(&can, h->d.device, b.device));
      if (!can) return fail(LBM_ENCCL, "device %d cannot access peer %d", h->d.device, b.device);
      cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fail(LBM_ENCCL, "cudaDeviceEnablePeerAccess: %s", cudaGetErrorString(e));
      cudaGetLastError();
    }
    pr.f[0] = b.f[0];
    pr.f[1] = b.f[1];
    pr.sync = (unsigned long long*)b.sync;
    pr.ipc = false;
  } else {
    CK(cudaIpcOpenMemHandle(&pr.f[0], b.ipc_f[0], cudaIpcMemLazyEnablePeerAccess));
    CK(cudaIpcOpenMemHandle(&pr.f[1], b.ipc_f[1], cudaIpcMemLazyEnablePeerAccess));
    void* sy = nullptr;
    CK(cudaIpcOpenMemHandle(&sy, b.ipc_sync, cudaIpcMemLazyEnablePeerAccess));
    pr.sync = (unsigned long long*)sy;
    pr.ipc = true;
  }
  pr.ps = b.ps;
  pr.nz = b.nz;
  pr.on = true;
  return 0;
}
}  // namespace

int lbm_halo_export(lbm_t* h, void* blob, size_t* bytes) {
  if (!h || !blob) return fail(LBM_EINVAL, "NULL argument");
  if (!h->geometry) return fail(LBM_ESTATE, "lbm_set_geometry must run before lbm_halo_export");
  if (h->g.aa) return fail(LBM_EINVAL, "z-slab halos need the AB scheme in this build");
  if (h->g.tiled && !h->gh[0]) return fail(LBM_EINVAL, "this tile handle is not a z-slab (no ghost planes)");
  DeviceGuard dg(h->d.device);
  HaloBlob b;
  memset(&b, 0, sizeof(b));
  b.magic = kHaloMagic;
  b.device = h->d.device;
  b.esize = h->esize;
  b.nz = h->g.nz;
  b.ny = h->g.ny;
  b.nxp = h->g.nxp;
  b.pid = (int64_t)getpid();
  b.ps = h->g.ps;
  b.tiled = h->g.tiled;
  // dense: the PDF buffers (ghost planes inside); tiles: the ghost-plane buffers
  void* const* ex = h->g.tiled ? h->gh : h->f;
  b.f[0] = ex[0];
  b.f[1] = ex[1];
  b.sync = h->sync;
  CK(cudaIpcGetMemHandle(&b.ipc_f[0], ex[0]));
  CK(cudaIpcGetMemHandle(&b.ipc_f[1], ex[1]));
  CK(cudaIpcGetMemHandle(&b.ipc_sync, h->sync));
  memset(blob, 0, LBM_HALO_BLOB_BYTES);
  memcpy(blob, &b, sizeof(b));
  if (bytes) *bytes = LBM_HALO_BLOB_BYTES;
  return 0;
}

int lbm_halo_connect(lbm_t* h, const void* lo_blob, const void* hi_blob) {
  if (!h) return fail(LBM_EINVAL, "NULL handle");
  if (!h->geometry) return fail(LBM_ESTATE, "lbm_set_geometry must run before lbm_halo_connect");
  if (h->g.tiled && !h->gh[0] && (lo_blob || hi_blob))
    return fail(LBM_EINVAL, "this tile handle is not a z-slab (no ghost planes)");
  if (h->g.pzw && (lo_blob || hi_blob))
    return fail(LBM_EINVAL, "a whole-domain periodic handle wraps z itself; it takes no halo");
  DeviceGuard dg(h->d.device);
  CK(cudaStreamSynchronize(h->stream));
  int rc = 0;
  HaloBlob b;
  if (lo_blob) {
    memcpy(&b, lo_blob, sizeof(b));
    if ((rc = open_peer(h, b, h->lo))) return rc;
  }
  if (hi_blob) {
    memcpy(&b, hi_blob, sizeof(b));
    if ((rc = open_peer(h, b, h->hi))) return rc;
  }
  if (h->esize == 4) preload_halo_kernels<float>(h); else preload_halo_kernels<double>(h);
  h->halo_dirty = true;
  return 0;
}

}  // extern "C"

// ------------------------------------------------------- scalar host math
template <typename T>
static void to_t(const double* in, T* out, int n) {
  for (int k = 0; k < n; ++k) out[k] = (T)in[k];
}
template <typename T>
static void from_t(const T* in, double* out, int n) {
  for (int k = 0; k < n; ++k) out[k] = (double)in[k];
}

template <typename T>
static int feq_t(double rho, const double* u3, double* out) {
  T e[Q];
  feq19<T>((T)rho, (T)u3[0], (T)u3[1], (T)u3[2], e);
  from_t(e, out, Q);
  return 0;
}

extern "C" int lbm19_feq(int32_t dtype, double rho, const double* u3, double* out19) {
  if (!u3 || !out19) return fail(LBM_EINVAL, "NULL argument");
  return dtype == LBM_F32 ? feq_t<float>(rho, u3, out19) : feq_t<double>(rho, u3, out19);
}

template <typename T>
static int moments_t(const double* f19, double* rho, double* u3) {
  T f[Q], r, a, b, c;
  to_t(f19, f, Q);
  moments19<T>(f, r, a, b, c);
  *rho = r;
  u3[0] = a;
  u3[1] = b;
  u3[2] = c;
  return 0;
}

extern "C" int lbm19_moments(int32_t dtype, const double* f19, double* rho, double* u3) {
  if (!f19 || !rho || !u3) return fail(LBM_EINVAL, "NULL argument");
  return dtype == LBM_F32 ? moments_t<float>(f19, rho, u3) : moments_t<double>(f19, rho, u3);
}

template <typename T>
static int collide_t(const double* f19, double omega, double* out) {
  T f[Q], r, a, b, c;
  to_t(f19, f, Q);
  moments19<T>(f, r, a, b, c);
  collide19<T>(f, r, a, b, c, (T)omega);
  from_t(f, out, Q);
  return 0;
}

extern "C" int lbm19_collide(int32_t dtype, const double* f19, double omega, double* out19) {
  if (!f19 || !out19) return fail(LBM_EINVAL, "NULL argument");
  return dtype == LBM_F32 ? collide_t<float>(f19, omega, out19) : collide_t<double>(f19, omega, out19);
}

template <typename T>
static int zhv_t(const double* f19, int orient, const double* u3, double* out) {
  T f[Q];
  to_t(f19, f, Q);
  zou_he_velocity19<T>(f, (uint32_t)orient, (T)u3[0], (T)u3[1], (T)u3[2]);
  from_t(f, out, Q);
  return 0;
}

extern "C" int lbm19_zou_he_velocity(int32_t dtype, const double* f19, int32_t orient, const double* u3, double* out19) {
  if (!f19 || !u3 || !out19) return fail(LBM_EINVAL, "NULL argument");
  if (orient < O_NORTH || orient > O_BOTTOM) return fail(LBM_EINVAL, "orientation must name a face, got %d", orient);
  return dtype == LBM_F32 ? zhv_t<float>(f19, orient, u3, out19) : zhv_t<double>(f19, orient, u3, out19);
}

template <typename T>
static int zhp_t(const double* f19, int orient, double rw, double* out) {
  T f[Q];
  to_t(f19, f, Q);
  zou_he_pressure19<T>(f, (uint32_t)orient, (T)rw);
  from_t(f, out, Q);
  return 0;
}

extern "C" int lbm19_zou_he_pressure(int32_t dtype, const double* f19, int32_t orient, double rho_wall, double* out19) {
  if (!f19 || !out19) return fail(LBM_EINVAL, "NULL argument");
  if (orient < O_NORTH || orient > O_BOTTOM) return fail(LBM_EINVAL, "orientation must name a face, got %d", orient);
  return dtype == LBM_F32 ? zhp_t<float>(f19, orient, rho_wall, out19) : zhp_t<double>(f19, orient, rho_wall, out19);
}


