// Sparse tile step kernels over brick records (AB: warp work list and
// CTA per tile, with the z-slab ghost exchange; A-A in place).
// Part of liblbm19 (included once, in order, by lbm19.cu).
#pragma once

// Storage (tile layouts): AoSoA f[tile][direction][in-tile slot], each
// (tile, direction) block contiguous (TN elements: 2 KB for 512 fp32 nodes),
// in-tile slots in sector-brick order (layout.cuh).  Element of (direction
// i, in-tile slot l) of tile t: t * (Q * TN) + i * TN + l.
//
// Measured alternative (round 2, profiles/ab_brick_records_r02.txt): 640-B
// brick records (19 direction sectors of one brick + pad, so a 128-B line
// never mixes live and dead bricks) cut the DRAM reads of the porous
// configs' partly live lines, but a warp's four bricks then touch four lines
// per load instead of one: +5 % at phi = 0.1, -9 to -26 % at phi >= 0.2 and
// on the vascular forest.  The per-direction blocks stay.

template <typename T>
struct Rec {
  static constexpr int BN = 32 / (int)sizeof(T);  // nodes per brick (one sector)
};

// Live-brick enumeration of one tile for the CTA-per-tile kernels: threads
// cover only the tile's live bricks (sector-sized bricks holding >= 1
// non-solid node, a 128-bit mask per tile), so a sparse tile costs lanes in
// proportion to its live sectors.  Words 4-7 of the mask mark uniform bricks
// (all FLUID / wall with full masks) whose flag words the step skips.
struct TileBricks {
  uint32_t m[4], u[4];
  int pre_cnt[4];
  int work, lbn, bn;
  bool dense_tile;
  __device__ __forceinline__ TileBricks(const uint32_t* __restrict__ bmask, long long t, const Geo& g, int tn) {
    lbn = g.lbx + g.lby + g.lbz;
    bn = 1 << lbn;
    int acc = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      u[q] = __ldg(bmask + 8LL * t + 4 + q);
      m[q] = __ldg(bmask + 8LL * t + q);
      pre_cnt[q] = acc;
      acc += __popc(m[q]);
    }
    work = ((acc << lbn) + 31) & ~31;   // whole warps; lanes past acc*bn idle
    dense_tile = acc == (tn >> lbn);    // every brick live: identity mapping
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

// Per in-tile slot neighbour table (built on the host for the handle's tile
// shape, 16 B per slot, L1-resident).  x: bits 0-55 the magnitudes of the
// in-tile slot deltas (14 bits each) to the x-, x+, y-, y+ neighbours, bits
// 56-61 whether each of the six neighbours lies across the tile face (the
// delta is then a wrap inside the neighbour tile: positive for "-", negative
// for "+"); y: bits 0-27 the z-, z+ magnitudes, bits 32-47 the slot itself.
struct TileUpLUT {
  int p, dxm, dxp, dym, dyp, dzm, dzp, cxm, cxp, cym, cyp, czm, czp;
  __device__ __forceinline__ TileUpLUT(const ulonglong2* __restrict__ lut, int slot) : TileUpLUT(__ldg(lut + slot)) {}
  __device__ __forceinline__ explicit TileUpLUT(const ulonglong2 e) {
    const unsigned cr = (unsigned)(e.x >> 56) & 63u;
    const int m0 = (int)(e.x & 16383u), m1 = (int)(e.x >> 14 & 16383u), m2 = (int)(e.x >> 28 & 16383u),
              m3 = (int)(e.x >> 42 & 16383u), m4 = (int)(e.y & 16383u), m5 = (int)(e.y >> 14 & 16383u);
    p = (int)(e.y >> 32 & 65535u);
    dxm = (cr & 1) ? m0 : -m0;
    dxp = (cr & 2) ? -m1 : m1;
    dym = (cr & 4) ? m2 : -m2;
    dyp = (cr & 8) ? -m3 : m3;
    dzm = (cr & 16) ? m4 : -m4;
    dzp = (cr & 32) ? -m5 : m5;
    cxm = (cr & 1) ? -1 : 0, cxp = (cr & 2) ? 1 : 0;
    cym = (cr & 4) ? -3 : 0, cyp = (cr & 8) ? 3 : 0;
    czm = (cr & 16) ? -9 : 0, czp = (cr & 32) ? 9 : 0;
  }
  // tile code (dx+1) + 3(dy+1) + 9(dz+1) of the node x - c_i
  __device__ __forceinline__ int code(int i) const {
    return 13 + (cx(i) == 1 ? cxm : (cx(i) == -1 ? cxp : 0)) + (cy(i) == 1 ? cym : (cy(i) == -1 ? cyp : 0)) +
           (cz(i) == 1 ? czm : (cz(i) == -1 ? czp : 0));
  }
  // in-tile slot of the node x - c_i (in the tile given by code(i))
  __device__ __forceinline__ int loc(int i) const {
    return p + (cx(i) == 1 ? dxm : (cx(i) == -1 ? dxp : 0)) + (cy(i) == 1 ? dym : (cy(i) == -1 ? dyp : 0)) +
           (cz(i) == 1 ? dzm : (cz(i) == -1 ? dzp : 0));
  }
};

// the 27 neighbour ranks of tile t as element offsets relative to the tile,
// one per lane (lanes 0-26; absent: 0, i.e. the own tile -- such links are masked)
template <typename T, int TN>
__device__ __forceinline__ int nbr_rel(const int* __restrict__ nbr27, int t, int lane) {
  int srel = 0;
  if (lane < 27) {
    const int v = __ldg(nbr27 + 27LL * t + lane);
    srel = v < 0 ? 0 : (v - t) * (Q * TN);
  }
  return srel;
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

// One CTA per kept tile, threads over the tile's live bricks.  Every warp
// keeps the 27 relative tile offsets in lanes 0-26 and fetches them with
// shuffles (all lanes take part, so the offsets are formed before dead lanes
// leave the iteration).  SEL: exact per-link select (a masked link never
// fetches the -- solid -- upstream slot); else speculative pull + bounce-back
// fix-up.  CUT: z-slab, tiles on the first / last tile plane exchange their
// boundary nodes' c_z populations through ghost planes (uniform per CTA).
template <typename T, int TN, int MINB, bool SEL = false, bool CUT = false>
__global__ void __launch_bounds__(TN < 256 ? TN : 256, MINB)
k_step_tiles_x(const T* __restrict__ pre, T* __restrict__ post, const uint32_t* __restrict__ flags,
               const int* __restrict__ nbr27, const T* __restrict__ bcv, const T* __restrict__ bcr, Geo g, T om,
               const uint32_t* __restrict__ bmask, const ulonglong2* __restrict__ lut,
               const TileHalo<T> TH = TileHalo<T>{}) {
  constexpr int BT = TN < 256 ? TN : 256;
  const int t = blockIdx.x;
  int tz0 = 0, tx0 = 0, ty0 = 0;
  bool cut = false;
  if (CUT) {
    tx0 = __ldg(TH.tiles + 3 * t) * g.ex;
    ty0 = __ldg(TH.tiles + 3 * t + 1) * g.ey;
    tz0 = __ldg(TH.tiles + 3 * t + 2) * g.ez;
    cut = tz0 == 0 || tz0 + g.ez >= g.nz;
  }
  const int lane = threadIdx.x & 31;
  const int srel = nbr_rel<T, TN>(nbr27, t, lane);
  const T* __restrict__ tb = pre + (size_t)t * (Q * TN);
  T* __restrict__ tp = post + (size_t)t * (Q * TN);
  const TileBricks tw(bmask, t, g, TN);
#pragma unroll 1
  for (int k = threadIdx.x - lane; k < tw.work; k += BT) {  // whole warps
    const int kk = k + lane;
    bool in;
    const int l = tw.slot(kk, in);
    const uint32_t w = tw.flag(flags, t, TN, l, in);
    const bool live = flag_type(w) != SOLID;
    const bool zfill = sector_needs_zero<T>(live) && g.zero_fill;
    const TileUpLUT up(lut, l);
    int off[Q];
#pragma unroll
    for (int i = 1; i < Q; ++i) off[i] = __shfl_sync(0xffffffffu, srel, up.code(i)) + up.loc(i);
    if (!live) {
      if (zfill && in) {
#pragma unroll
        for (int i = 0; i < Q; ++i) tp[up.p + i * TN] = (T)0;
      }
      continue;
    }
    const uint32_t miss = ~w & kMaskBits;
    T f[Q];
    f[0] = __ldg(tb + up.p);
#pragma unroll
    for (int i = 1; i < Q; ++i)
      f[i] = __ldg(tb + ((SEL && ((miss >> (opp(i) - 1)) & 1u)) ? up.p + opp(i) * TN : off[i] + i * TN));
    if (!SEL && miss) {
#pragma unroll
      for (int i = 1; i < Q; ++i)
        if ((miss >> (opp(i) - 1)) & 1u) f[i] = __ldg(tb + up.p + opp(i) * TN);
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
    for (int i = 0; i < Q; ++i) tp[up.p + i * TN] = f[i];
    if (CUT && cut) tile_ghost_push<T>(f, TH, g, x, y, z);
  }
}

#ifndef LBM_WL_WARPS
#define LBM_WL_WARPS 4
#endif
// warps per block of the work-list kernels (MINB is given per 8 warps);
// 4 measured 0-7 % faster than 8 or 2 (profiles/ab_warps_per_block_r01.txt)
constexpr int kWarpsPerBlock = LBM_WL_WARPS;

// ------------------------------------------------------------------ TMA
// Bulk-copy (TMA) primitives: 1-D cp.async.bulk global -> shared with
// mbarrier transaction counting, and the L2 bulk prefetch.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}

// one warp's share of the work list: {tile, brick index per lane group
// (bytes of words 1-2), uniform bits | count << 8}, decoded on the host
struct WarpItem {
  int t, l;
  bool in, uniform;
  template <typename T>
  __device__ __forceinline__ static WarpItem decode(const uint4 it, int lane, const Geo& g) {
    WarpItem W;
    const int lbn = g.lbx + g.lby + g.lbz;
    const int gi = lane >> lbn;  // brick group of this lane
    W.t = (int)it.x;
    W.in = gi < (int)((it.w >> 8) & 15u);
    const int b = (int)(((gi < 4 ? it.y : it.z) >> (8 * (gi & 3))) & 255u);
    W.l = (b << lbn) | (lane & ((1 << lbn) - 1));
    W.uniform = W.in && ((it.w >> gi) & 1u);
    return W;
  }
};

// Warp work list (the default for sparse tiles): one warp per group of
// live bricks of one tile (32 lanes = 4 fp32 / 8 fp64 bricks), so no lane
// idles for a tile's dead bricks and no CTA slot is held by a nearly empty
// tile.  The chain to the data loads is item -> (nbr27, slot table, flags)
// -> data.  Exact per-link select: masked links never fetch the upstream slot.
// CUT: z-slab ghost exchange for items of tiles on the first / last tile plane.
template <typename T, int TN, int MINB, bool CUT = false>
__global__ void __launch_bounds__(32 * kWarpsPerBlock, MINB * 8 / kWarpsPerBlock)
k_step_tiles_w(const T* __restrict__ pre, T* __restrict__ post, const uint32_t* __restrict__ flags,
               const int* __restrict__ nbr27, const T* __restrict__ bcv, const T* __restrict__ bcr, Geo g, T om,
               const uint4* __restrict__ items, int n_items, const ulonglong2* __restrict__ lut,
               const TileHalo<T> TH = TileHalo<T>{}) {
  const int wid = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (wid >= n_items) return;  // whole warps
  const WarpItem W = WarpItem::decode<T>(__ldg(items + wid), lane, g);
  const int t = W.t, l = W.l;
  const int srel = nbr_rel<T, TN>(nbr27, t, lane);
  const uint32_t w = W.uniform ? make_flag(kMaskBits, FLUID, 0, 0) : (W.in ? __ldg(flags + (size_t)t * TN + l) : 0u);
  const bool live = flag_type(w) != SOLID;
  const bool zfill = sector_needs_zero<T>(live) && g.zero_fill;
  const T* __restrict__ tb = pre + (size_t)t * (Q * TN);
  T* __restrict__ tp = post + (size_t)t * (Q * TN);
  // every lane must take part in the shuffles: dead lanes compute garbage
  // addresses they never use
  const TileUpLUT up(lut, l);
  int off[Q];
#pragma unroll
  for (int i = 1; i < Q; ++i) off[i] = __shfl_sync(0xffffffffu, srel, up.code(i)) + up.loc(i);
  if (!live) {
    if (zfill && W.in) {
#pragma unroll
      for (int i = 0; i < Q; ++i) tp[up.p + i * TN] = (T)0;
    }
    return;
  }
  const uint32_t miss = ~w & kMaskBits;
  T f[Q];
  f[0] = __ldg(tb + up.p);
#pragma unroll
  for (int i = 1; i < Q; ++i)
    f[i] = __ldg(tb + (((miss >> (opp(i) - 1)) & 1u) ? up.p + opp(i) * TN : off[i] + i * TN));
  int x = 0, y = 0, z = -1;
  bool cut = false;
  if (CUT) {
    const int tz0 = __ldg(TH.tiles + 3 * t + 2) * g.ez;
    cut = tz0 == 0 || tz0 + g.ez >= g.nz;
    if (cut) {
      brick_inv(g, l, x, y, z);
      x += __ldg(TH.tiles + 3 * t) * g.ex;
      y += __ldg(TH.tiles + 3 * t + 1) * g.ey;
      z += tz0;
      tile_ghost_gather<T>(f, miss, TH, g, x, y, z);
    }
  }
  bc_collide<T>(f, w, bcv, bcr, om);
#pragma unroll
  for (int i = 0; i < Q; ++i) tp[up.p + i * TN] = f[i];
  if (CUT && cut) tile_ghost_push<T>(f, TH, g, x, y, z);
}

// A-A z-slabs for tile layouts: like the dense A-A slabs, the neighbour
// step of a boundary node reads and writes the neighbouring slab's boundary
// plane directly in ITS tile storage (peer memory; its rank grid row of that
// tile plane locates the node), and mirrors the pushes into a 2 x 5-plane
// region appended to this slab's own buffer (offset Q * ps), where the
// phase-1 readback decoder (pre_index) finds them.  The node-local step needs
// nothing: the neighbour's pushes land in this slab's storage.
template <typename T>
struct TileAAHalo {
  T* f_lo;             // lower neighbour's tile storage (its top plane is plane lz_lo of tile plane row rank_lo)
  T* f_hi;             // upper neighbour's tile storage (its plane 0)
  const int* rank_lo;  // (gy, gx) ranks of the lower neighbour's top tile plane
  const int* rank_hi;  // (gy, gx) ranks of the upper neighbour's bottom tile plane
  int lz_lo;           // in-tile z of the lower neighbour's top plane
  T* mirror;           // own buffer + Q * ps: [kZm(j) x plane | kZp(j) x plane]
  const int* tiles;    // own tile coordinates
};

// element of direction d at node (x, y, plane lz of the given tile-plane row)
template <typename T>
__device__ __forceinline__ long long peer_tile_elem(const Geo& g, const int* __restrict__ rank_row, int x, int y,
                                                    int lz, int d) {
  if (x < 0) x += g.nx; else if (x >= g.nx) x -= g.nx;  // present links wrap only on periodic axes
  if (y < 0) y += g.ny; else if (y >= g.ny) y -= g.ny;
  const long long r = __ldg(rank_row + (y >> g.ley) * g.gx + (x >> g.lex));
  const int l = brick_x(g, x & (g.ex - 1)) + brick_y(g, y & (g.ey - 1)) + brick_z(g, lz);
  return (r * Q + d) * g.tn + l;
}

// pulls of a boundary node across the cut (replacing the meaningless values
// the in-slab gather produced for those links)
template <typename T>
__device__ __forceinline__ void tile_aa_cut_pull(T (&f)[Q], uint32_t miss, const TileAAHalo<T>& AH, const Geo& g,
                                                 int x, int y, int z) {
  if (z == 0 && AH.f_lo) {
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int i = kZp(j);  // c_z = +1: x - c_i is the lower neighbour's top plane, stored at F[opp(i)]
      if (!((miss >> (opp(i) - 1)) & 1u))
        f[i] = AH.f_lo[peer_tile_elem<T>(g, AH.rank_lo, x - cx(i), y - cy(i), AH.lz_lo, opp(i))];
    }
  }
  if (z == g.nz - 1 && AH.f_hi) {
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int i = kZm(j);
      if (!((miss >> (opp(i) - 1)) & 1u))
        f[i] = AH.f_hi[peer_tile_elem<T>(g, AH.rank_hi, x - cx(i), y - cy(i), 0, opp(i))];
    }
  }
}

// is push i of a node at z a cross-cut push (stored by tile_aa_cut_push, not in-slab)?
template <typename T>
__device__ __forceinline__ bool tile_aa_cut_link(const TileAAHalo<T>& AH, const Geo& g, int z, int i) {
  return (cz(i) == -1 && z == 0 && AH.f_lo) || (cz(i) == 1 && z == g.nz - 1 && AH.f_hi);
}

template <typename T>
__device__ __forceinline__ void tile_aa_cut_push(const T (&f)[Q], uint32_t miss, const TileAAHalo<T>& AH,
                                                 const Geo& g, int x, int y, int z) {
  const long long pn = (long long)g.nx * g.ny;
  if (z == 0 && AH.f_lo) {
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int i = kZm(j);
      if ((miss >> (i - 1)) & 1u) continue;
      AH.f_lo[peer_tile_elem<T>(g, AH.rank_lo, x + cx(i), y + cy(i), AH.lz_lo, i)] = f[i];
      AH.mirror[j * pn + ghost_row<T>(g, x + cx(i), y + cy(i))] = f[i];
    }
  }
  if (z == g.nz - 1 && AH.f_hi) {
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int i = kZp(j);
      if ((miss >> (i - 1)) & 1u) continue;
      AH.f_hi[peer_tile_elem<T>(g, AH.rank_hi, x + cx(i), y + cy(i), 0, i)] = f[i];
      AH.mirror[(5 + j) * pn + ghost_row<T>(g, x + cx(i), y + cy(i))] = f[i];
    }
  }
  __threadfence_system();
}

// A-A in place over the tile list (see k_step_dense_aa for the scheme):
// NB = 1 pulls F[opp(i)] at x - c_i and pushes to F[i] at x + c_i through
// the neighbour table; NB = 0 is node-local.
template <typename T, int TN, int NB, int MINB, bool CUT = false>
__global__ void __launch_bounds__(TN < 256 ? TN : 256, MINB)
k_step_tiles_aa(T* __restrict__ F, const uint32_t* __restrict__ flags, const int* __restrict__ nbr27,
                const T* __restrict__ bcv, const T* __restrict__ bcr, Geo g, T om,
                const uint32_t* __restrict__ bmask, const ulonglong2* __restrict__ lut,
                const TileAAHalo<T> AH = TileAAHalo<T>{}) {
  constexpr int BT = TN < 256 ? TN : 256;
  const int t = blockIdx.x;
  const int lane = threadIdx.x & 31;
  const int srel = NB ? nbr_rel<T, TN>(nbr27, t, lane) : 0;
  T* __restrict__ tb = F + (size_t)t * (Q * TN);
  const TileBricks tw(bmask, t, g, TN);
#pragma unroll 1
  for (int k = threadIdx.x - lane; k < tw.work; k += BT) {  // whole warps
    bool in;
    const int l = tw.slot(k + lane, in);
    const uint32_t w = tw.flag(flags, t, TN, l, in);
    const bool live = flag_type(w) != SOLID;  // no zero-fill under AA (see k_step_dense_aa)
    if (!NB) {
      if (!live) continue;
      const int p = l;
      T f[Q];
#pragma unroll
      for (int i = 0; i < Q; ++i) f[i] = LDA(tb + p + i * TN);
      bc_collide<T>(f, w, bcv, bcr, om);
#pragma unroll
      for (int i = 0; i < Q; ++i) tb[p + opp(i) * TN] = f[i];
      continue;
    }
    // neighbour step: the whole warp stays converged (solid lanes compute on
    // zeros and store nothing) so the offsets can be re-formed by shuffles
    // after the collision instead of being held in 18 registers
    const uint32_t miss = ~w & kMaskBits;
    T f[Q];
    {
      const TileUpLUT up(lut, l);
      f[0] = live ? LDA(tb + up.p) : (T)0;
#pragma unroll
      for (int i = 1; i < Q; ++i) {
        const int off = __shfl_sync(0xffffffffu, srel, up.code(i)) + up.loc(i);
        // exact per-link select: a masked link reads the node's own F[i]
        f[i] = live ? LDA(tb + (((miss >> (opp(i) - 1)) & 1u) ? up.p + i * TN : off + opp(i) * TN)) : (T)0;
      }
    }
    int x = 0, y = 0, z = -1;
    if (CUT) {
      brick_inv(g, l, x, y, z);
      x += __ldg(AH.tiles + 3 * t) * g.ex;
      y += __ldg(AH.tiles + 3 * t + 1) * g.ey;
      z += __ldg(AH.tiles + 3 * t + 2) * g.ez;
      if (live) tile_aa_cut_pull<T>(f, miss, AH, g, x, y, z);
    }
    bc_collide<T>(f, w, bcv, bcr, om);
    const int l2 = opaque(l);
    const TileUpLUT up2(lut, l2);
    if (live) tb[up2.p] = f[0];
#pragma unroll
    for (int i = 1; i < Q; ++i) {
      const int off = __shfl_sync(0xffffffffu, srel, up2.code(opp(i))) + up2.loc(opp(i));  // x + c_i
      const bool own = (miss >> (i - 1)) & 1u;
      if (live && (own || !CUT || !tile_aa_cut_link<T>(AH, g, z, i)))
        tb[own ? up2.p + opp(i) * TN : off + i * TN] = f[i];
    }
    if (CUT && live) tile_aa_cut_push<T>(f, miss, AH, g, x, y, z);
  }
}

// A-A over the warp work list (items as in k_step_tiles_w): same per-node
// work as k_step_tiles_aa, one warp per group of live bricks.  Any work
// distribution is race-free under A-A: a node reads and writes only its own
// slots (L) or the slots F[i][x + c_i] that only it reads (NB).
template <typename T, int TN, int NB, int MINB, bool CUT = false>
__global__ void __launch_bounds__(32 * kWarpsPerBlock, MINB * 8 / kWarpsPerBlock)
k_step_tiles_aa_w(T* __restrict__ F, const uint32_t* __restrict__ flags, const int* __restrict__ nbr27,
                  const T* __restrict__ bcv, const T* __restrict__ bcr, Geo g, T om, const uint4* __restrict__ items,
                  int n_items, const ulonglong2* __restrict__ lut, const TileAAHalo<T> AH = TileAAHalo<T>{}) {
  const int wid = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (wid >= n_items) return;  // whole warps
  const WarpItem W = WarpItem::decode<T>(__ldg(items + wid), lane, g);
  const int t = W.t, l = W.l;
  const int srel = NB ? nbr_rel<T, TN>(nbr27, t, lane) : 0;
  const uint32_t w = W.uniform ? make_flag(kMaskBits, FLUID, 0, 0) : (W.in ? __ldg(flags + (size_t)t * TN + l) : 0u);
  const bool live = flag_type(w) != SOLID;
  T* __restrict__ tb = F + (size_t)t * (Q * TN);
  if (!NB) {
    if (!live) return;
    const int p = l;
    T f[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) f[i] = LDA(tb + p + i * TN);
    bc_collide<T>(f, w, bcv, bcr, om);
#pragma unroll
    for (int i = 0; i < Q; ++i) tb[p + opp(i) * TN] = f[i];
    return;
  }
  const uint32_t miss = ~w & kMaskBits;
  T f[Q];
  {
    const TileUpLUT up(lut, l);
    f[0] = live ? LDA(tb + up.p) : (T)0;
#pragma unroll
    for (int i = 1; i < Q; ++i) {
      const int off = __shfl_sync(0xffffffffu, srel, up.code(i)) + up.loc(i);
      f[i] = live ? LDA(tb + (((miss >> (opp(i) - 1)) & 1u) ? up.p + i * TN : off + opp(i) * TN)) : (T)0;
    }
  }
  int x = 0, y = 0, z = -1;
  if (CUT) {
    brick_inv(g, l, x, y, z);
    x += __ldg(AH.tiles + 3 * t) * g.ex;
    y += __ldg(AH.tiles + 3 * t + 1) * g.ey;
    z += __ldg(AH.tiles + 3 * t + 2) * g.ez;
    if (live) tile_aa_cut_pull<T>(f, miss, AH, g, x, y, z);
  }
  bc_collide<T>(f, w, bcv, bcr, om);
  const int l2 = opaque(l);
  const TileUpLUT up2(lut, l2);
  if (live) tb[up2.p] = f[0];
#pragma unroll
  for (int i = 1; i < Q; ++i) {
    const int off = __shfl_sync(0xffffffffu, srel, up2.code(opp(i))) + up2.loc(opp(i));  // x + c_i
    const bool own = (miss >> (i - 1)) & 1u;
    if (live && (own || !CUT || !tile_aa_cut_link<T>(AH, g, z, i)))
      tb[own ? up2.p + opp(i) * TN : off + i * TN] = f[i];
  }
  if (CUT && live) tile_aa_cut_push<T>(f, miss, AH, g, x, y, z);
}

// TMA-staged tiles (variant 9; the north star's "TMA tile staging"):
// persistent CTAs walk the tile list (tile = blockIdx.x + k * gridDim.x)
// through an S-stage ring of tile images in shared memory.  For each tile,
// warp 0 arms the stage's mbarrier with the tile's live bytes and its lanes
// issue one cp.async.bulk per (direction, run of consecutive live bricks) --
// 19 copies of 2 KB for a full tile -- S - 1 tiles ahead of the compute, so
// the tile's own data is in flight without registers or LSU slots.  Dead
// bricks are never copied (their nodes are solid: masked links).  In-tile
// pulls read the stage, pulls across the tile faces read global memory,
// stores go straight to the post buffer.  Measured slower than the direct
// kernels (profiles/sparse_r02.md): 8-16 warps per SM leave the face loads'
// latency exposed, and every tile costs a CTA barrier.
template <typename T, int TN>
struct TmaCfg {
  static constexpr int BN = Rec<T>::BN;
  static constexpr int NB = TN / BN;                 // bricks per tile
  static constexpr int STAGE = Q * TN;               // elements per stage (a tile image)
  static constexpr int S = 2;
  static constexpr int THREADS = 256;
  static constexpr size_t SMEM = (size_t)S * STAGE * sizeof(T) + 16 * S;
};

template <typename T, int TN>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? 2 : 1)
k_step_tiles_tma(const T* __restrict__ pre, T* __restrict__ post, const uint32_t* __restrict__ flags,
                 const int* __restrict__ nbr27, const T* __restrict__ bcv, const T* __restrict__ bcr, Geo g, T om,
                 const uint32_t* __restrict__ bmask, const ulonglong2* __restrict__ lut, int n_tiles) {
  using C = TmaCfg<T, TN>;
  constexpr int BN = C::BN, S = C::S;
  extern __shared__ __align__(128) unsigned char tma_smem[];
  T* const stage0 = reinterpret_cast<T*>(tma_smem);
  unsigned long long* const full = reinterpret_cast<unsigned long long*>(tma_smem + (size_t)S * C::STAGE * sizeof(T));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  // warp 0: arm stage (k % S) and copy the live bricks of this CTA's k-th tile
  auto issue = [&](int k) {
    const int t = blockIdx.x + k * gridDim.x;
    if (t >= n_tiles) return;
    const int s = k % S;
    uint32_t m[4];
    int live = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      m[q] = __ldg(bmask + 8LL * t + q);
      live += __popc(m[q]);
    }
    if (lane == 0) mbar_expect_tx(&full[s], (unsigned)(live * Q * BN * (int)sizeof(T)));
    __syncwarp();
    const T* src = pre + (size_t)t * (Q * TN);
    T* dst = stage0 + (size_t)s * C::STAGE;
#pragma unroll
    for (int q = 0; q < (C::NB + 31) / 32; ++q) {
      // lane j starts a run if brick 32q + j is live and its predecessor in the word is not
      const uint32_t mq = m[q];
      const bool start = ((mq >> lane) & 1u) && (lane == 0 || !((mq >> (lane - 1)) & 1u));
      if (start) {
        const uint32_t rest = ~(mq >> lane);         // zeros shifted in above bit 31 - lane
        const int len = rest ? __ffs(rest) - 1 : 32;  // consecutive live bricks from lane (32: a full word)
        const int b0 = q * 32 + lane;
        for (int i = 0; i < Q; ++i)
          bulk_g2s(dst + i * TN + b0 * BN, src + i * TN + b0 * BN, (unsigned)(len * BN * sizeof(T)), &full[s]);
      }
    }
  };
  if (warp == 0)
    for (int k = 0; k < S - 1; ++k) issue(k);
#pragma unroll 1
  for (int k = 0;; ++k) {
    const int t = blockIdx.x + k * gridDim.x;
    if (t >= n_tiles) break;
    if (warp == 0) issue(k + S - 1);  // into the stage released at the end of k - 1
    const int s = k % S;
    const T* __restrict__ sb = stage0 + (size_t)s * C::STAGE;
    const int srel = nbr_rel<T, TN>(nbr27, t, lane);
    const T* __restrict__ tb = pre + (size_t)t * (Q * TN);
    T* __restrict__ tp = post + (size_t)t * (Q * TN);
    const TileBricks tw(bmask, t, g, TN);
    mbar_wait(&full[s], (unsigned)((k / S) & 1));
#pragma unroll 1
    for (int kk = threadIdx.x - lane; kk < tw.work; kk += C::THREADS) {  // whole warps
      bool in;
      const int l = tw.slot(kk + lane, in);
      const uint32_t w = tw.flag(flags, t, TN, l, in);
      const bool live = flag_type(w) != SOLID;
      const bool zfill = sector_needs_zero<T>(live) && g.zero_fill;
      const TileUpLUT up(lut, l);
      int off[Q];
      uint32_t intile = 0u;  // bit i: the node x - c_i lies in this tile (read the stage)
#pragma unroll
      for (int i = 1; i < Q; ++i) {
        const int c = up.code(i), loc = up.loc(i);
        const int rel = __shfl_sync(0xffffffffu, srel, c);  // all lanes take part
        intile |= (c == 13 ? 1u : 0u) << i;
        off[i] = c == 13 ? loc : rel + loc;
      }
      if (!live) {
        if (zfill && in) {
#pragma unroll
          for (int i = 0; i < Q; ++i) tp[l + i * TN] = (T)0;
        }
        continue;
      }
      const uint32_t miss = ~w & kMaskBits;
      T f[Q];
      f[0] = sb[l];
#pragma unroll
      for (int i = 1; i < Q; ++i) {
        if ((miss >> (opp(i) - 1)) & 1u)
          f[i] = sb[l + opp(i) * TN];
        else if ((intile >> i) & 1u)
          f[i] = sb[off[i] + i * TN];
        else
          f[i] = __ldg(tb + off[i] + i * TN);
      }
      bc_collide<T>(f, w, bcv, bcr, om);
#pragma unroll
      for (int i = 0; i < Q; ++i) tp[l + i * TN] = f[i];
    }
    __syncthreads();  // stage s is free again
  }
}
