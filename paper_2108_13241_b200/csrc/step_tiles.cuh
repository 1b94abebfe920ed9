// Sparse tile step kernels (AoSoA tiles, nbr27, live bricks): AB variants,
// z-slab ghost exchange, warp work list, shared-memory staging, A-A.
// Part of liblbm19 (included once, in order, by lbm19.cu).
#pragma once

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

// The same offsets from a per-slot table (one u64 per in-tile slot, built
// on the host for the handle's tile shape, L1-resident): bits 0-53 hold the
// six in-tile brick-order deltas' magnitudes (9 bits each: x-, x+, y-, y+,
// z-, z+), bits 54-59 whether the neighbour lies across the tile face (the
// delta is then positive -- a wrap inside the neighbour tile -- else
// negative for "-" and positive for "+").
struct TileUpLUT {
  int l, dxm, dxp, dym, dyp, dzm, dzp, cxm, cxp, cym, cyp, czm, czp;
  __device__ __forceinline__ TileUpLUT(const unsigned long long* __restrict__ lut, int slot) : l(slot) {
    const unsigned long long e = __ldg(lut + slot);
    const int mag[6] = {(int)(e & 511), (int)(e >> 9 & 511), (int)(e >> 18 & 511), (int)(e >> 27 & 511),
                        (int)(e >> 36 & 511), (int)(e >> 45 & 511)};
    const unsigned cr = (unsigned)(e >> 54) & 63u;
    dxm = (cr & 1) ? mag[0] : -mag[0];
    dxp = mag[1] * ((cr & 2) ? -1 : 1);
    dym = (cr & 4) ? mag[2] : -mag[2];
    dyp = mag[3] * ((cr & 8) ? -1 : 1);
    dzm = (cr & 16) ? mag[4] : -mag[4];
    dzp = mag[5] * ((cr & 32) ? -1 : 1);
    cxm = (cr & 1) ? -1 : 0, cxp = (cr & 2) ? 1 : 0;
    cym = (cr & 4) ? -3 : 0, cyp = (cr & 8) ? 3 : 0;
    czm = (cr & 16) ? -9 : 0, czp = (cr & 32) ? 9 : 0;
  }
  __device__ __forceinline__ int code(int i) const {
    return 13 + (cx(i) == 1 ? cxm : (cx(i) == -1 ? cxp : 0)) + (cy(i) == 1 ? cym : (cy(i) == -1 ? cyp : 0)) +
           (cz(i) == 1 ? czm : (cz(i) == -1 ? czp : 0));
  }
  __device__ __forceinline__ int loc(int i) const {
    return l + (cx(i) == 1 ? dxm : (cx(i) == -1 ? dxp : 0)) + (cy(i) == 1 ? dym : (cy(i) == -1 ? dyp : 0)) +
           (cz(i) == 1 ? dzm : (cz(i) == -1 ? dzp : 0));
  }
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

// MODE 7: the live-brick CTA-per-tile kernel without the shared-memory
// neighbour table and its block barrier: every warp keeps the 27 relative
// tile offsets in lanes 0-26 and fetches them with shuffles (all lanes take
// part, so the offsets are formed before dead lanes leave the iteration).
template <typename T, int TN, int MINB, bool SEL = false, bool CUT = false>
__global__ void __launch_bounds__(TN < 256 ? TN : 256, MINB)
k_step_tiles_x(const T* __restrict__ pre, T* __restrict__ post, const uint32_t* __restrict__ flags,
               const int* __restrict__ nbr27, const T* __restrict__ bcv, const T* __restrict__ bcr, Geo g, T om,
               const uint32_t* __restrict__ bmask, const unsigned long long* __restrict__ lut,
               const TileHalo<T> TH = TileHalo<T>{}) {
  constexpr int BT = TN < 256 ? TN : 256;
  const int t = blockIdx.x;
  // z-slab cut (CUT): tiles on the first / last tile plane exchange their
  // boundary nodes' c_z populations through ghost planes (uniform per CTA)
  int tz0 = 0, tx0 = 0, ty0 = 0;
  bool cut = false;
  if (CUT) {
    tx0 = __ldg(TH.tiles + 3 * t) * g.ex;
    ty0 = __ldg(TH.tiles + 3 * t + 1) * g.ey;
    tz0 = __ldg(TH.tiles + 3 * t + 2) * g.ez;
    cut = tz0 == 0 || tz0 + g.ez >= g.nz;
  }
  const int lane = threadIdx.x & 31;
  int srel = 0;
  if (lane < 27) {
    const int v = __ldg(nbr27 + 27LL * t + lane);
    srel = v < 0 ? 0 : (v - t) * (Q * TN);
  }
  const T* __restrict__ tb = pre + (size_t)t * (Q * TN);
  T* __restrict__ tp = post + (size_t)t * (Q * TN);
  const TileBricks tw(bmask, t, g, TN, true);
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
        for (int i = 0; i < Q; ++i) tp[i * TN + l] = (T)0;
      }
      continue;
    }
    const uint32_t miss = ~w & kMaskBits;
    T f[Q];
    f[0] = __ldg(tb + l);
#pragma unroll
    for (int i = 1; i < Q; ++i)  // SEL: masked links never fetch the (solid) upstream slot
      f[i] = __ldg(tb + ((SEL && ((miss >> (opp(i) - 1)) & 1u)) ? opp(i) * TN + l : i * TN + off[i]));
    if (!SEL && miss) {
#pragma unroll
      for (int i = 1; i < Q; ++i)
        if ((miss >> (opp(i) - 1)) & 1u) f[i] = __ldg(tb + opp(i) * TN + l);
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

#ifndef LBM_WL_WARPS
#define LBM_WL_WARPS 4
#endif
// warps per block of the work-list kernels (MINB is given per 8 warps);
// 4 measured 0-7 % faster than 8 or 2 (profiles/ab_warps_per_block_r01.txt)
constexpr int kWarpsPerBlock = LBM_WL_WARPS;

// Warp work list (MODE 5/8): one warp per group of live bricks of one tile
// (32 lanes = 4 fp32 / 8 fp64 bricks), so no lane idles for a tile's dead
// bricks or its last partial pass and no CTA slot is held by a nearly empty
// tile.  Each item is pre-decoded on the host: {tile, brick index per lane
// group (bytes of words 1-2), uniform bits | count << 8}; the chain to the
// data loads is item -> (nbr27, slot table, flags) -> data.  The 27
// neighbour offsets live in lanes 0-26 and are fetched with shuffles.
template <typename T, int TN, int MINB, bool SEL = false>
__global__ void __launch_bounds__(32 * kWarpsPerBlock, MINB * 8 / kWarpsPerBlock)
k_step_tiles_w(const T* __restrict__ pre, T* __restrict__ post, const uint32_t* __restrict__ flags,
               const int* __restrict__ nbr27, const T* __restrict__ bcv, const T* __restrict__ bcr, Geo g, T om,
               const uint4* __restrict__ items, int n_items, const unsigned long long* __restrict__ lut) {
  const int wid = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (wid >= n_items) return;  // whole warps
  const uint4 it = __ldg(items + wid);
  const int t = (int)it.x;
  int srel = 0;
  if (lane < 27) {
    const int v = __ldg(nbr27 + 27LL * t + lane);
    srel = v < 0 ? 0 : (v - t) * (Q * TN);
  }
  const int lbn = g.lbx + g.lby + g.lbz, bn = 1 << lbn;
  const int gi = lane >> lbn;  // brick group of this lane
  const bool in = gi < (int)((it.w >> 8) & 15u);
  const int b = (int)(((gi < 4 ? it.y : it.z) >> (8 * (gi & 3))) & 255u);
  const int l = (b << lbn) | (lane & (bn - 1));
  const bool uniform = in && ((it.w >> gi) & 1u);
  const uint32_t w = uniform ? make_flag(kMaskBits, FLUID, 0, 0) : (in ? __ldg(flags + (size_t)t * TN + l) : 0u);
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
  for (int i = 1; i < Q; ++i)  // SEL: masked links never fetch the (solid) upstream slot
    f[i] = __ldg(tb + ((SEL && ((miss >> (opp(i) - 1)) & 1u)) ? opp(i) * TN + l : i * TN + off[i]));
  if (!SEL && miss) {
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
                const uint32_t* __restrict__ bmask, const int* __restrict__ order,
                const unsigned long long* __restrict__ lut) {
  constexpr int BT = TN < 256 ? TN : 256;
  const int t = order ? __ldg(order + blockIdx.x) : (int)blockIdx.x;
  const int lane = threadIdx.x & 31;
  // neighbour ranks in lanes 0-26 (shuffles; no shared table, no barrier)
  int srel = 0;
  if (NB && lane < 27) {
    const int v = __ldg(nbr27 + 27LL * t + lane);
    srel = v < 0 ? 0 : (v - t) * (Q * TN);
  }
  T* __restrict__ tb = F + (size_t)t * (Q * TN);
  const TileBricks tw(bmask, t, g, TN, true);
#pragma unroll 1
  for (int k = threadIdx.x - lane; k < tw.work; k += BT) {  // whole warps
    bool in;
    const int l = tw.slot(k + lane, in);
    const uint32_t w = tw.flag(flags, t, TN, l, in);
    const bool live = flag_type(w) != SOLID;  // no zero-fill under AA (see k_step_dense_aa)
    if (!NB) {
      if (!live) continue;
      T f[Q];
#pragma unroll
      for (int i = 0; i < Q; ++i) f[i] = LDA(tb + i * TN + l);
      bc_collide<T>(f, w, bcv, bcr, om);
#pragma unroll
      for (int i = 0; i < Q; ++i) tb[opp(i) * TN + l] = f[i];
      continue;
    }
    // neighbour step: the whole warp stays converged (solid lanes compute on
    // zeros and store nothing) so the offsets can be re-formed by shuffles
    // after the collision instead of being held in 18 registers
    const uint32_t miss = ~w & kMaskBits;
    T f[Q];
    {
      const TileUpLUT up(lut, l);
      f[0] = live ? LDA(tb + l) : (T)0;
#pragma unroll
      for (int i = 1; i < Q; ++i) {
        const int off = __shfl_sync(0xffffffffu, srel, up.code(i)) + up.loc(i);
        // exact per-link select: a masked link reads the node's own F[i]
        f[i] = live ? LDA(tb + (((miss >> (opp(i) - 1)) & 1u) ? i * TN + l : opp(i) * TN + off)) : (T)0;
      }
    }
    bc_collide<T>(f, w, bcv, bcr, om);
    const int l2 = opaque(l);
    const TileUpLUT up2(lut, l2);
    if (live) tb[l2] = f[0];
#pragma unroll
    for (int i = 1; i < Q; ++i) {
      const int off = __shfl_sync(0xffffffffu, srel, up2.code(opp(i))) + up2.loc(opp(i));  // x + c_i
      if (live) tb[((miss >> (i - 1)) & 1u) ? opp(i) * TN + l2 : i * TN + off] = f[i];
    }
  }
}

// A-A over the warp work list (items as in k_step_tiles_w): same per-node
// work as k_step_tiles_aa, one warp per group of live bricks.  Any work
// distribution is race-free under A-A: a node reads and writes only its own
// slots (L) or the slots F[i][x + c_i] that only it reads (NB).
template <typename T, int TN, int NB, int MINB>
__global__ void __launch_bounds__(32 * kWarpsPerBlock, MINB * 8 / kWarpsPerBlock)
k_step_tiles_aa_w(T* __restrict__ F, const uint32_t* __restrict__ flags, const int* __restrict__ nbr27,
                  const T* __restrict__ bcv, const T* __restrict__ bcr, Geo g, T om, const uint4* __restrict__ items,
                  int n_items, const unsigned long long* __restrict__ lut) {
  const int wid = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (wid >= n_items) return;  // whole warps
  const uint4 it = __ldg(items + wid);
  const int t = (int)it.x;
  int srel = 0;
  if (NB && lane < 27) {
    const int v = __ldg(nbr27 + 27LL * t + lane);
    srel = v < 0 ? 0 : (v - t) * (Q * TN);
  }
  const int lbn = g.lbx + g.lby + g.lbz, bn = 1 << lbn;
  const int gi = lane >> lbn;
  const bool in = gi < (int)((it.w >> 8) & 15u);
  const int b = (int)(((gi < 4 ? it.y : it.z) >> (8 * (gi & 3))) & 255u);
  const int l = (b << lbn) | (lane & (bn - 1));
  const bool uniform = in && ((it.w >> gi) & 1u);
  const uint32_t w = uniform ? make_flag(kMaskBits, FLUID, 0, 0) : (in ? __ldg(flags + (size_t)t * TN + l) : 0u);
  const bool live = flag_type(w) != SOLID;
  T* __restrict__ tb = F + (size_t)t * (Q * TN);
  if (!NB) {
    if (!live) return;
    T f[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) f[i] = LDA(tb + i * TN + l);
    bc_collide<T>(f, w, bcv, bcr, om);
#pragma unroll
    for (int i = 0; i < Q; ++i) tb[opp(i) * TN + l] = f[i];
    return;
  }
  const uint32_t miss = ~w & kMaskBits;
  T f[Q];
  {
    const TileUpLUT up(lut, l);
    f[0] = live ? LDA(tb + l) : (T)0;
#pragma unroll
    for (int i = 1; i < Q; ++i) {
      const int off = __shfl_sync(0xffffffffu, srel, up.code(i)) + up.loc(i);
      f[i] = live ? LDA(tb + (((miss >> (opp(i) - 1)) & 1u) ? i * TN + l : opp(i) * TN + off)) : (T)0;
    }
  }
  bc_collide<T>(f, w, bcv, bcr, om);
  const int l2 = opaque(l);
  const TileUpLUT up2(lut, l2);
  if (live) tb[l2] = f[0];
#pragma unroll
  for (int i = 1; i < Q; ++i) {
    const int off = __shfl_sync(0xffffffffu, srel, up2.code(opp(i))) + up2.loc(opp(i));  // x + c_i
    if (live) tb[((miss >> (i - 1)) & 1u) ? opp(i) * TN + l2 : i * TN + off] = f[i];
  }
}
