// Device geometry pipeline: flag words (layouts.py:173-188 on the device),
// tile keep/compaction/neighbour table (layouts.py:263-269, 389-401 in 3-D),
// launch-order keys, uniform-chunk and live-brick masks.
// Part of liblbm19 (included once, in order, by lbm19.cu).
#pragma once

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
  if (z < 0) return glo ? glo[(long long)y * g.nx + x] & 7u : SOLID;
  if (z >= g.nz) return ghi ? ghi[(long long)y * g.nx + x] & 7u : SOLID;
  return type[((long long)z * g.ny + y) * g.nx + x] & 7u;
}

// descriptors as uploaded (packed and range-checked on the host, lbm19.cu
// upload_descriptors): type | orientation << 3, and the bc index byte
__device__ __forceinline__ uint32_t node_flag(const uint8_t* __restrict__ type,
                                              const uint8_t* __restrict__ bcb,
                                              const uint8_t* __restrict__ glo,
                                              const uint8_t* __restrict__ ghi, const Geo& g,
                                              int x, int y, int z) {
  const long long n = ((long long)z * g.ny + y) * g.nx + x;
  const uint32_t t = type[n] & 7u;
  const uint32_t o = type[n] >> 3;
  const uint32_t b = bcb[n];
  uint32_t m = 0;
  if (t != SOLID) {
#pragma unroll
    for (int j = 1; j < Q; ++j)
      if (type_at(type, glo, ghi, g, x + cx(j), y + cy(j), z + cz(j)) != SOLID) m |= 1u << (j - 1);
  }
  return make_flag(m, t, o, b);
}

// dense: one thread per (padded) flag entry
__global__ void k_flags_dense(uint32_t* __restrict__ flags, const uint8_t* __restrict__ type,
                              const uint8_t* __restrict__ bcb,
                              const uint8_t* __restrict__ glo, const uint8_t* __restrict__ ghi,
                              Geo g, unsigned long long* nonsolid) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = blockIdx.z;
  if (x >= g.nxp) return;
  uint32_t w = 0;
  if (x < g.nx) w = node_flag(type, bcb, glo, ghi, g, x, y, z);
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
      if (x < g.nx && y < g.ny && z < g.nz && (type[((long long)z * g.ny + y) * g.nx + x] & 7u) != SOLID) any = 1;
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


// tiles: one thread per slot of the kept tiles
__global__ void k_flags_tile(uint32_t* __restrict__ flags, const int* __restrict__ tiles,
                             const uint8_t* __restrict__ type, const uint8_t* __restrict__ bcb,
                             const uint8_t* __restrict__ glo,
                             const uint8_t* __restrict__ ghi, Geo g, long long nslots,
                             unsigned long long* nonsolid) {
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
    if (x < g.nx && y < g.ny && z < g.nz) w = node_flag(type, bcb, glo, ghi, g, x, y, z);
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
