// Dense step kernels: the fused pull gather / bounce-back / Zou-He / BGK /
// store (kernel.py:72-141) for AB and A-A, plus the z-slab halo kernels.
// Part of liblbm19 (included once, in order, by lbm19.cu).
#pragma once

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
  int zmode; // planes this launch covers: 0 all, 1 the two boundary planes, 2 the interior
};

// z of this block under a Halo's zmode (boundary planes first on z-slabs,
// so the neighbours may start their next step while the interior runs)
__device__ __forceinline__ int slab_z(int bz, int zmode, int nz) {
  return zmode == 0 ? bz : (zmode == 1 ? (bz ? nz - 1 : 0) : bz + 1);
}

// Ordering words (device memory): sync[0] written by the lower neighbour,
// sync[1] by the upper one, sync[2] this slab's own epoch.  The epoch lives
// on the device, so wait / step / signal sequences replay from a CUDA graph.
__global__ void k_halo_wait(const unsigned long long* sync, int need_lo, int need_hi, int* err) {
  const long long t0 = clock64();
  const volatile unsigned long long* vs = sync;
  const unsigned long long target = vs[2];
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
                              unsigned long long* own) {
  const unsigned long long value = *own + 1;
  *own = value;
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
  // slot of (x, y - cy_i, z - cz_i): the y / z part of up()
  __device__ __forceinline__ unsigned up_yz(unsigned s, int i) const {
    return s + (cy(i) == 1 ? ym : (cy(i) == -1 ? yp : 0u)) + (cz(i) == 1 ? zm : (cz(i) == -1 ? zp : 0u));
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
  const int y = blockIdx.y, z = slab_z(blockIdx.z, H.zmode, g.nz);
  if (x >= g.nxp) return;  // whole warps (nxp % 32 == 0)
  // 32-bit unsigned slot arithmetic (slabs up to 2^32 slots; negative
  // offsets wrap modulo 2^32 and land on the right slot)
  const unsigned fi = ((unsigned)z * g.ny + y) * g.nxp + x;
  const unsigned s = fi + (unsigned)g.plane;
  const uint32_t ub = __ldg(ubits + (fi >> 10));
  const bool uni = (ub >> ((fi >> 5) & 31)) & 1u;  // warp-uniform: one chunk = one warp
  if (uni && !((z == 0 && H.lo[0]) || (z == g.nz - 1 && H.hi[0]))) {
    // uniform chunk (all FLUID / wall, full masks) off the halo planes: no
    // flag word, no bounce-back, no closure, no zero fill -- the same
    // arithmetic as the general path below, without its control flow
    const UpOffsets o(g, x, y, z);
    T f[Q];
    f[0] = __ldg(P.pre[0] + s);
#pragma unroll
    for (int i = 1; i < Q; ++i) f[i] = __ldg(P.pre[i] + o.up(s, i));
    T rho, vx, vy, vz;
    moments19(f, rho, vx, vy, vz);
    collide19(f, rho, vx, vy, vz, om);
#pragma unroll
    for (int i = 0; i < Q; ++i) P.post[i][s] = f[i];
    return;
  }
  const uint32_t w = uni ? make_flag(kMaskBits, FLUID, 0, 0) : __ldg(flags + fi);
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

#ifdef LBM_EXPERIMENTS
// Dense AB step with 128-bit accesses: four consecutive x-nodes per thread,
// 19 LDG.128 + 19 STG.128 per quad.  Directions with c_x = 0 load the
// upstream quad directly; c_x = +-1 load the aligned quad of the upstream row
// and take the one element that crosses into the neighbouring quad from the
// adjacent lane (__shfl_up/down), or from memory at warp ends.  Closed-x edge
// values are masked links and are replaced by the bounce-back fix-up; on a
// periodic x axis the wrapped elements are reloaded.  fp32 only, no halo.
template <int MINB>
__global__ void __launch_bounds__(128, MINB)
k_step_dense_v4(const Planes<float> P, const uint32_t* __restrict__ flags, const uint32_t* __restrict__ ubits,
                const float* __restrict__ bcv, const float* __restrict__ bcr, Geo g, float om) {
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int x0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const int y = blockIdx.y, z = blockIdx.z;
  const bool act = x0 < g.nxp;
  const unsigned fi = ((unsigned)z * g.ny + y) * g.nxp + (act ? x0 : 0);
  const unsigned s = fi + (unsigned)g.plane;
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  if (act) {
    const uint32_t ub = __ldg(ubits + (fi >> 10));
    if ((ub >> ((fi >> 5) & 31)) & 1u) {
#pragma unroll
      for (int k = 0; k < 4; ++k) w[k] = make_flag(kMaskBits, FLUID, 0, 0);
    } else {
      const uint4 fw = __ldg(reinterpret_cast<const uint4*>(flags + fi));
      w[0] = fw.x, w[1] = fw.y, w[2] = fw.z, w[3] = fw.w;
    }
  }
  bool any = false;
#pragma unroll
  for (int k = 0; k < 4; ++k) any |= flag_type(w[k]) != SOLID;
  // the other quad of this quad's 32-B sector sits in lane ^ 1
  const bool partner = __shfl_xor_sync(FULL, (int)any, 1) != 0;
  const UpOffsets o(g, 0, y, z);
  float4 v[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const unsigned r = s + (cy(i) == 1 ? o.ym : (cy(i) == -1 ? o.yp : 0u)) + (cz(i) == 1 ? o.zm : (cz(i) == -1 ? o.zp : 0u));
    const float4 a = __ldg(reinterpret_cast<const float4*>(P.pre[i] + r));
    if (cx(i) == 0) {
      v[i] = a;
    } else if (cx(i) == 1) {  // upstream x - 1
      float pw = __shfl_up_sync(FULL, a.w, 1);
      if (lane == 0) pw = (act && x0 > 0) ? __ldg(P.pre[i] + r - 1) : 0.f;
      if (g.px && x0 == 0 && act) pw = __ldg(P.pre[i] + r + (g.nx - 1));
      v[i] = make_float4(pw, a.x, a.y, a.z);
    } else {                 // upstream x + 1
      float nx_ = __shfl_down_sync(FULL, a.x, 1);
      if (lane == 31) nx_ = (act && x0 + 4 < g.nxp) ? __ldg(P.pre[i] + r + 4) : 0.f;
      v[i] = make_float4(a.y, a.z, a.w, nx_);
      if (g.px && act && x0 <= g.nx - 1 && g.nx - 1 < x0 + 4) {
        const float wv = __ldg(P.pre[i] + r - x0);  // x = 0 of the upstream row
        const int k = g.nx - 1 - x0;
        if (k == 0) v[i].x = wv; else if (k == 1) v[i].y = wv; else if (k == 2) v[i].z = wv; else v[i].w = wv;
      }
    }
  }
  if (!act || !(any || (partner && g.zero_fill))) return;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float f[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) f[i] = k == 0 ? v[i].x : (k == 1 ? v[i].y : (k == 2 ? v[i].z : v[i].w));
    const uint32_t wk = w[k];
    if (flag_type(wk) != SOLID) {
      const uint32_t miss = ~wk & kMaskBits;
      if (miss) {
#pragma unroll
        for (int i = 1; i < Q; ++i)
          if ((miss >> (opp(i) - 1)) & 1u) f[i] = __ldg(P.pre[opp(i)] + s + k);
      }
      bc_collide<float>(f, wk, bcv, bcr, om);
    } else {
#pragma unroll
      for (int i = 0; i < Q; ++i) f[i] = 0.f;  // solid: storage stays 0 (full-sector stores)
    }
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      if (k == 0) v[i].x = f[i]; else if (k == 1) v[i].y = f[i]; else if (k == 2) v[i].z = f[i]; else v[i].w = f[i];
    }
  }
#pragma unroll
  for (int i = 0; i < Q; ++i) *reinterpret_cast<float4*>(P.post[i] + s) = v[i];
}
#endif  // LBM_EXPERIMENTS

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

// z-slabs under A-A: the neighbour step of a boundary plane reads and writes
// the neighbouring slab's boundary plane directly (peer memory, H.hi = the
// upper slab's plane 0, c_z = +1 directions; H.lo = the lower slab's top
// plane, c_z = -1 directions).  By the single-owner property these locations
// belong to this thread alone within the step; the per-step wait/signal
// orders them against the neighbours' node-local steps.  The pushes are also
// mirrored into this slab's own ghost plane, where the phase-1 readback
// decoder (pre_index) finds them.
template <typename T>
__device__ __forceinline__ unsigned peer_row(const Geo& g, int x, int y) {
  if (x < 0) x += g.nx; else if (x >= g.nx) x -= g.nx;  // present links wrap only on periodic axes
  if (y < 0) y += g.ny; else if (y >= g.ny) y -= g.ny;
  return (unsigned)y * g.nxp + x;
}

template <typename T, int NB, int MINB>
__global__ void __launch_bounds__(128, MINB) k_step_dense_aa(const Planes1<T> P, const uint32_t* __restrict__ flags,
                                                      const uint32_t* __restrict__ ubits,
                                                      const T* __restrict__ bcv, const T* __restrict__ bcr,
                                                      Geo g, T om, const Halo<T> H) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, z = slab_z(blockIdx.z, H.zmode, g.nz);
  if (x >= g.nxp) return;
  const unsigned fi = ((unsigned)z * g.ny + y) * g.nxp + x;
  const unsigned s = fi + (unsigned)g.plane;
  const uint32_t ub = __ldg(ubits + (fi >> 10));
  const bool uni = (ub >> ((fi >> 5) & 31)) & 1u;  // warp-uniform: one chunk = one warp
  if (NB && uni && !((z == 0 && H.lo[0]) || (z == g.nz - 1 && H.hi[0]))) {
    // uniform chunk (all FLUID / wall, full masks) off the slab cut: every
    // link present, no closure -- the arithmetic of the general path below
    // without its selects and fix-ups
    const UpOffsets o(g, x, y, z);
    T f[Q];
    f[0] = LDA(P.f[0] + s);
#pragma unroll
    for (int i = 1; i < Q; ++i) f[i] = LDA(P.f[opp(i)] + o.up(s, i));
    T rho, vx, vy, vz;
    moments19(f, rho, vx, vy, vz);
    collide19(f, rho, vx, vy, vz, om);
    const unsigned s2 = opaque(s);
    const UpOffsets o2(g, opaque(x), opaque(y), opaque(z));
    P.f[0][s2] = f[0];
#pragma unroll
    for (int i = 1; i < Q; ++i) P.f[i][o2.up(s2, opp(i))] = f[i];
    return;
  }
  const uint32_t w = uni ? make_flag(kMaskBits, FLUID, 0, 0) : __ldg(flags + fi);
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
    const bool top = z == g.nz - 1 && H.hi[0], bot = z == 0 && H.lo[0];
    if (top || bot) {
      // upstream across the cut: the neighbour slab's boundary plane
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        if (top) {
          const int i = kZm(j);  // c_z = -1: pulls from z + 1, stored at F_U[opp(i) = kZp(j)]
          if (!((miss >> (opp(i) - 1)) & 1u)) f[i] = H.hi[j][peer_row<T>(g, x - cx(i), y - cy(i))];
        }
        if (bot) {
          const int i = kZp(j);  // c_z = +1: pulls from z - 1, stored at F_L[opp(i) = kZm(j)]
          if (!((miss >> (opp(i) - 1)) & 1u)) f[i] = H.lo[j][peer_row<T>(g, x - cx(i), y - cy(i))];
        }
      }
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
    if (top || bot) {
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        if (top) {
          const int i = kZp(j);  // pushed into the upper slab's plane 0 (the ghost copy stays as a mirror)
          if ((miss >> (i - 1)) & 1u) continue;
          H.hi[j][peer_row<T>(g, x + cx(i), y + cy(i))] = f[i];
        }
      }
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        if (bot) {
          const int i = kZm(j);
          if ((miss >> (i - 1)) & 1u) continue;
          H.lo[j][peer_row<T>(g, x + cx(i), y + cy(i))] = f[i];
        }
      }
      __threadfence_system();
    }
  } else {
#pragma unroll
    for (int i = 1; i < Q; ++i) f[i] = LDA(P.f[i] + s);
    bc_collide<T>(f, w, bcv, bcr, om);
#pragma unroll
    for (int i = 0; i < Q; ++i) P.f[opp(i)][s] = f[i];
  }
}

#ifdef LBM_EXPERIMENTS
// A-A neighbour step (phase 0 -> 1) with row-aligned pushes.  The ten
// directions with c_x != 0 push to x + c_i, one element off the warp's
// 128-B line: every such warp store wrote 2 partial sectors (read-modify-
// write in L2).  Here a node hands those values through shared memory to
// the thread of its CTA that owns column x + c_x, which stores the whole
// row segment aligned -- only the CTA's two edge columns and periodic wraps
// store directly.  Same pulls, arithmetic and single-owner locations as
// k_step_dense_aa<NB = 1>, so the result is bitwise the same.  Measured
// 8 % SLOWER on C2 (0.81 vs 0.887 of the roofline, profiles/aa_r02.md): the
// barrier and 12 B of spills cost more than the partial sectors it removes.
// the directions with c_x != 0: 1 3 5 6 7 8 11 12 13 14
__host__ __device__ constexpr int kXShift(int j) { return j < 2 ? 1 + 2 * j : (j < 6 ? j + 3 : j + 5); }

template <typename T, int MINB>
__global__ void __launch_bounds__(128, MINB) k_step_dense_aa_nb(const Planes1<T> P, const uint32_t* __restrict__ flags,
                                                         const uint32_t* __restrict__ ubits,
                                                         const T* __restrict__ bcv, const T* __restrict__ bcr,
                                                         Geo g, T om, const Halo<T> H) {
  __shared__ T shv[10][128];
  __shared__ uint32_t shm[128];  // bit j: this column pushes kXShift(j) through shv
  const int tid = threadIdx.x;
  const int x = blockIdx.x * 128 + tid;
  const int y = blockIdx.y, z = slab_z(blockIdx.z, H.zmode, g.nz);
  const bool valid = x < g.nx;   // padding columns take part in the barrier only
  const unsigned fi = ((unsigned)z * g.ny + y) * g.nxp + (valid ? x : 0);
  const unsigned s = fi + (unsigned)g.plane;
  uint32_t w = 0u;
  if (valid) {
    const uint32_t ub = __ldg(ubits + (fi >> 10));
    w = ((ub >> ((fi >> 5) & 31)) & 1u) ? make_flag(kMaskBits, FLUID, 0, 0) : __ldg(flags + fi);
  }
  const bool live = valid && flag_type(w) != SOLID;
  const uint32_t miss = ~w & kMaskBits;
  uint32_t pushm = 0u;
  if (live) {
    T f[Q];
    f[0] = LDA(P.f[0] + s);
    {
      const UpOffsets o(g, x, y, z);
#pragma unroll
      for (int i = 1; i < Q; ++i) f[i] = LDA(P.f[opp(i)] + o.up(s, i));  // speculative, always a valid slot
    }
    if (miss) {
#pragma unroll
      for (int i = 1; i < Q; ++i)
        if ((miss >> (opp(i) - 1)) & 1u) f[i] = LDA(P.f[i] + s);
    }
    const bool top = z == g.nz - 1 && H.hi[0], bot = z == 0 && H.lo[0];
    if (top || bot) {
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        if (top) {
          const int i = kZm(j);
          if (!((miss >> (opp(i) - 1)) & 1u)) f[i] = H.hi[j][peer_row<T>(g, x - cx(i), y - cy(i))];
        }
        if (bot) {
          const int i = kZp(j);
          if (!((miss >> (opp(i) - 1)) & 1u)) f[i] = H.lo[j][peer_row<T>(g, x - cx(i), y - cy(i))];
        }
      }
    }
    bc_collide<T>(f, w, bcv, bcr, om);
    const unsigned s2 = opaque(s);
    const UpOffsets o2(g, opaque(x), opaque(y), opaque(z));
    P.f[0][s2] = f[0];
    int jx = 0;
#pragma unroll
    for (int i = 1; i < Q; ++i) {
      if ((miss >> (i - 1)) & 1u) {
        P.f[opp(i)][s2] = f[i];  // masked: own slot
      } else if (cx(i) == 0) {
        P.f[i][o2.up(s2, opp(i))] = f[i];  // x + c_i in the same column: aligned
      } else {
        const int xt = x + cx(i), tt = tid + cx(i);
        if (xt >= 0 && xt < g.nx && tt >= 0 && tt < 128) {
          shv[jx][tid] = f[i];
          pushm |= 1u << jx;
        } else {
          P.f[i][o2.up(s2, opp(i))] = f[i];  // CTA edge or periodic wrap: direct
        }
      }
      if (cx(i) != 0) ++jx;
    }
    if (top || bot) {
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        if (top) {
          const int i = kZp(j);
          if ((miss >> (i - 1)) & 1u) continue;
          H.hi[j][peer_row<T>(g, x + cx(i), y + cy(i))] = f[i];
        }
      }
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        if (bot) {
          const int i = kZm(j);
          if ((miss >> (i - 1)) & 1u) continue;
          H.lo[j][peer_row<T>(g, x + cx(i), y + cy(i))] = f[i];
        }
      }
      __threadfence_system();
    }
  }
  shm[tid] = pushm;
  __syncthreads();
  if (!valid) return;
  // receive: column x stores, for each x-shifted direction, the value pushed
  // by x - c_x of the same row into row (y + c_y, z + c_z) -- one aligned
  // 128-B line per warp
  const UpOffsets o3(g, x, y, z);
#pragma unroll
  for (int j = 0; j < 10; ++j) {
    const int i = kXShift(j);
    const int ts = tid - cx(i);
    if (ts >= 0 && ts < 128 && ((shm[ts] >> j) & 1u)) P.f[i][o3.up_yz(s, opp(i))] = shv[j][ts];
  }
}
#endif  // LBM_EXPERIMENTS
