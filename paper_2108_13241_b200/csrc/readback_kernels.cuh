// Initialisation and readback kernels (kernel.py:190-237, 285-311;
// validation.py:209-215), all decoding the A-A state through pre_index().
// Part of liblbm19 (included once, in order, by lbm19.cu).
#pragma once

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

// ------------------------------------------------ copy-bandwidth micro-bench
// Device versions of the reference's layout copy kernels (layouts.py:443-470):
// the achievable HBM copy bandwidth for each access pattern, used as the
// roofline calibration next to MEASURED_PEAKS.json.
// one pass, no grid-stride loop: each CTA copies 4 x blockDim 16-B elements,
// four independent loads in flight per thread (streaming cache hints)
__global__ void k_copy_dense(const double2* __restrict__ src, double2* __restrict__ dst, long long n2) {
  const long long i0 = (long long)blockIdx.x * blockDim.x * 4 + threadIdx.x;
  double2 v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const long long i = i0 + (long long)k * blockDim.x;
    if (i < n2) v[k] = __ldcs(src + i);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const long long i = i0 + (long long)k * blockDim.x;
    if (i < n2) __stcs(dst + i, v[k]);
  }
}
__global__ void k_copy_masked(const double* __restrict__ src, double* __restrict__ dst,
                              const uint8_t* __restrict__ mask, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (__ldg(mask + i)) dst[i] = __ldg(src + i);
}
// one CTA per chunk of `chunk` nodes; base offsets from a table (pointer tiles) or implicit
__global__ void k_copy_chunked(const double* __restrict__ src, double* __restrict__ dst,
                               const long long* __restrict__ base, int chunk) {
  const long long b = base ? __ldg(base + blockIdx.x) : (long long)blockIdx.x * chunk;
  for (int j = threadIdx.x; j < chunk; j += blockDim.x) dst[b + j] = __ldg(src + b + j);
}
__global__ void k_count_diff(const double* __restrict__ a, const double* __restrict__ b, long long n,
                             unsigned long long* bad) {
  unsigned long long c = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    c += a[i] != b[i];
  if (c) atomicAdd(bad, c);
}
__global__ void k_iota(double* __restrict__ a, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    a[i] = (double)i;
}

