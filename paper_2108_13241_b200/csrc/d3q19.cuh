// D3Q19 lattice tables and per-node arithmetic (host + device).
//
// Every floating-point operation goes through `ar<T>::add/sub/mul/div`, which
// on the device are the explicitly rounded intrinsics (__fadd_rn, __fmul_rn,
// __fdiv_rn, ... -- never contracted into FMA) and on the host plain IEEE
// operations compiled with -ffp-contract=off.  The expression trees follow
// the reference's per-node functions one for one, generalised to D3Q19:
//   feq  : pkg/src/sparselbm/lattice.py:202-218  (feq9)
//   moments: lattice.py:220-231 (moments9), opposite-pair-first grouping
//   collide: lattice.py:233-246 (collide9)
//   Zou-He : pkg/src/sparselbm/boundaries.py:159-197, six faces after
//            Hecht & Harting
// so a kernel step is bit-identical to the CPU restatement in oracle/.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define LBM_HD __host__ __device__ __forceinline__
#else
#define LBM_HD inline
#endif

namespace lbm {

// ---------------------------------------------------------------- lattice
//            0  1  2   3   4  5   6   7   8  9  10 11  12  13  14 15  16  17  18
// cx {0, 1, 0, -1, 0, 1, -1, -1, 1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0}
// cy {0, 0, 1, 0, -1, 1, 1, -1, -1, 0, 0, 0, 0, 0, 0, 1, -1, -1, 1}
// cz {0, 0, 0, 0, 0, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 1, -1}
// opp {0, 3, 4, 1, 2, 7, 8, 5, 6, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17}

constexpr int Q = 19;
// pure functions of i (no table in host memory), so device code folds them
// after unrolling; the numbering is the table in the comment above
constexpr int cx(int i) {
  return (i == 1 || i == 5 || i == 8 || i == 11 || i == 14) ? 1
         : (i == 3 || i == 6 || i == 7 || i == 12 || i == 13) ? -1 : 0;
}
constexpr int cy(int i) {
  return (i == 2 || i == 5 || i == 6 || i == 15 || i == 18) ? 1
         : (i == 4 || i == 7 || i == 8 || i == 16 || i == 17) ? -1 : 0;
}
constexpr int cz(int i) {
  return (i == 9 || i == 11 || i == 13 || i == 15 || i == 17) ? 1
         : (i == 10 || i == 12 || i == 14 || i == 16 || i == 18) ? -1 : 0;
}
constexpr int opp(int i) {
  return i == 0 ? 0 : i <= 4 ? (i <= 2 ? i + 2 : i - 2) : i <= 8 ? (i <= 6 ? i + 2 : i - 2)
                                                           : ((i & 1) ? i + 1 : i - 1);
}
constexpr int cc(int i, int a) { return a == 0 ? cx(i) : (a == 1 ? cy(i) : cz(i)); }
constexpr int dir_of(int x, int y, int z) {
  for (int i = 0; i < Q; ++i)
    if (cx(i) == x && cy(i) == y && cz(i) == z) return i;
  return -1;
}

// node types / orientations (reference layouts.py:55-70 + the two z faces)
enum : uint32_t { SOLID = 0, FLUID = 1, BOUNCE_BACK_WALL = 2, VELOCITY_BC = 3, PRESSURE_BC = 4 };
enum : uint32_t { O_NONE = 0, O_NORTH = 1, O_SOUTH = 2, O_EAST = 3, O_WEST = 4, O_TOP = 5, O_BOTTOM = 6 };

// packed flag word: bits 0-17 neighbour mask, 18-20 type, 21-23 orientation,
// 24-31 bc_index
constexpr uint32_t kMaskBits = 0x3FFFFu;
LBM_HD uint32_t flag_type(uint32_t w) { return (w >> 18) & 7u; }
LBM_HD uint32_t flag_orient(uint32_t w) { return (w >> 21) & 7u; }
LBM_HD uint32_t flag_bc(uint32_t w) { return w >> 24; }
LBM_HD uint32_t make_flag(uint32_t mask, uint32_t type, uint32_t orient, uint32_t bc) {
  return (mask & kMaskBits) | (type << 18) | (orient << 21) | ((bc & 0xFFu) << 24);
}

// ------------------------------------------------------ rounded arithmetic
template <typename T> struct ar;
template <> struct ar<float> {
#if defined(__CUDA_ARCH__)
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  // 0 / b for finite-or-infinite nonzero b is a signed zero (sign(a) ^ sign(b));
  // __fdiv_rn sends a zero dividend down its slow path (FCHK), which every
  // node of a flow with an exactly zero momentum component would pay
  static __device__ __forceinline__ float div(float a, float b) {
    if (a == 0.f && b != 0.f && b == b) return __int_as_float((__float_as_int(a) ^ __float_as_int(b)) & 0x80000000);
    return __fdiv_rn(a, b);
  }
#else
  static inline float add(float a, float b) { return a + b; }
  static inline float sub(float a, float b) { return a - b; }
  static inline float mul(float a, float b) { return a * b; }
  static inline float div(float a, float b) { return a / b; }
#endif
};
template <> struct ar<double> {
#if defined(__CUDA_ARCH__)
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) {
    if (a == 0.0 && b != 0.0 && b == b)
      return __longlong_as_double((__double_as_longlong(a) ^ __double_as_longlong(b)) & (long long)0x8000000000000000ULL);
    return __ddiv_rn(a, b);
  }
#else
  static inline double add(double a, double b) { return a + b; }
  static inline double sub(double a, double b) { return a - b; }
  static inline double mul(double a, double b) { return a * b; }
  static inline double div(double a, double b) { return a / b; }
#endif
};

// constants rounded from double exactly like numpy's dt(1.0 / 3.0)
template <typename T> struct K {
  static constexpr T w0 = (T)(1.0 / 3.0);
  static constexpr T wa = (T)(1.0 / 18.0);
  static constexpr T wd = (T)(1.0 / 36.0);
  static constexpr T c05 = (T)0.5;
  static constexpr T c15 = (T)1.5;
  static constexpr T c3 = (T)3.0;
  static constexpr T c13 = (T)(1.0 / 3.0);
  static constexpr T c16 = (T)(1.0 / 6.0);
  static constexpr T zero = (T)0.0;
  static constexpr T one = (T)1.0;
  static constexpr T two = (T)2.0;
};

// e_i = w rho (one_m + t + 0.5 t t), Python evaluation order
template <typename T>
LBM_HD T eq_term(T wr, T one_m, T t, bool neg) {
  using A = ar<T>;
  T lin = neg ? A::sub(one_m, t) : A::add(one_m, t);
  T sq = A::mul(A::mul(K<T>::c05, t), t);
  return A::mul(wr, A::add(lin, sq));
}

template <typename T>
LBM_HD void feq19(T rho, T vx, T vy, T vz, T* e) {
  using A = ar<T>;
  T uu = A::add(A::add(A::mul(vx, vx), A::mul(vy, vy)), A::mul(vz, vz));
  T one_m = A::sub(K<T>::one, A::mul(K<T>::c15, uu));
  T tx = A::mul(K<T>::c3, vx), ty = A::mul(K<T>::c3, vy), tz = A::mul(K<T>::c3, vz);
  T txy_p = A::add(tx, ty), txy_m = A::sub(tx, ty);
  T txz_p = A::add(tx, tz), txz_m = A::sub(tx, tz);
  T tyz_p = A::add(ty, tz), tyz_m = A::sub(ty, tz);
  T r0 = A::mul(K<T>::w0, rho), ra = A::mul(K<T>::wa, rho), rd = A::mul(K<T>::wd, rho);
  e[0] = A::mul(r0, one_m);
  e[1] = eq_term(ra, one_m, tx, false);
  e[2] = eq_term(ra, one_m, ty, false);
  e[3] = eq_term(ra, one_m, tx, true);
  e[4] = eq_term(ra, one_m, ty, true);
  e[5] = eq_term(rd, one_m, txy_p, false);
  e[6] = eq_term(rd, one_m, txy_m, true);
  e[7] = eq_term(rd, one_m, txy_p, true);
  e[8] = eq_term(rd, one_m, txy_m, false);
  e[9] = eq_term(ra, one_m, tz, false);
  e[10] = eq_term(ra, one_m, tz, true);
  e[11] = eq_term(rd, one_m, txz_p, false);
  e[12] = eq_term(rd, one_m, txz_p, true);
  e[13] = eq_term(rd, one_m, txz_m, true);
  e[14] = eq_term(rd, one_m, txz_m, false);
  e[15] = eq_term(rd, one_m, tyz_p, false);
  e[16] = eq_term(rd, one_m, tyz_p, true);
  e[17] = eq_term(rd, one_m, tyz_m, true);
  e[18] = eq_term(rd, one_m, tyz_m, false);
}

// density sum with opposite pairs first
template <typename T>
LBM_HD T density19(const T* f) {
  using A = ar<T>;
  T a = A::add(A::add(A::add(f[1], f[3]), A::add(f[2], f[4])), A::add(f[9], f[10]));
  T e = A::add(A::add(A::add(A::add(f[5], f[7]), A::add(f[6], f[8])),
                      A::add(A::add(f[11], f[12]), A::add(f[13], f[14]))),
               A::add(A::add(f[15], f[16]), A::add(f[17], f[18])));
  return A::add(A::add(f[0], a), e);
}

template <typename T>
LBM_HD void momentum19(const T* f, T& mx, T& my, T& mz) {
  using A = ar<T>;
  T d1 = A::sub(f[5], f[7]), d2 = A::sub(f[8], f[6]);
  T e11 = A::sub(f[11], f[12]), e13 = A::sub(f[13], f[14]);
  T g15 = A::sub(f[15], f[16]), g17 = A::sub(f[17], f[18]);
  mx = A::add(A::add(A::sub(f[1], f[3]), A::add(d1, d2)), A::sub(e11, e13));
  my = A::add(A::add(A::sub(f[2], f[4]), A::sub(d1, d2)), A::sub(g15, g17));
  mz = A::add(A::add(A::sub(f[9], f[10]), A::add(e11, e13)), A::add(g15, g17));
}

template <typename T>
LBM_HD void moments19(const T* f, T& rho, T& vx, T& vy, T& vz) {
  using A = ar<T>;
  rho = density19(f);
  if (rho == K<T>::zero) {
    rho = vx = vy = vz = K<T>::zero;
    return;
  }
  T mx, my, mz;
  momentum19(f, mx, my, mz);
  vx = A::div(mx, rho);
  vy = A::div(my, rho);
  vz = A::div(mz, rho);
}

template <typename T>
LBM_HD void collide19(T* f, T rho, T vx, T vy, T vz, T om) {
  using A = ar<T>;
  T e[Q];
  feq19(rho, vx, vy, vz, e);
#pragma unroll
  for (int i = 0; i < Q; ++i) f[i] = A::sub(f[i], A::mul(om, A::sub(f[i], e[i])));
}

// ------------------------------------------------------------------ Zou-He
// Face with inward normal n = S * e_AX.  Known populations: c.n == 0 (`par`,
// 9 of them) and c.n < 0 (`out`, 5).  Unknowns c.n > 0 are rebuilt:
//   rho   = (sum_par + 2 sum_out) / (1 - u.n)
//   f_n   = f_-n + (1/3) rho u.n
//   f_n+t = f_-n-t + (1/6) rho (u.n + u.t) - N_t,
//   N_t   = 1/2 sum_par f (c.t) - (1/3) rho u.t
// Summation orders (ascending direction index, left fold) match
// oracle/lattice19.py exactly.
template <typename T, int AX, int S>
LBM_HD T face_sum(const T* f) {
  using A = ar<T>;
  T sp = K<T>::zero, so = K<T>::zero;
  bool fp = true, fo = true;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    if (cc(i, AX) == 0) {
      sp = fp ? f[i] : A::add(sp, f[i]);
      fp = false;
    }
  }
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    if (cc(i, AX) * S < 0) {
      so = fo ? f[i] : A::add(so, f[i]);
      fo = false;
    }
  }
  return A::add(sp, A::mul(K<T>::two, so));
}

struct FaceTables {
  int nd;                       // direction equal to the normal n
  int B[4], sig[4];             // tangent axis and sign per tangent
  int tgt[4], src[4];           // unknown n+t and its opposite -n-t
  int p[4][3], m[4][3];         // c.t = +1 / -1 directions with c.n == 0
};
constexpr FaceTables make_face(int AX, int S) {
  FaceTables z{};
  int nv[3] = {0, 0, 0};
  nv[AX] = S;
  z.nd = dir_of(nv[0], nv[1], nv[2]);
  const int tax0 = AX == 0 ? 1 : 0, tax1 = AX == 2 ? 1 : 2;
  for (int k = 0; k < 4; ++k) {
    const int B = k < 2 ? tax0 : tax1, BP = k < 2 ? tax1 : tax0;
    const int sig = (k % 2 == 0) ? 1 : -1;
    int t[3] = {0, 0, 0}, tp[3] = {0, 0, 0};
    t[B] = sig;
    tp[BP] = 1;
    z.B[k] = B;
    z.sig[k] = sig;
    z.tgt[k] = dir_of(nv[0] + t[0], nv[1] + t[1], nv[2] + t[2]);
    z.src[k] = opp(z.tgt[k]);
    z.p[k][0] = dir_of(t[0], t[1], t[2]);
    z.p[k][1] = dir_of(t[0] + tp[0], t[1] + tp[1], t[2] + tp[2]);
    z.p[k][2] = dir_of(t[0] - tp[0], t[1] - tp[1], t[2] - tp[2]);
    z.m[k][0] = dir_of(-t[0], -t[1], -t[2]);
    z.m[k][1] = dir_of(-t[0] + tp[0], -t[1] + tp[1], -t[2] + tp[2]);
    z.m[k][2] = dir_of(-t[0] - tp[0], -t[1] - tp[1], -t[2] - tp[2]);
  }
  return z;
}

template <typename T, int AX, int S>
LBM_HD void zou_he_velocity_face(T* f, T ux, T uy, T uz) {
  using A = ar<T>;
  constexpr FaceTables z = make_face(AX, S);
  const T u3[3] = {ux, uy, uz};
  T ua = u3[AX];
  T un = S > 0 ? ua : -ua;
  T rho = A::div(face_sum<T, AX, S>(f), A::sub(K<T>::one, un));
  f[z.nd] = A::add(f[opp(z.nd)], A::mul(A::mul(K<T>::c13, rho), un));
  // tangential axes ascending, sign + then - (oracle/lattice19.py order)
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    T ub = u3[z.B[k]];
    T ut = z.sig[k] > 0 ? ub : -ub;
    T tsum = A::sub(A::add(A::add(f[z.p[k][0]], f[z.p[k][1]]), f[z.p[k][2]]),
                    A::add(A::add(f[z.m[k][0]], f[z.m[k][1]]), f[z.m[k][2]]));
    T nt = A::sub(A::mul(K<T>::c05, tsum), A::mul(A::mul(K<T>::c13, rho), ut));
    f[z.tgt[k]] = A::sub(A::add(f[z.src[k]], A::mul(A::mul(K<T>::c16, rho), A::add(un, ut))), nt);
  }
}

template <typename T, int AX, int S>
LBM_HD void zou_he_pressure_face(T* f, T rho_wall) {
  using A = ar<T>;
  T un = A::sub(K<T>::one, A::div(face_sum<T, AX, S>(f), rho_wall));
  T ua = S > 0 ? un : -un;
  T z = K<T>::zero;
  if (AX == 0) zou_he_velocity_face<T, AX, S>(f, ua, z, z);
  else if (AX == 1) zou_he_velocity_face<T, AX, S>(f, z, ua, z);
  else zou_he_velocity_face<T, AX, S>(f, z, z, ua);
}

template <typename T>
LBM_HD void zou_he_velocity19(T* f, uint32_t orient, T ux, T uy, T uz) {
  switch (orient) {
    case O_NORTH: zou_he_velocity_face<T, 1, -1>(f, ux, uy, uz); break;
    case O_SOUTH: zou_he_velocity_face<T, 1, 1>(f, ux, uy, uz); break;
    case O_EAST: zou_he_velocity_face<T, 0, -1>(f, ux, uy, uz); break;
    case O_WEST: zou_he_velocity_face<T, 0, 1>(f, ux, uy, uz); break;
    case O_TOP: zou_he_velocity_face<T, 2, -1>(f, ux, uy, uz); break;
    case O_BOTTOM: zou_he_velocity_face<T, 2, 1>(f, ux, uy, uz); break;
    default: break;
  }
}

template <typename T>
LBM_HD void zou_he_pressure19(T* f, uint32_t orient, T rho_wall) {
  switch (orient) {
    case O_NORTH: zou_he_pressure_face<T, 1, -1>(f, rho_wall); break;
    case O_SOUTH: zou_he_pressure_face<T, 1, 1>(f, rho_wall); break;
    case O_EAST: zou_he_pressure_face<T, 0, -1>(f, rho_wall); break;
    case O_WEST: zou_he_pressure_face<T, 0, 1>(f, rho_wall); break;
    case O_TOP: zou_he_pressure_face<T, 2, -1>(f, rho_wall); break;
    case O_BOTTOM: zou_he_pressure_face<T, 2, 1>(f, rho_wall); break;
    default: break;
  }
}

// float64 initial equilibrium in numpy's evaluation order (reference
// kernel.py:219-223): W rho (1 + 3 cv + 4.5 cv cv - 1.5 vv)
LBM_HD double init_eq(int i, double rho, double vx, double vy, double vz) {
  using A = ar<double>;
  const double W = i == 0 ? 1.0 / 3.0 : ((i <= 4 || i == 9 || i == 10) ? 1.0 / 18.0 : 1.0 / 36.0);
  double vv = A::add(A::add(A::mul(vx, vx), A::mul(vy, vy)), A::mul(vz, vz));
  double cv = A::add(A::add(A::mul((double)cx(i), vx), A::mul((double)cy(i), vy)),
                     A::mul((double)cz(i), vz));
  double in = A::sub(A::add(A::add(1.0, A::mul(3.0, cv)), A::mul(A::mul(4.5, cv), cv)),
                     A::mul(1.5, vv));
  return A::mul(A::mul(W, rho), in);
}

}  // namespace lbm
