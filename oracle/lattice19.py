"""ORACLE (test infrastructure only) -- D3Q19 lattice tables and per-node math.

Nothing in the shipped package imports this module: only tests/, the
`smoke()` checker in __graft_entry__.py and bench.py's CPU-baseline leg may
use it, and only as the checker (or the timed CPU reference arm).

This is the CPU restatement of the reference's per-node arithmetic,
generalised from D2Q9 to D3Q19 with the same expression trees:

* direction numbering: the reference D2Q9 set keeps indices 0-8
  (reference pkg/src/sparselbm/lattice.py:4-10, 28-29) and the z-moving
  directions follow;
* `feq19` follows `feq9` (lattice.py:202-218): one_m = 1 - 1.5 u.u,
  t = 3 c.u, e_i = w_i rho (one_m + t + 0.5 t t);
* `moments19` follows `moments9` (lattice.py:220-231): opposite-pair-first
  summation so the rest state is a bitwise fixed point, u = 0 when rho == 0;
* `collide19` follows `collide9` (lattice.py:233-246): f - om (f - e);
* `zou_he_velocity19` / `zou_he_pressure19` generalise
  pkg/src/sparselbm/boundaries.py:159-197 to six faces (Hecht & Harting
  2010).

Constants are baked in at the requested precision (lattice.py:188-199), so
the float32 variant really computes in 32-bit arithmetic.  Numba compiles
without fastmath, i.e. without FMA contraction or reassociation, so every
operation here is one IEEE-rounded operation in the written order.
"""

from functools import lru_cache

import numpy as np
from numba import njit

Q = 19
D = 3

#            0  1  2   3   4  5   6   7   8  9  10 11  12  13  14 15  16  17  18
CX = np.array([0, 1, 0, -1, 0, 1, -1, -1, 1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0],
              dtype=np.int8)
CY = np.array([0, 0, 1, 0, -1, 1, 1, -1, -1, 0, 0, 0, 0, 0, 0, 1, -1, -1, 1],
              dtype=np.int8)
CZ = np.array([0, 0, 0, 0, 0, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 1, -1],
              dtype=np.int8)
OPP = np.array([0, 3, 4, 1, 2, 7, 8, 5, 6, 10, 9, 12, 11, 14, 13, 16, 15, 18,
                17], dtype=np.int8)
W = np.array([1.0 / 3.0] + [1.0 / 18.0] * 4 + [1.0 / 36.0] * 4
             + [1.0 / 18.0] * 2 + [1.0 / 36.0] * 8, dtype=np.float64)

# node types / orientations (reference layouts.py:55-70, plus the z faces)
SOLID, FLUID, BOUNCE_BACK_WALL, VELOCITY_BC, PRESSURE_BC = 0, 1, 2, 3, 4
NONE, NORTH, SOUTH, EAST, WEST, TOP, BOTTOM = 0, 1, 2, 3, 4, 5, 6

# inward normal (axis, sign) per orientation: WEST is the x = 0 face, so the
# normal points +x; NORTH is y = n_y - 1, normal -y; TOP is z = n_z - 1.
NORMAL_AXIS = np.array([-1, 1, 1, 0, 0, 2, 2], dtype=np.int64)
NORMAL_SIGN = np.array([0, -1, 1, -1, 1, -1, 1], dtype=np.int64)

# projection bridge: D2Q9 direction k <- D3Q19 directions with (cx, cy) == c_k
PROJECTION = ((0, 9, 10), (1, 11, 14), (2, 15, 18), (3, 12, 13), (4, 16, 17),
              (5,), (6,), (7,), (8,))


def _dir_of(cx, cy, cz):
    for i in range(Q):
        if CX[i] == cx and CY[i] == cy and CZ[i] == cz:
            return i
    raise ValueError((cx, cy, cz))


def _c(i):
    return (int(CX[i]), int(CY[i]), int(CZ[i]))


def zou_he_tables():
    """Per-orientation index tables for the face closure (Appendix A.3).

    par[o]    9 directions with c.n == 0, ascending index (left-fold order)
    out[o]    5 directions with c.n < 0, ascending index
    nd[o]     the direction equal to n, and ndo[o] its opposite
    tan_*[o]  per tangent t (tangential axes ascending, sign + then -):
              tgt (n+t), src (-n-t), sign of u.t, axis of t, the three
              c.t = +1 and three c.t = -1 directions summed for N_t
    """
    n_or = 7
    par = np.zeros((n_or, 9), np.int64)
    out = np.zeros((n_or, 5), np.int64)
    nd = np.zeros(n_or, np.int64)
    ndo = np.zeros(n_or, np.int64)
    tan_tgt = np.zeros((n_or, 4), np.int64)
    tan_src = np.zeros((n_or, 4), np.int64)
    tan_axis = np.zeros((n_or, 4), np.int64)
    tan_sign = np.zeros((n_or, 4), np.int64)
    tan_pos = np.zeros((n_or, 4, 3), np.int64)
    tan_neg = np.zeros((n_or, 4, 3), np.int64)
    for o in range(1, n_or):
        a, s = int(NORMAL_AXIS[o]), int(NORMAL_SIGN[o])
        cs = [_c(i) for i in range(Q)]
        par[o] = [i for i in range(Q) if cs[i][a] == 0]
        out[o] = [i for i in range(Q) if cs[i][a] * s < 0]
        n = [0, 0, 0]
        n[a] = s
        nd[o] = _dir_of(*n)
        ndo[o] = OPP[nd[o]]
        tax = [b for b in range(3) if b != a]
        k = 0
        for b in tax:
            bp = [bb for bb in tax if bb != b][0]
            for sig in (1, -1):
                t = [0, 0, 0]
                t[b] = sig
                tp = [0, 0, 0]
                tp[bp] = 1
                v = [n[j] + t[j] for j in range(3)]
                tan_tgt[o, k] = _dir_of(*v)
                tan_src[o, k] = OPP[tan_tgt[o, k]]
                tan_axis[o, k] = b
                tan_sign[o, k] = sig
                # c.t = +1 group: t, t + t', t - t'; c.t = -1 group: -t, -t + t', -t - t'
                tan_pos[o, k] = [_dir_of(*t),
                                 _dir_of(*[t[j] + tp[j] for j in range(3)]),
                                 _dir_of(*[t[j] - tp[j] for j in range(3)])]
                tan_neg[o, k] = [_dir_of(*[-t[j] for j in range(3)]),
                                 _dir_of(*[-t[j] + tp[j] for j in range(3)]),
                                 _dir_of(*[-t[j] - tp[j] for j in range(3)])]
                k += 1
    return par, out, nd, ndo, tan_tgt, tan_src, tan_axis, tan_sign, tan_pos, tan_neg


ZH = zou_he_tables()


def node_ops(dtype):
    """Compiled per-node math specialised to float32 or float64."""
    return _node_ops(np.dtype(dtype).name)


@lru_cache(maxsize=None)
def _node_ops(dtype_name):
    dt = np.dtype(dtype_name).type
    w0 = dt(1.0 / 3.0)
    wa = dt(1.0 / 18.0)
    wd = dt(1.0 / 36.0)
    c05 = dt(0.5)
    c15 = dt(1.5)
    c3 = dt(3.0)
    c13 = dt(1.0 / 3.0)
    c16 = dt(1.0 / 6.0)
    zero = dt(0.0)
    one = dt(1.0)
    two = dt(2.0)
    (par_t, out_t, nd_t, ndo_t, tgt_t, src_t, tax_t, tsg_t, tpos_t,
     tneg_t) = ZH
    n_ax = NORMAL_AXIS
    n_sg = NORMAL_SIGN

    @njit(inline="always", cache=True)
    def feq19(rho, vx, vy, vz, e):
        one_m = one - c15 * (vx * vx + vy * vy + vz * vz)
        tx = c3 * vx
        ty = c3 * vy
        tz = c3 * vz
        txy_p = tx + ty
        txy_m = tx - ty
        txz_p = tx + tz
        txz_m = tx - tz
        tyz_p = ty + tz
        tyz_m = ty - tz
        r0 = w0 * rho
        ra = wa * rho
        rd = wd * rho
        e[0] = r0 * one_m
        e[1] = ra * (one_m + tx + c05 * tx * tx)
        e[2] = ra * (one_m + ty + c05 * ty * ty)
        e[3] = ra * (one_m - tx + c05 * tx * tx)
        e[4] = ra * (one_m - ty + c05 * ty * ty)
        e[5] = rd * (one_m + txy_p + c05 * txy_p * txy_p)
        e[6] = rd * (one_m - txy_m + c05 * txy_m * txy_m)
        e[7] = rd * (one_m - txy_p + c05 * txy_p * txy_p)
        e[8] = rd * (one_m + txy_m + c05 * txy_m * txy_m)
        e[9] = ra * (one_m + tz + c05 * tz * tz)
        e[10] = ra * (one_m - tz + c05 * tz * tz)
        e[11] = rd * (one_m + txz_p + c05 * txz_p * txz_p)
        e[12] = rd * (one_m - txz_p + c05 * txz_p * txz_p)
        e[13] = rd * (one_m - txz_m + c05 * txz_m * txz_m)
        e[14] = rd * (one_m + txz_m + c05 * txz_m * txz_m)
        e[15] = rd * (one_m + tyz_p + c05 * tyz_p * tyz_p)
        e[16] = rd * (one_m - tyz_p + c05 * tyz_p * tyz_p)
        e[17] = rd * (one_m - tyz_m + c05 * tyz_m * tyz_m)
        e[18] = rd * (one_m + tyz_m + c05 * tyz_m * tyz_m)

    @njit(inline="always", cache=True)
    def moments19(f):
        # opposite-pair grouping: exact at rest
        a = ((f[1] + f[3]) + (f[2] + f[4])) + (f[9] + f[10])
        e = (((f[5] + f[7]) + (f[6] + f[8]))
             + ((f[11] + f[12]) + (f[13] + f[14]))) \
            + ((f[15] + f[16]) + (f[17] + f[18]))
        rho = f[0] + a + e
        if rho == zero:
            return zero, zero, zero, zero
        d1 = f[5] - f[7]
        d2 = f[8] - f[6]
        e11 = f[11] - f[12]
        e13 = f[13] - f[14]
        g15 = f[15] - f[16]
        g17 = f[17] - f[18]
        mx = ((f[1] - f[3]) + (d1 + d2)) + (e11 - e13)
        my = ((f[2] - f[4]) + (d1 - d2)) + (g15 - g17)
        mz = ((f[9] - f[10]) + (e11 + e13)) + (g15 + g17)
        return rho, mx / rho, my / rho, mz / rho

    @njit(inline="always", cache=True)
    def collide19(f, rho, vx, vy, vz, om, e):
        feq19(rho, vx, vy, vz, e)
        for i in range(19):
            f[i] = f[i] - om * (f[i] - e[i])

    @njit(inline="always", cache=True)
    def face_sums(f, o):
        sp = f[par_t[o, 0]]
        for k in range(1, 9):
            sp = sp + f[par_t[o, k]]
        so = f[out_t[o, 0]]
        for k in range(1, 5):
            so = so + f[out_t[o, k]]
        return sp + two * so

    @njit(inline="always", cache=True)
    def zou_he_velocity19(f, o, ux, uy, vz):
        a = n_ax[o]
        if a == 0:
            ua = ux
        elif a == 1:
            ua = uy
        else:
            ua = vz
        un = ua if n_sg[o] > 0 else -ua
        rho = face_sums(f, o) / (one - un)
        f[nd_t[o]] = f[ndo_t[o]] + c13 * rho * un
        for k in range(4):
            b = tax_t[o, k]
            if b == 0:
                ub = ux
            elif b == 1:
                ub = uy
            else:
                ub = vz
            ut = ub if tsg_t[o, k] > 0 else -ub
            p = tpos_t[o, k]
            m = tneg_t[o, k]
            tsum = (f[p[0]] + f[p[1]] + f[p[2]]) - (f[m[0]] + f[m[1]] + f[m[2]])
            nt = c05 * tsum - c13 * rho * ut
            f[tgt_t[o, k]] = f[src_t[o, k]] + c16 * rho * (un + ut) - nt

    @njit(inline="always", cache=True)
    def zou_he_pressure19(f, o, rho_wall):
        un = one - face_sums(f, o) / rho_wall
        a = n_ax[o]
        ua = un if n_sg[o] > 0 else -un
        if a == 0:
            zou_he_velocity19(f, o, ua, zero, zero)
        elif a == 1:
            zou_he_velocity19(f, o, zero, ua, zero)
        else:
            zou_he_velocity19(f, o, zero, zero, ua)

    class _Ops:
        pass

    ops = _Ops()
    ops.dtype = np.dtype(dtype_name)
    ops.feq19 = feq19
    ops.moments19 = moments19
    ops.collide19 = collide19
    ops.zou_he_velocity19 = zou_he_velocity19
    ops.zou_he_pressure19 = zou_he_pressure19
    return ops
