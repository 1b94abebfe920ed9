"""ORACLE (test infrastructure only) -- independent plain-loop D3Q19 step.

A deliberately plain transcription in the spirit of the reference's own test
oracle (pkg/tests/reference_lbm.py:1-145): Python loops over nodes, neighbour
checks done on the node-type grid directly (no masks), the equilibrium in
its textbook form w (1 + 3 c.u + 4.5 (c.u)^2 - 1.5 u.u) and the Zou-He
closures written generically from the face normal (Hecht & Harting 2010).
It imports nothing from the Numba oracle, so it is an independent check on
it (agreement within 1e-12 in float64, the reference's own bar,
t/test_kernel.py:106-116).  Only for small grids (<= 12^3, <= 25 steps).
"""

import numpy as np

VEL = [(0, 0, 0), (1, 0, 0), (0, 1, 0), (-1, 0, 0), (0, -1, 0), (1, 1, 0),
       (-1, 1, 0), (-1, -1, 0), (1, -1, 0), (0, 0, 1), (0, 0, -1), (1, 0, 1),
       (-1, 0, -1), (-1, 0, 1), (1, 0, -1), (0, 1, 1), (0, -1, -1), (0, -1, 1),
       (0, 1, -1)]
REFLECT = [VEL.index(tuple(-c for c in v)) for v in VEL]
WEIGHT = [1 / 3 if sum(map(abs, v)) == 0 else 1 / 18 if sum(map(abs, v)) == 1
          else 1 / 36 for v in VEL]
SOLID, FLUID, WALL, VELOCITY, PRESSURE = 0, 1, 2, 3, 4
# orientation -> inward normal
NORMAL = {1: (0, -1, 0), 2: (0, 1, 0), 3: (-1, 0, 0), 4: (1, 0, 0),
          5: (0, 0, -1), 6: (0, 0, 1)}


def dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def ref_equilibrium(rho, u):
    uu = dot(u, u)
    return np.array([WEIGHT[i] * rho * (1 + 3 * dot(VEL[i], u)
                                        + 4.5 * dot(VEL[i], u) ** 2 - 1.5 * uu)
                     for i in range(19)])


def ref_moments(f):
    rho = float(sum(f))
    if rho == 0.0:
        return 0.0, (0.0, 0.0, 0.0)
    m = [sum(f[i] * VEL[i][a] for i in range(19)) for a in range(3)]
    return rho, tuple(mi / rho for mi in m)


def ref_zou_he_velocity(f, side, u):
    f = f.copy()
    n = NORMAL[side]
    un = dot(u, n)
    tang = sum(f[i] for i in range(19) if dot(VEL[i], n) == 0)
    leaving = sum(f[i] for i in range(19) if dot(VEL[i], n) < 0)
    rho = (tang + 2 * leaving) / (1 - un)
    for i in range(19):
        if dot(VEL[i], n) <= 0:
            continue
        j = REFLECT[i]
        if VEL[i] == n:
            f[i] = f[j] + rho * un / 3
        else:
            t = tuple(VEL[i][a] - n[a] for a in range(3))
            nt = 0.5 * sum(f[k] * dot(VEL[k], t) for k in range(19)
                           if dot(VEL[k], n) == 0) - rho * dot(u, t) / 3
            f[i] = f[j] + rho * (un + dot(u, t)) / 6 - nt
    return f


def ref_zou_he_pressure(f, side, rho0):
    n = NORMAL[side]
    tang = sum(f[i] for i in range(19) if dot(VEL[i], n) == 0)
    leaving = sum(f[i] for i in range(19) if dot(VEL[i], n) < 0)
    un = 1 - (tang + 2 * leaving) / rho0
    return ref_zou_he_velocity(f, side, tuple(un * c for c in n))


def ref_initialize(types, bc_vel, bc_rho, bc_index, rho0=1.0, v0=(0, 0, 0)):
    nz, ny, nx = types.shape
    f = np.zeros((19, nz, ny, nx))
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                t = types[z, y, x]
                if t == SOLID:
                    continue
                rho, u = float(rho0), tuple(float(v) for v in v0)
                b = bc_index[z, y, x]
                if t == VELOCITY:
                    u = tuple(bc_vel[b])
                elif t == PRESSURE:
                    rho = bc_rho[b]
                f[:, z, y, x] = ref_equilibrium(rho, u)
    return f


def ref_step(f, types, orient, bc_vel, bc_rho, bc_index, omega,
             periodic=(False, False, False)):
    nz, ny, nx = types.shape
    dims = (nx, ny, nz)
    out = np.zeros_like(f)
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                t = types[z, y, x]
                if t == SOLID:
                    continue
                g = np.empty(19)
                for i in range(19):
                    src = [x - VEL[i][0], y - VEL[i][1], z - VEL[i][2]]
                    inside = True
                    for a in range(3):
                        if periodic[a]:
                            src[a] %= dims[a]
                        elif not 0 <= src[a] < dims[a]:
                            inside = False
                    if inside and types[src[2], src[1], src[0]] != SOLID:
                        g[i] = f[i, src[2], src[1], src[0]]
                    else:
                        g[i] = f[REFLECT[i], z, y, x]
                b = bc_index[z, y, x]
                if t == VELOCITY:
                    g = ref_zou_he_velocity(g, orient[z, y, x], tuple(bc_vel[b]))
                elif t == PRESSURE:
                    g = ref_zou_he_pressure(g, orient[z, y, x], bc_rho[b])
                rho, u = ref_moments(g)
                feq = ref_equilibrium(rho, u)
                out[:, z, y, x] = g - omega * (g - feq)
    return out


def ref_run(f, types, orient, bc_vel, bc_rho, bc_index, omega, steps,
            periodic=(False, False, False)):
    for _ in range(steps):
        f = ref_step(f, types, orient, bc_vel, bc_rho, bc_index, omega, periodic)
    return f
