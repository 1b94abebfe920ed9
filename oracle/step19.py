"""ORACLE (test infrastructure only) -- the D3Q19 fused pull stream + BGK
collide step on the CPU (Numba, parallel over nodes), and a small
Simulation-like driver around it.

`step_kernel(dtype)` restates `_step_kernel(...).step` of the reference
(pkg/src/sparselbm/kernel.py:72-141) line by line in 3-D over canonical
(19, nz, ny, nx) buffers:

1. skip SOLID nodes (kernel.py:78-80);
2. gather f_i from the upstream node x - c_i when the mask bit of opp(i) is
   set, else reflect the node's own f_opp(i) (link-wise bounce-back,
   kernel.py:84-116); periodic axes wrap;
3. VELOCITY_BC / PRESSURE_BC nodes apply the Zou-He closure of their
   orientation (kernel.py:118-127);
4. moments, BGK relaxation, node-local store (kernel.py:129-141).

`initial_state` restates Simulation.initialize (kernel.py:190-237): float64
equilibrium with imposed boundary values, cast to the storage dtype; solid
nodes stay zero.  `macroscopic` restates Simulation.macroscopic_fields
(kernel.py:285-311) in float64 with the kernel's pair grouping.
"""

from functools import lru_cache

import numpy as np
from numba import njit, prange

from . import lattice19 as L
from .geometry19 import neighbor_masks


def step_kernel(dtype):
    return _step_kernel(np.dtype(dtype).name)


@lru_cache(maxsize=None)
def _step_kernel(dtype_name):
    ops = L.node_ops(dtype_name)
    dt = np.dtype(dtype_name)
    moments19 = ops.moments19
    collide19 = ops.collide19
    zhv = ops.zou_he_velocity19
    zhp = ops.zou_he_pressure19
    CX, CY, CZ, OPP = L.CX, L.CY, L.CZ, L.OPP
    SOLID, VEL, PRES = L.SOLID, L.VELOCITY_BC, L.PRESSURE_BC

    @njit(parallel=True, cache=True)
    def step(pre, post, types, masks, orient, bc_index, bc_vel, bc_rho, omega):
        nz, ny, nx = types.shape
        for row in prange(nz * ny):
            y = row % ny
            z = row // ny
            # per-row scratch (numba cannot keep a per-node array in registers)
            f = np.empty(19, dtype=dt)
            e = np.empty(19, dtype=dt)
            for x in range(nx):
                t = types[z, y, x]
                if t == SOLID:
                    continue
                m = masks[z, y, x]
                f[0] = pre[0, z, y, x]
                for i in range(1, 19):
                    o = OPP[i]
                    if m & (np.uint32(1) << np.uint32(o - 1)):
                        xs = x - CX[i]
                        ys = y - CY[i]
                        zs = z - CZ[i]
                        if xs < 0:
                            xs += nx
                        elif xs >= nx:
                            xs -= nx
                        if ys < 0:
                            ys += ny
                        elif ys >= ny:
                            ys -= ny
                        if zs < 0:
                            zs += nz
                        elif zs >= nz:
                            zs -= nz
                        f[i] = pre[i, zs, ys, xs]
                    else:
                        f[i] = pre[o, z, y, x]
                if t == VEL:
                    b = bc_index[z, y, x]
                    zhv(f, orient[z, y, x], bc_vel[b, 0], bc_vel[b, 1],
                        bc_vel[b, 2])
                elif t == PRES:
                    b = bc_index[z, y, x]
                    zhp(f, orient[z, y, x], bc_rho[b])
                rho, vx, vy, vz = moments19(f)
                collide19(f, rho, vx, vy, vz, omega, e)
                for i in range(19):
                    post[i, z, y, x] = f[i]

    return step


@njit(cache=True)
def _first_nonfinite(pre, types):
    nz, ny, nx = types.shape
    for i in range(19):
        for z in range(nz):
            for y in range(ny):
                for x in range(nx):
                    if types[z, y, x] != 0 and not np.isfinite(pre[i, z, y, x]):
                        return i, x, y, z
    return -1, -1, -1, -1


def equilibrium_planes(rho, vx, vy, vz):
    """float64 equilibrium exactly as Simulation.initialize computes it
    (reference kernel.py:219-223), one plane per direction."""
    vv = vx * vx + vy * vy + vz * vz
    planes = np.empty((19,) + np.shape(rho))
    for i in range(19):
        cv = L.CX[i] * vx + L.CY[i] * vy + L.CZ[i] * vz
        planes[i] = L.W[i] * rho * (1.0 + 3.0 * cv + 4.5 * cv * cv - 1.5 * vv)
    return planes


def initial_state(types, bc_index, bc_kind, bc_vel, bc_rho, dtype, rho0=1.0,
                  v0=(0.0, 0.0, 0.0)):
    types = np.asarray(types, dtype=np.uint8)
    shape = types.shape
    rho = np.broadcast_to(np.asarray(rho0, dtype=np.float64), shape).copy()
    vx = np.broadcast_to(np.asarray(v0[0], dtype=np.float64), shape).copy()
    vy = np.broadcast_to(np.asarray(v0[1], dtype=np.float64), shape).copy()
    vz = np.broadcast_to(np.asarray(v0[2], dtype=np.float64), shape).copy()
    for idx in range(len(bc_kind)):
        sel_v = (types == L.VELOCITY_BC) & (bc_index == idx)
        sel_p = (types == L.PRESSURE_BC) & (bc_index == idx)
        if bc_kind[idx] == 0 and sel_v.any():
            vx[sel_v], vy[sel_v], vz[sel_v] = bc_vel[idx]
        elif bc_kind[idx] == 1 and sel_p.any():
            rho[sel_p] = bc_rho[idx]
    planes = equilibrium_planes(rho, vx, vy, vz)
    f = np.zeros((19,) + shape, dtype=dtype)
    ns = types != L.SOLID
    for i in range(19):
        f[i][ns] = planes[i][ns].astype(dtype)
    return f


def macroscopic(f, types):
    f = f.astype(np.float64)
    a = ((f[1] + f[3]) + (f[2] + f[4])) + (f[9] + f[10])
    e = (((f[5] + f[7]) + (f[6] + f[8])) + ((f[11] + f[12]) + (f[13] + f[14]))) \
        + ((f[15] + f[16]) + (f[17] + f[18]))
    r = f[0] + a + e
    d1 = f[5] - f[7]
    d2 = f[8] - f[6]
    e11 = f[11] - f[12]
    e13 = f[13] - f[14]
    g15 = f[15] - f[16]
    g17 = f[17] - f[18]
    mx = ((f[1] - f[3]) + (d1 + d2)) + (e11 - e13)
    my = ((f[2] - f[4]) + (d1 - d2)) + (g15 - g17)
    mz = ((f[9] - f[10]) + (e11 + e13)) + (g15 + g17)
    ok = (types != L.SOLID) & (r != 0.0)
    ux = np.zeros_like(r)
    uy = np.zeros_like(r)
    uz = np.zeros_like(r)
    ux[ok] = mx[ok] / r[ok]
    uy[ok] = my[ok] / r[ok]
    uz[ok] = mz[ok] / r[ok]
    r = np.where(types != L.SOLID, r, 0.0)
    return r, ux, uy, uz


class OracleSim:
    """Minimal driver: same semantics as the product's Simulation over
    canonical (19, nz, ny, nx) host arrays."""

    def __init__(self, types, orient, bc_index, bc_kind, bc_vel, bc_rho, omega,
                 dtype=np.float64, periodic=(False, False, False)):
        self.types = np.ascontiguousarray(types, dtype=np.uint8)
        self.orient = np.ascontiguousarray(orient, dtype=np.uint8)
        self.bc_index = np.ascontiguousarray(bc_index, dtype=np.int32)
        self.bc_kind = np.asarray(bc_kind, dtype=np.uint8)
        self.dtype = np.dtype(dtype)
        nb = max(len(self.bc_kind), 1)
        self.bc_vel = np.zeros((nb, 3), dtype=self.dtype)
        self.bc_rho = np.zeros(nb, dtype=self.dtype)
        if len(self.bc_kind):
            self.bc_vel[:len(bc_vel)] = np.asarray(bc_vel, dtype=np.float64)
            self.bc_rho[:len(bc_rho)] = np.asarray(bc_rho, dtype=np.float64)
        self._bc_vel64 = np.asarray(bc_vel, dtype=np.float64).reshape(-1, 3)
        self._bc_rho64 = np.asarray(bc_rho, dtype=np.float64)
        self.omega = self.dtype.type(omega)
        self.periodic = tuple(bool(p) for p in periodic)
        self.masks = neighbor_masks(self.types, self.periodic)
        self._kernel = step_kernel(self.dtype)
        self.pre = None
        self.post = None
        self.step_count = 0

    def initialize(self, rho0=1.0, v0=(0.0, 0.0, 0.0)):
        self.pre = initial_state(self.types, self.bc_index, self.bc_kind,
                                 self._bc_vel64, self._bc_rho64, self.dtype,
                                 rho0, v0)
        self.post = np.zeros_like(self.pre)
        self.step_count = 0

    def step(self, n=1):
        for _ in range(n):
            self._kernel(self.pre, self.post, self.types, self.masks,
                         self.orient, self.bc_index, self.bc_vel, self.bc_rho,
                         self.omega)
            self.pre, self.post = self.post, self.pre
            self.step_count += 1

    run = step

    def macroscopic_fields(self):
        return macroscopic(self.pre, self.types)

    def total_mass(self):
        return float(self.pre[:, self.types != L.SOLID].astype(np.float64).sum())

    def first_nonfinite(self):
        return _first_nonfinite(self.pre, self.types)
