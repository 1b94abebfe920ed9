"""CPU model of the A-A in-place scheme (the index algebra the CUDA kernels
k_step_dense_aa / k_step_tiles_aa and the readback decoder pre_index()
implement), checked bitwise against the oracle's two-buffer pull kernel
(reference pkg/kernel.py:72-141).  Test infrastructure only: the per-node
math is the oracle's (oracle/lattice19.py), the addressing is the scheme's.

  phase 0 (even step count): F[opp(i)][x] = pre_i(x)
  phase 1 (odd):             pre_i(x) = F[i][x + c_i] if link i present,
                             else F[opp(i)][x]
  neighbour step (0 -> 1):   f_i = F[opp(i)][x - c_i] if link opp(i) present else F[i][x];
                             collide; f*_i -> F[i][x + c_i] if link i present else F[opp(i)][x]
  local step (1 -> 0):       f_i = F[i][x]; collide; f*_i -> F[opp(i)][x]
"""

from functools import lru_cache

import numpy as np
import pytest
from numba import njit

from helpers import oracle_sim, random_mixed_geometry3
from oracle import geometry19 as G
from oracle import lattice19 as L


@lru_cache(maxsize=None)
def _aa_kernels(dtype_name):
    ops = L.node_ops(dtype_name)
    dt = np.dtype(dtype_name)
    moments19, collide19 = ops.moments19, ops.collide19
    zhv, zhp = ops.zou_he_velocity19, ops.zou_he_pressure19
    CX, CY, CZ, OPP = L.CX, L.CY, L.CZ, L.OPP
    SOLID, VEL, PRES = L.SOLID, L.VELOCITY_BC, L.PRESSURE_BC

    @njit(cache=False)
    def wrap(v, n):
        return v + n if v < 0 else (v - n if v >= n else v)

    @njit(cache=False)
    def step(F, types, masks, orient, bc_index, bc_vel, bc_rho, omega, neighbour):
        nz, ny, nx = types.shape
        f = np.empty(19, dtype=dt)
        e = np.empty(19, dtype=dt)
        for z in range(nz):
            for y in range(ny):
                for x in range(nx):
                    t = types[z, y, x]
                    if t == SOLID:
                        continue
                    m = masks[z, y, x]
                    f[0] = F[0, z, y, x]
                    for i in range(1, 19):
                        o = OPP[i]
                        if neighbour:
                            if m & (np.uint32(1) << np.uint32(o - 1)):
                                f[i] = F[o, wrap(z - CZ[i], nz), wrap(y - CY[i], ny), wrap(x - CX[i], nx)]
                            else:
                                f[i] = F[i, z, y, x]
                        else:
                            f[i] = F[i, z, y, x]
                    if t == VEL:
                        b = bc_index[z, y, x]
                        zhv(f, orient[z, y, x], bc_vel[b, 0], bc_vel[b, 1], bc_vel[b, 2])
                    elif t == PRES:
                        b = bc_index[z, y, x]
                        zhp(f, orient[z, y, x], bc_rho[b])
                    rho, vx, vy, vz = moments19(f)
                    collide19(f, rho, vx, vy, vz, omega, e)
                    F[0, z, y, x] = f[0]
                    for i in range(1, 19):
                        o = OPP[i]
                        if neighbour and (m & (np.uint32(1) << np.uint32(i - 1))):
                            F[i, wrap(z + CZ[i], nz), wrap(y + CY[i], ny), wrap(x + CX[i], nx)] = f[i]
                        else:
                            F[o, z, y, x] = f[i]

    return step


def encode_phase0(pre):
    """Initial AA state: F[opp(i)][x] = pre_i(x)."""
    return np.ascontiguousarray(pre[np.asarray(L.OPP)])


def decode(F, phase, types, masks):
    """The reference's pre buffer from the AA state (pre_index() on the device)."""
    nz, ny, nx = types.shape
    opp = np.asarray(L.OPP)
    if phase == 0:
        out = F[opp].copy()
    else:
        out = np.empty_like(F)
        out[0] = F[0]
        zz, yy, xx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        for i in range(1, 19):
            present = (masks >> np.uint32(i - 1)) & 1
            zs = (zz + L.CZ[i]) % nz
            ys = (yy + L.CY[i]) % ny
            xs = (xx + L.CX[i]) % nx
            out[i] = np.where(present == 1, F[i][zs, ys, xs], F[opp[i]])
    out[:, types == L.SOLID] = 0
    return out


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("seed,periodic_z", [(1, False), (2, True), (3, False)])
def test_aa_model_bitwise_vs_oracle(dtype, seed, periodic_z):
    c = random_mixed_geometry3(seed, n=(11, 9, 8), periodic_z=periodic_z)
    omega = 1.0 / (3 * 0.08 + 0.5)
    ref = oracle_sim(c, omega, dtype)
    ref.initialize(1.0)
    masks = G.neighbor_masks(c["types"], c["periodic"])
    assert np.array_equal(masks, ref.masks)
    F = encode_phase0(ref.pre)
    step = _aa_kernels(np.dtype(dtype).name)
    types = c["types"]
    args = (types, masks, ref.orient, ref.bc_index, ref.bc_vel, ref.bc_rho, ref.omega)
    assert np.array_equal(decode(F, 0, types, masks), ref.pre)
    for k in range(7):
        step(F, *args, k % 2 == 0)
        ref.step(1)
        assert np.array_equal(decode(F, (k + 1) % 2, types, masks), ref.pre), k + 1


def test_aa_locations_have_one_owner():
    """Race freedom: in the neighbour step every storage location read by a
    node is the one it writes back, and no location is written twice."""
    c = random_mixed_geometry3(4, n=(10, 8, 6), periodic_z=True)
    ref = oracle_sim(c, 1.2, np.float64)
    types, masks = c["types"], ref.masks
    nz, ny, nx = types.shape
    reads, writes = {}, {}
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                if types[z, y, x] == L.SOLID:
                    continue
                m = int(masks[z, y, x])
                for i in range(1, 19):
                    o = int(L.OPP[i])
                    cx, cy, cz = int(L.CX[i]), int(L.CY[i]), int(L.CZ[i])
                    if m >> (o - 1) & 1:
                        r = (o, (z - cz) % nz, (y - cy) % ny, (x - cx) % nx)
                    else:
                        r = (i, z, y, x)
                    w = ((i, (z + cz) % nz, (y + cy) % ny, (x + cx) % nx)
                         if m >> (i - 1) & 1 else (o, z, y, x))
                    assert r not in reads and w not in writes
                    reads[r] = (z, y, x)
                    writes[w] = (z, y, x)
    assert set(reads) == set(writes)
    assert all(reads[k] == writes[k] for k in reads)
