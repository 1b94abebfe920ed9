"""ORACLE (test infrastructure only) -- the CPU oracle run on one z-slab with
ghost planes, for checking the multi-GPU decomposition logic
on CPU processes (torch.distributed gloo).

The slab's planes [z0, z1) are extended by one ghost plane below and above
(the neighbouring ranks' boundary planes; wrapped on a periodic z axis;
SOLID outside a closed domain), the ordinary oracle step runs on the
extended block with z treated as closed, and after every step the two
boundary planes travel to the neighbours' ghost planes.  The interior
planes must then equal the single-domain oracle bitwise.
"""

import numpy as np

from . import lattice19 as L
from .step19 import OracleSim


class SlabOracle:
    def __init__(self, types, orient, bc_index, bc_kind, bc_vel, bc_rho, omega, dtype,
                 periodic, z0, z1):
        nz = types.shape[0]
        self.z0, self.z1 = z0, z1
        idx = [z0 - 1] + list(range(z0, z1)) + [z1]
        ghost_ok = []
        for z in (z0 - 1, z1):
            ghost_ok.append(0 <= z < nz or periodic[2])
        idx = [z % nz for z in idx]
        t = types[idx].copy()
        o = orient[idx].copy()
        b = bc_index[idx].copy()
        if not ghost_ok[0]:
            t[0], o[0], b[0] = L.SOLID, 0, -1
        if not ghost_ok[1]:
            t[-1], o[-1], b[-1] = L.SOLID, 0, -1
        self.sim = OracleSim(t, o, b, bc_kind, bc_vel, bc_rho, omega, dtype=dtype,
                             periodic=(periodic[0], periodic[1], False))

    def initialize(self, rho0=1.0, v0=(0.0, 0.0, 0.0)):
        self.sim.initialize(rho0, v0)

    def step(self, exchange):
        """One step; `exchange(bottom_plane, top_plane) -> (ghost_lo, ghost_hi)`
        ships the (19, ny, nx) boundary planes and returns the neighbours'
        (None where there is no neighbour)."""
        self.sim.step(1)
        pre = self.sim.pre
        lo, hi = exchange(pre[:, 1].copy(), pre[:, -2].copy())
        if lo is not None:
            pre[:, 0] = lo
        if hi is not None:
            pre[:, -1] = hi

    @property
    def interior(self):
        return self.sim.pre[:, 1:-1]
