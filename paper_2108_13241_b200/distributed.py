"""z-slab domain decomposition.

One process (or one Simulation) per GPU owns the contiguous global planes
[z0, z1).  Its node descriptors are the slab's planes; the node types of
the planes z0 - 1 and z1 (wrapped on a periodic z axis, absent otherwise)
let the device build bit-exact neighbour masks at the cut.  The step kernel
stores the outgoing c_z = +-1 populations of the two boundary planes
straight into the neighbours' ghost planes (peer memory), so there is no
separate exchange collective; device-side flags order the steps.
"""

from dataclasses import dataclass

import numpy as np

from .geometry import Geometry, Provenance
from .layouts import NodeDescriptorField


@dataclass
class SlabSpec:
    z0: int
    nz_global: int
    ghost_lo: np.ndarray | None   # (ny, nx) node types of plane z0 - 1, None = outside
    ghost_hi: np.ndarray | None   # (ny, nx) node types of plane z1, None = outside


def split_z(nz, parts):
    """Balanced contiguous z ranges [(z0, z1), ...]."""
    if parts < 1 or parts > nz:
        raise ValueError(f"cannot split {nz} planes into {parts} slabs")
    base, extra = divmod(nz, parts)
    out, z = [], 0
    for r in range(parts):
        n = base + (1 if r < extra else 0)
        out.append((z, z + n))
        z += n
    return out


def split_z_balanced(type_tag, parts, align=1):
    """Contiguous z ranges [(z0, z1), ...] with cuts on multiples of `align`
    (the tile edge for tile layouts, so every slab starts on a tile plane)
    that balance the non-solid node count -- the unit of work of a sparse
    step.  Each slab keeps at least one aligned block."""
    nz = type_tag.shape[0]
    nblk = -(-nz // align)
    if parts < 1 or parts > nblk:
        raise ValueError(f"cannot split {nz} planes into {parts} slabs aligned to {align}")
    per_plane = np.count_nonzero(type_tag.reshape(nz, -1), axis=1)
    per_blk = np.add.reduceat(per_plane, np.arange(0, nz, align))
    cum = np.concatenate([[0], np.cumsum(per_blk)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, parts):
        # block boundary closest to the r-th share, leaving room for the rest
        b = int(np.argmin(np.abs(cum - total * r / parts)))
        b = min(max(b, cuts[-1] + 1), nblk - (parts - r))
        cuts.append(b)
    cuts.append(nblk)
    return [(c0 * align, min(c1 * align, nz)) for c0, c1 in zip(cuts[:-1], cuts[1:])]


def neighbours(rank, world, periodic_z):
    lo = rank - 1 if rank > 0 else (world - 1 if periodic_z and world > 1 else None)
    hi = rank + 1 if rank < world - 1 else (0 if periodic_z and world > 1 else None)
    return lo, hi


def slab_geometry(geometry, z0, z1):
    """Cut planes [z0, z1) of a global Geometry into a slab Geometry and its
    SlabSpec (ghost node types included)."""
    d = geometry.descriptors
    nz = d.type_tag.shape[0]
    per = d.periodic
    sl = slice(z0, z1)
    local = NodeDescriptorField(d.type_tag[sl], d.bc_index[sl], d.orientation[sl], periodic=per)
    g = Geometry(descriptors=local, boundary_values=geometry.boundary_values,
                 porosity=geometry.porosity,
                 provenance=Provenance(case=geometry.provenance.case,
                                       params=dict(geometry.provenance.params),
                                       seed=geometry.provenance.seed))
    if z1 - z0 == nz:
        return g, None
    glo = d.type_tag[z0 - 1] if z0 > 0 else (d.type_tag[nz - 1] if per[2] else None)
    ghi = d.type_tag[z1] if z1 < nz else (d.type_tag[0] if per[2] else None)
    spec = SlabSpec(z0=z0, nz_global=nz, ghost_lo=None if glo is None else glo.copy(),
                    ghost_hi=None if ghi is None else ghi.copy())
    return g, spec


def connect_local(sims, periodic_z):
    """Wire in-process slab Simulations (list ordered by z) to each other."""
    blobs = [s.halo_blob() for s in sims]
    for r, s in enumerate(sims):
        lo, hi = neighbours(r, len(sims), periodic_z)
        s.connect_halo(None if lo is None else blobs[lo], None if hi is None else blobs[hi])


def connect_distributed(sim, periodic_z, group=None):
    """Exchange halo blobs over torch.distributed and wire this rank's slab to
    its z neighbours (rank - 1 below, rank + 1 above)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    blobs = [None] * world
    dist.all_gather_object(blobs, sim.halo_blob(), group=group)
    lo, hi = neighbours(rank, world, periodic_z)
    sim.connect_halo(None if lo is None else blobs[lo], None if hi is None else blobs[hi])
    dist.barrier(group)


def channel_slab(n_x, n_y, nz_local, rank, world, inlet_u=0.05, outlet_rho=1.0):
    """Rank `rank`'s slab of the z-periodic channel (config C2 per GPU, weak
    scaling): global extent n_x x n_y x (nz_local * world), every plane the
    same, so the slab is built directly without the global arrays."""
    from .geometry import VelocityInlet, build_channel
    g = build_channel(n_x, n_y, nz_local, VelocityInlet((inlet_u, 0.0, 0.0)),
                      outlet_rho=outlet_rho, periodic_z=True)
    if world == 1:
        return g, None
    plane = g.descriptors.type_tag[0].copy()
    return g, SlabSpec(z0=rank * nz_local, nz_global=nz_local * world, ghost_lo=plane,
                       ghost_hi=plane.copy())


def duct_slab(n_x, n_y, nz_local, rank, world, u_in=0.05, outlet_rho=1.0):
    """Rank `rank`'s slab of the z-duct (config C5): velocity inlet on the
    global z = 0 plane, pressure outlet on the last plane, bounce-back x/y
    faces; built per slab (the global arrays never exist)."""
    from .geometry import build_duct_z, from_arrays
    full = build_duct_z(n_x, n_y, 3, u_in=u_in, outlet_rho=outlet_rho)
    d = full.descriptors
    nzg = nz_local * world
    z0 = rank * nz_local
    idx = [0 if z == 0 else (2 if z == nzg - 1 else 1) for z in range(z0, z0 + nz_local)]
    g = from_arrays("duct_z", d.type_tag[idx], full.boundary_values, d.bc_index[idx],
                    d.orientation[idx], params=full.provenance.params)
    if world == 1:
        return g, None
    ghost = lambda z: None if not 0 <= z < nzg else d.type_tag[0 if z == 0 else (2 if z == nzg - 1 else 1)].copy()
    return g, SlabSpec(z0=z0, nz_global=nzg, ghost_lo=ghost(z0 - 1), ghost_hi=ghost(z0 + nz_local))
