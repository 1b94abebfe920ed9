"""Tile-layout z-slabs on ONE GPU: the porous 512^3 medium as 1, 2 or 4
in-process slabs (cut on tile planes, balanced by non-solid count), each on
its own stream; measures the ghost-plane exchange cost of the slab kernel."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_13241_b200 as lb
from paper_2108_13241_b200.distributed import connect_local, slab_geometry, split_z_balanced

steps, tile = 200, (4, 8, 16)
scheme = sys.argv[1] if len(sys.argv) > 1 else "ab"   # "aa": A-A tile slabs (round 2)
geom = lb.build_porous_random(512, 0.5, seed=0, radius_range=(4, 32))
params = lb.FlowParams.from_viscosity(U=0.05, L=511, nu=0.5)
one = lb.Simulation(geom, params, layout="pointer_tile", scalar=np.float32, tile=tile, scheme=scheme)
one.initialize(1.008); one.step(20); one.step(steps)
nons = one.active_node_count
print({"scheme": scheme, "kernel": "work list" if one.stats().tile_work_list else "CTA per tile", "slabs": 1, "ms_per_step": one.last_step_ms / steps, "mlups": nons * steps / one.last_step_ms / 1e3}, flush=True)
one.close()
for k in (2, 4):
    sims = []
    for z0, z1 in split_z_balanced(geom.descriptors.type_tag, k, align=tile[2]):
        g, spec = slab_geometry(geom, z0, z1)
        sims.append(lb.Simulation(g, params, layout="pointer_tile", scalar=np.float32, tile=tile, slab=spec,
                                  scheme=scheme))
    connect_local(sims, False)
    for s in sims: s.initialize(1.008)
    for s in sims: s.step(20, block=False)
    for s in sims: s.synchronize()
    for s in sims: s.step(steps, block=False)
    for s in sims: s.synchronize()
    ms = max(s.last_step_ms for s in sims)
    print({"scheme": scheme, "slabs": k, "ms_per_step": ms / steps, "mlups": nons * steps / ms / 1e3}, flush=True)
    for s in sims: s.close()
