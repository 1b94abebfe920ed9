"""Halo overhead of the fused z-slab exchange on ONE GPU: k slabs of a
512^2 x 512 z-periodic channel in one process (device pointers, one stream
each) vs the same domain as one handle.  Same device, so this measures the
kernel-side cost of the peer stores + wait/signal ordering, not NVLink."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_13241_b200 as lb
from paper_2108_13241_b200.distributed import channel_slab, connect_local

steps = 200
scheme = sys.argv[1] if len(sys.argv) > 1 else "ab"
params = lb.FlowParams.from_viscosity(U=0.05, L=511, nu=0.25)
g, _ = channel_slab(512, 512, 512, 0, 1)
one = lb.Simulation(g, params, scalar=np.float32, scheme=scheme)
one.initialize(1.0)
one.step(20)
one.step(steps)
t1 = one.last_step_ms
one.close()
print({"scheme": scheme, "slabs": 1, "ms_per_step": t1 / steps, "mlups": 512**3 * steps / t1 / 1e3}, flush=True)
for k in (2, 4):
    sims = []
    for r in range(k):
        gr, spec = channel_slab(512, 512, 512 // k, r, k)
        sims.append(lb.Simulation(gr, params, scalar=np.float32, slab=spec, scheme=scheme))
    connect_local(sims, True)
    for s in sims:
        s.initialize(1.0)
    for s in sims:
        s.step(20, block=False)
    for s in sims:
        s.synchronize()
    t0 = time.perf_counter()
    for s in sims:
        s.step(steps, block=False)
    for s in sims:
        s.synchronize()
    wall = time.perf_counter() - t0
    ms = max(s.last_step_ms for s in sims)
    print({"scheme": scheme, "slabs": k, "ms_per_step": ms / steps, "wall_ms_per_step": wall * 1e3 / steps,
           "mlups": 512**3 * steps / ms / 1e3}, flush=True)
    for s in sims:
        s.close()
