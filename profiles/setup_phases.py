"""Wall-clock phases of Simulation() for a sparse workload (LBM_TIMING=1 adds the C-side phases)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_13241_b200 as lb
from bench import build_workload
w = sys.argv[1] if len(sys.argv) > 1 else "porous512"
geom, params, layout, desc, rho0 = build_workload(w)
for rep in range(2):
    t = [time.perf_counter()]
    sim = lb.Simulation(geom, params, layout=layout, scalar=np.float32); t.append(time.perf_counter())
    sim.initialize(rho0); t.append(time.perf_counter())
    sim.step(100); t.append(time.perf_counter())
    f = sim.macroscopic_fields(); t.append(time.perf_counter())
    sim.close()
    print(w, [round(x, 3) for x in np.diff(t)], flush=True)
