"""Wall-clock phases of the e2e path of bench.py (public API, host buffers)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_13241_b200 as lb

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
geom = lb.build_channel(512, 512, 512, lb.VelocityInlet((0.05, 0.0, 0.0)))
params = lb.FlowParams.from_viscosity(U=0.05, L=511, nu=0.25)
for rep in range(2):
    t = [time.perf_counter()]
    sim = lb.Simulation(geom, params, layout="dense", scalar=np.float32)
    t.append(time.perf_counter())
    sim.initialize(1.0)
    t.append(time.perf_counter())
    sim.step(steps)
    t.append(time.perf_counter())
    f = sim.macroscopic_fields()
    t.append(time.perf_counter())
    sim.close()
    d = np.diff(t)
    print({"create": round(d[0], 3), "init": round(d[1], 3), "step": round(d[2], 3),
           "readback": round(d[3], 3), "total": round(t[-1] - t[0], 3),
           "e2e_mlups": round(sim_n := 512**3 * steps / (t[-1] - t[0]) / 1e6)}, flush=True)
