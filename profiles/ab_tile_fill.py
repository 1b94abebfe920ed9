"""A/B of tile shapes on one geometry per workload (built once, shapes
alternating in-process), with the node fill of the kept tiles for each shape:
the data behind the fill-based default tile choice.  Usage (GPU box):
python profiles/ab_tile_fill.py porous512@0.1 ... > gpurun_out/ab_tile_fill.txt"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2108_13241_b200 as lb  # noqa: E402

SHAPES = [tuple(int(v) for v in t.split(",")) for t in
          os.environ.get("SHAPES", "4,4,8 4,4,4 2,4,4 2,4,8").split()]
SCHEME = os.environ.get("SCHEME", "ab")
SCALAR = np.dtype(os.environ.get("SCALAR", "float32"))


def fill(live, t):
    tx, ty, tz = t
    nz, ny, nx = live.shape
    a = live.reshape(nz // tz, tz, ny // ty, ty, nx // tx, tx).sum(axis=(1, 3, 5))
    return float(a.sum() / (np.count_nonzero(a) * tx * ty * tz))


for w in sys.argv[1:]:
    geom, params, layout, _, rho0 = bench.build_workload(w)
    live = geom.descriptors.type_tag != 0
    fills = {str(t): round(fill(live, t), 4) for t in SHAPES}
    for rep in range(2):
        for t in SHAPES:
            sim = lb.Simulation(geom, params, layout=layout, scalar=SCALAR, tile=t, scheme=SCHEME)
            sim.initialize(rho0)
            r = lb.benchmark(sim, 50, 500)
            print(json.dumps({"workload": w, "tile": t, "rep": rep, "scheme": SCHEME, "scalar": SCALAR.name, "mlups": round(r.p_lups / 1e6),
                              "frac": round(r.u_b_with_flags, 4), "fill": fills[str(t)],
                              "work_list": bool(sim._handle.stats().tile_work_list)}), flush=True)
            sim.close()
