"""Multi-GPU leg of bench.py (launched by torchrun, one rank per GPU).

Default: weak scaling of config C5: every rank owns a 1024 x 1024 x 256
z-slab of the duct 1024 x 1024 x (256 N) (velocity inlet at z = 0, pressure
outlet at the top; N = 8 is the full 1024 x 1024 x 2048 domain).  Rank 0
also times its slab geometry ALONE on its GPU (no neighbours) after the
multi-rank run, so the line carries the per-GPU solo rate the weak-scaling
efficiency is measured against.  --workload channel512 runs the C2 ring
(512^3 per rank, z-periodic), --workload c5 the strong-scaling split.  The step
kernel stores the outgoing c_z = +-1 populations of its two boundary planes
straight into the neighbours' ghost planes (CUDA IPC peer memory over
NVLink), device flags order the steps.  Timing: barrier + synchronize, K
steps timed with CUDA events on each rank's solver stream, MAX over ranks.
"""

import json
import os
import time

import numpy as np


def run_multi(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_2108_13241_b200 as lb
    from bench import METRIC, PDF_BYTES_PER_NODE_F32, ClockSampler, measured_peak
    from paper_2108_13241_b200.distributed import channel_slab, connect_distributed, duct_slab

    if os.environ.get("LBM_BENCH_SAME_GPU") == "1":
        # functional check of the multi-rank path on a single-GPU box: every
        # rank on device 0, gloo plumbing (NCCL refuses two ranks per GPU)
        local = 0
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
        dev = "cpu"
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dev = "cuda"
    workload = args.workload or "duct"
    scaling = "weak"
    if workload == "c5":
        # strong scaling of the whole C5 domain: 2048 / N planes per GPU (AB
        # fits from N = 2; N = 1 is bench.py --workload c5 with the A-A scheme)
        if 2048 % world:
            raise SystemExit(f"c5 needs N dividing 2048, got {world}")
        geom, spec = duct_slab(1024, 1024, 2048 // world, rank, world)
        params = lb.FlowParams.from_viscosity(U=0.05, L=1023, nu=0.1)
        desc = (f"C5 strong scaling: D3Q19 duct 1024x1024x2048 along z in {world} z-slabs of "
                f"1024x1024x{2048 // world}, velocity inlet / pressure outlet, fp32")
        periodic = False
        scaling = "strong"
    elif workload in ("duct", "c5weak"):
        geom, spec = duct_slab(1024, 1024, 256, rank, world)
        params = lb.FlowParams.from_viscosity(U=0.05, L=1023, nu=0.1)
        desc = (f"C5: D3Q19 duct 1024x1024x{256 * world} along z, z-slabs of 1024x1024x256 per "
                "GPU, velocity inlet / pressure outlet, fp32")
        periodic = False
    else:
        geom, spec = channel_slab(512, 512, 512, rank, world)
        params = lb.FlowParams.from_viscosity(U=0.05, L=511, nu=0.25)
        desc = (f"C2 weak scaling: D3Q19 channel 512x512x{512 * world} (z-periodic ring), "
                "z-slab of 512^3 per GPU, fp32")
        periodic = True
    scheme = args.scheme or "ab"
    sim = lb.Simulation(geom, params, layout="dense", scalar=np.float32, device=local, slab=spec,
                        scheme=scheme)
    connect_distributed(sim, periodic_z=periodic)
    sim.initialize(1.0)
    sim.step(args.warmup)
    launches0 = sim.launches_total
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        clk.mark_start()
        t0 = time.perf_counter()
        sim.step(args.steps)
        t1 = time.perf_counter()
        clk.mark_end()
    dist.barrier()
    ms = sim.last_step_ms
    t = torch.tensor([ms, t1 - t0], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, wall_max = float(t[0]), float(t[1])
    nons = torch.tensor([sim.active_node_count], dtype=torch.float64, device=dev)
    dist.all_reduce(nons)
    total_nons = float(nons[0])
    launches = sim.launches_total - launches0
    clocks = clk.summary()
    mlups = total_nons * args.steps / (ms_max / 1e3) / 1e6
    peak, peak_src = measured_peak()
    per_gpu_nodes = total_nons / world
    # algorithmic bytes as at N = 1: 152 B per non-solid node + the flag /
    # bitmap bytes the step reads, plus the halo planes pushed to the peers
    meta = float(sim.stats().meta_bytes_per_step)
    nx, ny = geom.dims[0], geom.dims[1]
    halo = 2 * 5 * nx * ny * 4 if spec is not None else 0
    alg = per_gpu_nodes * PDF_BYTES_PER_NODE_F32 + meta + halo
    achieved = alg / (ms_max / args.steps / 1e3) / 1e9
    finite = True
    try:
        sim.check_finite()
    except Exception:
        finite = False
    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": mlups, "unit": "MLUPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": desc, "layout": "dense", "scheme": scheme,
                       "nodes_per_gpu": int(per_gpu_nodes),
                       "l2": "state per GPU >> 126 MB L2 (no flush needed)",
                       "parallelism": f"z-slab x{world}, fused peer-store halo (CUDA IPC)"},
            "mlups_per_gpu": mlups / world,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                         "alg_bytes_per_gpu_launch": alg, "alg_bytes_per_node": alg / per_gpu_nodes},
            "e2e": None, "gpu_launches": int(launches), "clocks": clocks,
            "wall_s_max": wall_max, "finite": finite,
        }
    sim.close()
    del sim
    # e2e through the public API: slab geometry upload + halo wiring +
    # initialize + step(K) + macroscopic readback, wall clock, max over ranks
    dist.barrier()
    t0 = time.perf_counter()
    s2 = lb.Simulation(geom, params, layout="dense", scalar=np.float32, device=local, slab=spec,
                       scheme=scheme)
    connect_distributed(s2, periodic_z=periodic)
    s2.initialize(1.0)
    s2.step(args.steps)
    fields = s2.macroscopic_fields()
    t1 = time.perf_counter()
    te = torch.tensor([t1 - t0], dtype=torch.float64, device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    d = geom.descriptors
    h2d = d.type_tag.nbytes + d.orientation.nbytes + d.bc_index.nbytes
    d2h = sum(a.nbytes for a in fields)
    del fields
    s2.close()
    # rank 0: the same slab geometry alone on its GPU (no halo), same K / W
    solo = None
    dist.barrier()
    if rank == 0 and workload != "c5":
        if workload == "channel512":
            g1 = lb.build_channel(512, 512, 512, lb.VelocityInlet((0.05, 0.0, 0.0)))
        else:
            g1 = lb.build_duct_z(1024, 1024, 256)
        s1 = lb.Simulation(g1, params, layout="dense", scalar=np.float32, device=local, scheme=scheme)
        s1.initialize(1.0)
        s1.step(args.warmup)
        s1.step(args.steps)
        solo = {"value": s1.active_node_count * args.steps / (s1.last_step_ms / 1e3) / 1e6,
                "unit": "MLUPS", "what": "rank 0's slab extent as a standalone domain on its GPU "
                "(no neighbours), same K / W, CUDA events",
                "weak_scaling_efficiency": None}
        solo["weak_scaling_efficiency"] = (mlups / world) / solo["value"]
        s1.close()
        del s1, g1
    dist.barrier()
    if rank == 0:
        line["solo_mlups_per_gpu"] = solo
        line["e2e"] = {"value": total_nons * args.steps / float(te[0]) / 1e6, "unit": "MLUPS",
                       "h2d_bytes_per_step": world * h2d / args.steps,
                       "d2h_bytes_per_step": world * d2h / args.steps,
                       "what": "per rank: Simulation(slab) + halo wiring + initialize + step(K) + "
                               "macroscopic_fields(), wall clock, max over ranks"}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
