"""Benchmark of the D3Q19 fused stream + BGK-collide hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload channel512|porous512|vascular1024|duct]

One JSON line on rank 0 (contract in the task statement):
  value  whole-job MLUPS over non-solid nodes, inputs resident in HBM,
         CUDA events on the solver stream around K steps, max over ranks;
  e2e    the same metric through the public Python API end to end
         (geometry upload, initialize, step(K), macroscopic readback);
  roofline  the step kernel's algorithmic bytes (156 B per non-solid node:
         19 reads + 19 writes fp32 + the 4-byte flag word) / average launch
         time, against MEASURED_PEAKS.json hbm_gbs;
  cpu_baseline  the CPU oracle (Numba port of the reference kernel) on the
         host cores, bounded sample of the same workload.
--impl reference times that CPU implementation alone (the reference arm).
N = 1 default: C2 (dense channel 512^3), plus a `sparse` block with C3
(porous 512^3 at phi ~0.5 and ~0.1) and C4 (vascular 1024^3) measured in the
same run.
N > 1 (torchrun): z-slab decomposition of the C5 duct 1024x1024x(256 N), one
rank per GPU, halo planes exchanged inside the step kernel (weak scaling;
N = 8 is the full 1024x1024x2048 domain); rank 0 also reports its slab's
solo rate (bench_multi.py).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MLUPS per GPU and whole box (1/2/4/8 B200) and % of HBM roofline vs CPU ref"
DEFAULT_SCHEME = "ab"
BYTES_PER_NODE_F32 = 19 * 4 * 2 + 4     # with one flag word per node
PDF_BYTES_PER_NODE_F32 = 19 * 4 * 2


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def expected_kernel(layout, scheme, dtype, tile_work_list):
    """Name prefix of the step kernel the library launches for this
    configuration (csrc/lbm19.cu launch_step / launch_tiles)."""
    t = "float" if dtype == "f32" else "double"
    if layout in ("tile", "pointer_tile"):
        if scheme == "aa":
            return f"k_step_tiles_aa_w<{t}" if tile_work_list else f"k_step_tiles_aa<{t}"
        return f"k_step_tiles_w<{t}" if tile_work_list else f"k_step_tiles_x<{t}"
    return f"k_step_dense_aa<{t}" if scheme == "aa" else f"k_step_dense<{t}"


def ncu_traffic(workload, dtype, scheme, tile, kernel_prefix):
    """Per-launch DRAM bytes (read + write) of the step kernel from a
    committed `ncu --set full` capture of the SAME configuration
    (profiles/ncu_summary.json entries keyed by workload, dtype, scheme,
    tile and kernel), else None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            entries = json.load(fh)["entries"]
    except Exception:
        return None
    for e in entries:
        if (e.get("workload") == workload and e.get("dtype") == dtype and e.get("scheme") == scheme
                and (e.get("tile") or None) == (list(tile) if tile else None)
                and str(e.get("kernel", "")).replace("void ", "").startswith(kernel_prefix)):
            return e.get("dram_bytes_per_launch")
    return None


def measure_device(lb, workload, geom, params, layout, scheme, tile, dtype, rho0, device, steps,
                   warmup):
    """Device-timed K steps (inputs resident in HBM, CUDA events on the
    solver stream) with the roofline figures of the step kernel."""
    scalar = np.float32 if dtype == "f32" else np.float64
    esz = np.dtype(scalar).itemsize
    sim = lb.Simulation(geom, params, layout=layout, scalar=scalar, device=device, scheme=scheme,
                        tile=tile)
    sim.initialize(rho0)
    with ClockSampler(device) as clk:
        sim.step(warmup)
        launches0 = sim.launches_total
        clk.mark_start()
        sim.step(steps)    # CUDA events on the solver stream around K launches
        clk.mark_end()
    ms = sim.last_step_ms
    launches = sim.launches_total - launches0
    clocks = clk.summary()
    nons = sim.active_node_count
    st = sim.stats()
    mlups = nons * steps / (ms / 1e3) / 1e6
    peak, _ = measured_peak()
    per_launch_ms = ms / launches
    # algorithmic bytes per launch: 19 reads + 19 writes per non-solid node,
    # plus the flag / index bytes this design's step reads (dense: flag words
    # of non-uniform warp chunks + the uniform-chunk bitmap; tiles: nbr27 +
    # brick masks + flag words of live bricks + the work list)
    alg_bytes = nons * 2 * 19 * esz + int(st.meta_bytes_per_step)
    achieved = alg_bytes / (per_launch_ms / 1e3) / 1e9
    sane = bool(np.isfinite(sim.total_mass()))
    tiled = layout in ("tile", "pointer_tile")
    kern = expected_kernel(layout, scheme, dtype, bool(st.tile_work_list))
    tile = sim.tile if tiled else None     # the facade's choice when tile is None
    sim.close()
    del sim
    return {"value": mlups, "unit": "MLUPS", "mlups": mlups, "frac": achieved / peak, "steps": steps,
            "achieved_gbs": achieved, "ms": ms, "ms_per_step": ms / steps,
            "per_launch_ms": per_launch_ms, "alg_bytes": alg_bytes, "alg_bytes_per_launch": alg_bytes,
            "alg_bytes_per_node": alg_bytes / nons, "nons": nons, "non_solid_nodes": int(nons),
            "porosity": nons / float(st.n_nodes), "stats": st, "launches": launches,
            "gpu_launches": int(launches), "clocks": clocks, "finite": sane, "kernel": kern,
            "tile_kernel": (("warp work list" if st.tile_work_list else "CTA per tile") if tiled else None),
            "tile": list(tile) if tiled else None,
            "traffic": ncu_traffic(workload, dtype, scheme, tile, kern)}


def build_workload(name, rank=0, world=1):
    import paper_2108_13241_b200 as lb
    if name == "channel512":
        geom = lb.build_channel(512, 512, 512, lb.VelocityInlet((0.05, 0.0, 0.0)))
        params = lb.FlowParams.from_viscosity(U=0.05, L=511, nu=0.25)
        desc = ("C2: D3Q19 dense channel 512^3, velocity inlet u=0.05 (x=0), pressure "
                "outlet rho=1 (x=511), bounce-back y walls, periodic z, nu=0.25")
        return geom, params, "dense", desc, 1.0
    if name == "cavity64":
        geom = lb.build_cavity(64, 64, 64, 0.1)
        params = lb.FlowParams.from_reynolds(U=0.1, L=63, Re=100)
        desc = "C1: D3Q19 lid-driven cavity 64^3, Re 100(L2-resident; parity config)"
        return geom, params, "dense", desc, 1.0
    if name.startswith("porous512@"):
        phi = float(name.split("@")[1])
        geom = lb.build_porous_random(512, phi, seed=0, radius_range=(4, 32))
        params = lb.FlowParams.from_viscosity(U=0.05, L=511, nu=0.5)
        desc = (f"C3: D3Q19 random-sphere porous medium 512^3, phi target {phi} "
                f"(achieved {geom.porosity:.3f}), pointer-tile")
        return geom, params, "pointer_tile", desc, 1.008
    if name == "porous512":
        geom = lb.build_porous_random(512, 0.5, seed=0, radius_range=(4, 32))
        params = lb.FlowParams.from_viscosity(U=0.05, L=511, nu=0.5)
        desc = ("C3: D3Q19 random-sphere porous medium 512^3, phi~0.5, pointer-tile, "
                "pressure 1.016 -> 1.0")
        return geom, params, "pointer_tile", desc, 1.008
    if name == "vascular1024":
        geom = lb.build_vascular(1024, seed=0, fluid_fraction=0.05)
        params = lb.FlowParams.from_viscosity(U=0.05, L=1023, nu=0.1)
        desc = "C4: D3Q19 vascular tube forest 1024^3, ~5% non-solid, pointer-tile"
        return geom, params, "pointer_tile", desc, 1.0
    if name == "c5":
        geom = lb.build_duct_z(1024, 1024, 2048)
        params = lb.FlowParams.from_viscosity(U=0.05, L=1023, nu=0.1)
        desc = ("C5 whole domain on one GPU: D3Q19 duct 1024x1024x2048 along z, velocity inlet "
                "z=0, pressure outlet z=2047, bounce-back x/y faces (fp32 needs the AA scheme)")
        return geom, params, "dense", desc, 1.0
    if name == "duct":
        geom = lb.build_duct_z(1024, 1024, 256)
        params = lb.FlowParams.from_viscosity(U=0.05, L=1023, nu=0.1)
        desc = "C5 slab: D3Q19 duct 1024x1024x256 along z"
        return geom, params, "dense", desc, 1.0
    raise SystemExit(f"unknown workload {name}")


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region.

    The sampler starts before the warm-up (nvidia-smi needs ~0.1 s to produce
    its first row); mark_start() / mark_end() bracket the timed region and
    summary() keeps the rows stamped inside it -- or, for a region shorter
    than the 20 ms sampling interval, the rows nearest to it (within 0.1 s),
    and says so."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None
        self.t0 = self.t1 = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *exc):
        if self.proc is not None:
            # a region shorter than nvidia-smi's start-up: wait (<= 0.5 s) for
            # the first row, taken while the clocks are still at their load value
            t_end = time.time() + 0.5
            while time.time() < t_end:
                try:
                    if os.path.getsize(self.path) > 0:
                        break
                except OSError:
                    break
                time.sleep(0.01)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        import datetime
        rows = []
        try:
            with open(self.path) as fh:
                for line in fh:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 10:
                        try:
                            ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                        except ValueError:
                            ts = None
                        rows.append((ts, parts[1:]))
            os.unlink(self.path)
        except Exception:
            pass
        window = "whole sampler run"
        if self.t0 is not None and self.t1 is not None and rows:
            inside = [r for r in rows if r[0] is not None and self.t0 <= r[0] <= self.t1]
            if inside:
                rows, window = inside, "inside the timed region"
            else:
                near = [r for r in rows if r[0] is not None and self.t0 - 0.1 <= r[0] <= self.t1 + 0.1]
                if near:
                    rows, window = near, "within 0.1 s of a timed region shorter than the sampling interval"
                else:
                    after = [r for r in rows if r[0] is not None and self.t1 < r[0] <= self.t1 + 0.5][:1]
                    rows, window = after, ("first row after a timed region shorter than nvidia-smi's start-up "
                                           "(within 0.5 s)")
        rows = [r[1] for r in rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows), "window": window}


CPU_SLAB_NZ = 32   # the CPU sample: 512 x 512 x 32 z-periodic slab of C2


def _cpu_port_sim(duct=False):
    import numba

    from oracle.step19 import OracleSim
    import paper_2108_13241_b200 as lb
    cores = len(os.sched_getaffinity(0))
    numba.set_num_threads(cores)
    if duct:   # the multi-GPU workload (C5 duct): a 1024 x 1024 x 8 slab of it
        geom = lb.build_duct_z(1024, 1024, CPU_SLAB_NZ // 4)
        omega = lb.FlowParams.from_viscosity(U=0.05, L=1023, nu=0.1).omega
    else:
        geom = lb.build_channel(512, 512, CPU_SLAB_NZ, lb.VelocityInlet((0.05, 0.0, 0.0)))
        omega = lb.FlowParams.from_viscosity(U=0.05, L=511, nu=0.25).omega
    d = geom.descriptors
    kinds, vel, rho = geom.boundary_values.as_arrays()
    sim = OracleSim(d.type_tag, d.orientation, d.bc_index, kinds, vel, rho, omega,
                    dtype=np.float32, periodic=d.periodic)
    sim.initialize(1.0)
    return sim, int(np.count_nonzero(d.type_tag)), cores


def _cpu_protocol(steps, warmup, duct=False):
    where = (f"1024x1024x{CPU_SLAB_NZ // 4} slab of the C5 duct (same per-node work as C5)" if duct else
             f"512x512x{CPU_SLAB_NZ} z-periodic slab of the C2 channel (same per-node work as C2)")
    return (f"one protocol for both arms: {where}, fp32, Numba port of the reference kernel (oracle/step19.py) "
            f"parallel over rows with numba threads = host cores; {warmup} warm-up step(s) (JIT), then "
            f"{steps} steps timed as one continuous wall-clock region")


def cpu_baseline(workload_name, steps=190):
    """The reference's CPU path (the Numba port, oracle/step19.py) on the host
    cores: a bounded ~20 s sample of C2-type work, the same protocol as the
    --impl reference arm (only the step count differs)."""
    sim, nons, cores = _cpu_port_sim()
    sim.step(1)   # JIT
    t0 = time.perf_counter()
    sim.step(steps)
    v = nons * steps / (time.perf_counter() - t0) / 1e6
    return {"value": v, "unit": "MLUPS", "cores": cores, "kind": "port",
            "sample": _cpu_protocol(steps, 1) + f" ({nons * steps / 1e6:.0f} M node updates)"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # each timed step = one step of the CPU port on the sample slab of the
    # workload our arm runs at this N (C2 at N = 1, the C5 duct at N > 1)
    duct = int(os.environ.get("WORLD_SIZE", str(args.gpus))) > 1
    sim, nons, cores = _cpu_port_sim(duct)
    sim.step(max(args.warmup, 1))
    t0 = time.perf_counter()
    sim.step(args.steps)
    dt = time.perf_counter() - t0
    v = nons * args.steps / dt / 1e6
    sample = _cpu_protocol(args.steps, max(args.warmup, 1), duct)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "MLUPS",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": ("C5 duct 1024x1024x(256 N) (CPU sample slab)" if duct else
                                    "C2 channel 512^3 (CPU sample slab)"), "sample_nodes": nons},
            "cpu_baseline": {"value": v, "unit": "MLUPS", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": "MLUPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=100)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None)
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"],
                    help="storage/arithmetic type (the reference's Simulation defaults to float64)")
    ap.add_argument("--tile", default="auto",
                    help="tile edges x,y,z for tile layouts, or 'auto' (the API default: 4x4x8, or 4x4x4 "
                         "when the kept 4x4x8 tiles are < 70 %% non-solid; profiles/tile_sweep_r02ag.txt, "
                         "profiles/ab_tile_fill_r02al.txt)")
    ap.add_argument("--layout", default=None, choices=["dense", "tile", "pointer_tile", "bitmask_node"],
                    help="override the workload's storage layout (design experiments)")
    ap.add_argument("--scheme", default=None, choices=["ab", "aa"],
                    help="PDF storage: two buffers (ab) or one in place (aa)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sparse", action="store_true",
                    help="skip the C3/C4 sparse block of the default (C2) line")
    ap.add_argument("--variants", default=None,
                    help="comma list of step-kernel variants to time in-process (tuning)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
        return

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        from bench_multi import run_multi
        run_multi(args, rank, world, local)
        return

    import paper_2108_13241_b200 as lb
    workload = args.workload or "channel512"
    # CPU baseline first, before this process creates a CUDA context (measured
    # ~40 % slower afterwards on the shared host: profiles/cpu_baseline_check_r01.txt)
    cpu = None
    if not args.no_cpu and not args.variants:
        try:
            cpu = cpu_baseline(workload)
        except Exception as exc:  # reported, never fatal for the GPU number
            cpu = {"value": None, "error": repr(exc)}
    geom, params, layout, desc, rho0 = build_workload(workload)
    layout = args.layout or layout
    scheme = args.scheme or ("aa" if workload == "c5" else DEFAULT_SCHEME)
    tile = None if args.tile == "auto" else tuple(int(v) for v in args.tile.split(","))
    scalar = np.float32 if args.dtype == "f32" else np.float64
    esz = np.dtype(scalar).itemsize
    if args.variants:
        for v in args.variants.split(","):
            # "3" selects LBM_STEP_VARIANT=3; "KEY=VAL;KEY=VAL" sets library switches
            if "=" in v:
                for kv in v.split(";"):
                    k, val = kv.split("=")
                    os.environ[k] = val
            else:
                os.environ["LBM_STEP_VARIANT"] = v
            sim = lb.Simulation(geom, params, layout=layout, scalar=scalar, device=local,
                                scheme=scheme, tile=tile)
            sim.initialize(rho0)
            sim.step(args.warmup)
            sim.step(args.steps)
            ms = sim.last_step_ms
            nons = sim.active_node_count
            mlups = nons * args.steps / (ms / 1e3) / 1e6
            peak, _ = measured_peak()
            alg = nons * 2 * 19 * esz + int(sim.stats().meta_bytes_per_step)
            frac = alg / (ms / args.steps / 1e3) / 1e9 / peak
            print(json.dumps({"workload": workload, "variant": v, "tile": list(sim.tile), "mlups": round(mlups),
                              "frac": round(frac, 4), "alg_B_per_node": round(alg / nons, 2),
                              "ms_per_step": ms / args.steps}), flush=True)
            sim.close()
        return
    dev = measure_device(lb, workload, geom, params, layout, scheme, tile, args.dtype, rho0, local,
                         args.steps, args.warmup)
    st, nons, ms, launches, clocks = dev["stats"], dev["nons"], dev["ms"], dev["launches"], dev["clocks"]
    mlups, per_launch_ms = dev["mlups"], dev["per_launch_ms"]
    peak, peak_src = measured_peak()
    alg_bytes, achieved, sane = dev["alg_bytes"], dev["achieved_gbs"], dev["finite"]

    e2e = None
    if not args.no_e2e:
        d = geom.descriptors
        h2d = d.type_tag.nbytes + d.orientation.nbytes + d.bc_index.nbytes
        nx, ny, nz = geom.dims
        # result read back: (rho, u) in f64, or rho alone past 2^30 nodes (host RAM)
        big = nx * ny * nz > (1 << 30)
        d2h = (1 if big else 4) * 8 * nx * ny * nz
        t0 = time.perf_counter()
        s2 = lb.Simulation(geom, params, layout=layout, scalar=scalar, device=local,
                           scheme=scheme, tile=tile)
        t_setup = time.perf_counter() - t0
        s2.initialize(rho0)
        t_init = time.perf_counter()
        s2.step(args.steps)
        t_step = time.perf_counter()
        fields = s2.density_field() if big else s2.macroscopic_fields()
        t1 = time.perf_counter()
        if os.environ.get("LBM_TIMING") == "1":
            sys.stderr.write(f"[bench timing] e2e readback call {1e3 * (t1 - t_step):.3f} ms\n")
        e2e = {"value": nons * args.steps / (t1 - t0) / 1e6, "unit": "MLUPS",
               "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
               "what": "Simulation(geometry) [descriptor upload] + initialize + step(K) + "
                       + ("density_field() [f64 rho readback]" if big else
                          "macroscopic_fields() [f64 rho,u readback]") + ", wall clock",
               # the device geometry pipeline: descriptor upload, flag words,
               # tile keep/scan/compaction/nbr27, brick masks
               "setup_s": t_setup, "setup_mnodes_per_s": nx * ny * nz / t_setup / 1e6,
               "init_s": t_init - t0 - t_setup, "step_s": t_step - t_init, "readback_s": t1 - t_step,
               "readback_gbs": d2h / (t1 - t_step) / 1e9}
        del fields
        s2.close()

    # second calibration: this library's own device copy kernel on a 4 GiB
    # block (the reference's copy micro-benchmark, dense pattern)
    copy_gbs = None
    try:
        copy_gbs = lb.copy_bandwidth_bench("dense", 4 << 30, repetitions=20, warmup=3, device=local) / 1e9
    except Exception:
        copy_gbs = None


    # driver-visible sparse configs (C3 at two porosities, C4), measured in
    # this same run with the same K / W: the >= 70 % sparse target
    sparse = None
    if workload == "channel512" and args.dtype == "f32" and not args.no_sparse:
        sparse = {}
        for w in ("porous512", "porous512@0.1", "vascular1024"):
            try:
                g2, p2, l2, d2, r2 = build_workload(w)
                # at least 500 timed steps (0.3-1 s), so the clock sampler sees the region
                m = measure_device(lb, w, g2, p2, l2, DEFAULT_SCHEME, tile, args.dtype, r2, local,
                                   max(args.steps, 500), args.warmup)
                sparse[w] = {k: m[k] for k in ("value", "unit", "frac", "achieved_gbs", "ms_per_step", "steps",
                                               "alg_bytes_per_launch", "alg_bytes_per_node",
                                               "traffic", "non_solid_nodes", "porosity", "tile", "tile_kernel",
                                               "gpu_launches", "clocks")}
                sparse[w]["workload"] = d2
                del g2
            except Exception as exc:  # reported, never fatal for the headline
                sparse[w] = {"error": repr(exc)}

    line = {
        "metric": METRIC, "value": mlups, "unit": "MLUPS", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": desc, "layout": layout, "scheme": scheme,
                   "tile": dev["tile"],
                   "tile_kernel": (("warp work list" if st.tile_work_list else "CTA per tile")
                                   if layout in ("tile", "pointer_tile") else None),
                   "nodes": int(st.n_nodes),
                   "non_solid_nodes": int(nons), "tiles": int(st.n_tiles),
                   "l2": "state 2x19 planes >> 126 MB L2 (no flush needed)",
                   "parallelism": "single GPU"},
        "mlups_per_gpu": mlups,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": dev["traffic"],
                     "peak_source": peak_src,
                     "alg_bytes_per_launch": alg_bytes,
                     "alg_bytes_per_node": alg_bytes / nons,
                     "meta_bytes_per_launch": int(st.meta_bytes_per_step),
                     "copy_gbs": copy_gbs,
                     "frac_of_copy": (achieved / copy_gbs) if copy_gbs else None,
                     "frac_152B": nons * 152 / (per_launch_ms / 1e3) / 1e9 / peak if esz == 4 else None,
                     "frac_156B": nons * 156 / (per_launch_ms / 1e3) / 1e9 / peak if esz == 4 else None},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
        "finite": sane,
    }
    if sparse is not None:
        line["sparse"] = sparse
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
