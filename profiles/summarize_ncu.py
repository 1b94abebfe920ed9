"""Summarise the ncu captures brought back in gpurun_out/ into
profiles/ncu_summary.json (read by bench.py for roofline.traffic) and
profiles/ncu_<tag>.md.

    python profiles/summarize_ncu.py <tag> [--dtype f32] [--scheme ab] [--tile x,y,z (default: from the capture's bench line)] [workload ...]

Entries are keyed by (workload, dtype, scheme, tile, kernel): bench.py only
takes `roofline.traffic` from a capture of the same configuration.
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
METRICS = [
    ("Kernel Name", "kernel"),
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_of_ncu_peak"),
    ("launch__registers_per_thread", "registers"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("sm__maximum_warps_per_active_cycle_pct", "occupancy_limit_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("smsp__inst_executed.sum", "warp_instructions"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_pct"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_long_scoreboard"),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
              "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def raw(rep):
    """Rows of `ncu -i rep --page raw --csv`; `rep` may also be that CSV,
    exported on the GPU box (profile.sh) so the large .ncu-rep stays there."""
    if rep.endswith(".csv"):
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {}
        for name, key in METRICS:
            if name in hdr:
                i = hdr.index(name)
                v = vals[i]
                try:
                    v = float(v.replace(",", "")) * UNIT_SCALE.get(units[i], 1.0)
                except ValueError:
                    pass
                d[key] = v
        out.append(d)
    return out


DENSE = ("channel512", "cavity64", "c5", "duct")


def logged_tile(tag, w):
    """The tile the captured bench run used: config.tile of its JSON line
    (ncu_<tag>_<w>.log, written by profile.sh)."""
    with open(os.path.join(OUT, f"ncu_{tag}_{w}.log")) as fh:
        for line in fh:
            if line.startswith("{"):
                return json.loads(line)["config"]["tile"]
    raise SystemExit(f"no bench line in ncu_{tag}_{w}.log: pass --tile")


def main():
    argv = sys.argv[1:]
    opts = {"--dtype": "f32", "--scheme": "ab", "--tile": "log"}
    rest = []
    while argv:
        a = argv.pop(0)
        if a in opts:
            opts[a] = argv.pop(0)
        else:
            rest.append(a)
    tag, wls = rest[0], rest[1:] or ["channel512"]
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    entries = json.load(open(path)).get("entries", []) if os.path.exists(path) else []
    md = [f"# ncu summary `{tag}` (`--set full --clock-control none`, one step-kernel launch; "
          f"{opts['--dtype']}, scheme {opts['--scheme']})\n",
          "| workload | kernel | ms | DRAM read GB | DRAM write GB | regs | warps active % | "
          "issue active % | L2 hit % | tensor pipe % |", "|---|---|---|---|---|---|---|---|---|---|"]
    for w in wls:
        rep = os.path.join(OUT, f"prof_{tag}_{w}.ncu-rep")
        if not os.path.exists(rep):
            rep = os.path.join(OUT, f"raw_{tag}_{w}.csv")
        if not os.path.exists(rep):
            continue
        k = raw(rep)[0]
        traffic = k["dram_read"] + k["dram_write"]
        if w.split("@")[0] in DENSE:
            tile = None
        elif opts["--tile"] == "log":
            tile = logged_tile(tag, w)
        else:
            tile = [int(v) for v in opts["--tile"].split(",")]
        e = {"workload": w, "dtype": opts["--dtype"], "scheme": opts["--scheme"], "tile": tile,
             "tag": tag, "kernel": k["kernel"].split("(")[0],
             "duration_ms": k["duration"] * 1e3, "dram_bytes_per_launch": traffic,
             "dram_read": k["dram_read"], "dram_write": k["dram_write"],
             "registers": k.get("registers"), "warps_active_pct": k.get("warps_active_pct"),
             "issue_active_pct": k.get("issue_active_pct"), "l2_hit_pct": k.get("l2_hit_pct"),
             "tensor_pipe_pct": k.get("tensor_pipe_pct"),
             "stall_long_scoreboard": k.get("stall_long_scoreboard")}
        key = lambda x: (x["workload"], x["dtype"], x["scheme"], x["tile"], x["kernel"])
        entries = [x for x in entries if key(x) != key(e)] + [e]
        md.append(f"| {w} | `{e['kernel']}` | {k['duration'] * 1e3:.3f} | "
                  f"{k['dram_read'] / 1e9:.3f} | {k['dram_write'] / 1e9:.3f} | {k.get('registers')} | "
                  f"{k.get('warps_active_pct', 0):.1f} | {k.get('issue_active_pct', 0):.1f} | "
                  f"{k.get('l2_hit_pct', 0):.1f} | {k.get('tensor_pipe_pct', 0) or 0:.1f} |")
    with open(path, "w") as fh:
        json.dump({"entries": entries}, fh, indent=1)
    with open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w") as fh:
        fh.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
