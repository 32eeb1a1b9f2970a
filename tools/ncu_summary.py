"""Summarise ncu outputs into committed profiles/ files.

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/X_launches.txt
    python tools/ncu_summary.py full gpurun_out/radiomap.ncu-rep > profiles/X_full.txt
    python tools/ncu_summary.py traffic gpurun_out/k_map_trace.ncu-rep > profiles/traffic_k_map_trace.json
"""

import collections
import csv
import io
import json
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers",
    "smsp__average_warp_latency_issue_stalled_no_instruction",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    agg = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        agg.setdefault(k, []).append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"# ncu launch list ({path}); gpu__time_duration.sum, --clock-control none")
    print(f"# cold-cache, serialised per-launch times; shares are what matters")
    print(f"{'kernel':58s} {'launches':>8s} {'total ms':>10s} {'avg ms':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:58s} {len(v):8d} {sum(v) / 1e6:10.3f} {sum(v) / len(v) / 1e6:10.4f} "
              f"{100 * sum(v) / tot:6.1f}%")


def _raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def _dur(vals):
    try:
        return float(vals.get("gpu__time_duration.sum", "0").replace(",", ""))
    except ValueError:
        return 0.0


def full(rep):
    """Raw metrics of the longest launch in the report + its details sections."""
    raw = _raw(rep)
    best = max(range(len(raw)), key=lambda i: _dur(raw[i][0]))
    for vals, units in raw[best:best + 1]:
        print(f"## {vals.get('Kernel Name', '?')[:120]}  (longest of {len(raw)} captured launches,"
              f" #{best})")
        for m in FULL_METRICS:
            if m in vals:
                print(f"{m:70s} {vals[m]:>16s} {units.get(m, '')}")
        # warp stall reasons (cycles per issued instruction) and local-memory traffic
        stalls = []
        for m, v in vals.items():
            if m.startswith("smsp__average_warps_issue_stalled_") and m.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v.replace(",", "")), m[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        if stalls:
            print("# stall reasons (warps stalled per issued instruction)")
            for v, name in sorted(stalls, reverse=True)[:12]:
                print(f"  stall_{name:40s} {v:8.3f}")
        for m, v in sorted(vals.items()):
            if "mem_local" in m and (m.endswith(".sum") or m.endswith(".pct")):
                print(f"{m:70s} {v:>16s} {units.get(m, '')}")
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    print("\n## details (sections)")
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ix = [hdr.index(c) for c in ("Section Name", "Metric Name", "Metric Unit", "Metric Value")]
    idc = hdr.index("ID") if "ID" in hdr else None
    ids = sorted({r[idc] for r in rows[1:] if idc is not None and len(r) > idc}, key=int)
    want = ids[best] if ids and best < len(ids) else None
    for r in rows[1:]:
        if want is not None and r[idc] != want:
            continue
        if len(r) > ix[3] and r[ix[1]]:
            sec, name, unit, val = (r[i] for i in ix)
            if sec in ("Warp State Statistics", "Scheduler Statistics", "Occupancy",
                       "Memory Workload Analysis", "GPU Speed Of Light Throughput",
                       "Compute Workload Analysis", "Launch Statistics"):
                print(f"{sec:32s} {name:45s} {val:>16s} {unit}")


def traffic(rep):
    """Mean dram bytes (read + write) per launch over every launch in the report."""
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per, ms = [], []
    name = ""
    for vals, units in _raw(rep):
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(vals[m].replace(",", "")) * scale[units[m]]
        per.append(b)
        name = vals.get("Kernel Name", "")[:80]
    print(json.dumps({"kernel": name, "dram_bytes_per_launch": sum(per) / len(per),
                      "launches": len(per), "min": min(per), "max": max(per),
                      "source": rep}))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](sys.argv[2])
