"""Summarise ncu captures and launch lists of one gpurun session into
profiles/<tag>_ncu_summary.json (committed; gpurun_out/ is scratch).

usage: python tools/ncu_summary.py <tag> [gpurun_out/<tag>]
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__block_size", "launch__grid_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.per_cycle_active",
    "smsp__warps_eligible.avg.per_cycle_active", "smsp__average_warp_latency_per_inst_issued.ratio",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__inst_executed.sum",
    "smsp__thread_inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_bytes.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{vals[i]} {units[i]}".strip()
        res.append(d)
    return res


def details(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "details", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    keep = []
    for r in csv.reader(io.StringIO(out)):
        if len(r) > 14 and r[11] in ("Scheduler Statistics", "Warp State Statistics", "Occupancy",
                                     "Compute Workload Analysis", "Launch Statistics",
                                     "Memory Workload Analysis"):
            keep.append({"section": r[11], "metric": r[12], "unit": r[13], "value": r[14]})
    return keep


def launches(path):
    rows = list(csv.DictReader(l for l in open(path) if l.startswith('"')))
    agg = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0]
        a = agg.setdefault(k, {"launches": 0, "ns": 0.0})
        a["launches"] += 1
        a["ns"] += float(r["Metric Value"].replace(",", ""))
    tot = sum(a["ns"] for a in agg.values()) or 1.0
    for a in agg.values():
        a["share"] = a["ns"] / tot
    return agg


def main():
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join("gpurun_out", tag)
    os.makedirs("profiles", exist_ok=True)
    summary = {"tag": tag}
    for f in sorted(os.listdir(src)):
        p = os.path.join(src, f)
        if f.endswith(".ncu-rep"):
            summary[f] = {"raw": raw(p), "details": details(p)}
        elif f.endswith("launches.csv"):
            summary[f] = launches(p)
        elif f.endswith(".json") or f in ("pytest_gpu.log", "smoke.log"):
            summary[f] = open(p).read()[-3000:]
    json.dump(summary, open(os.path.join("profiles", f"{tag}_ncu_summary.json"), "w"), indent=1)
    for k, v in summary.items():
        if isinstance(v, dict) and "raw" in v:
            print(k, json.dumps(v["raw"], indent=1))
        elif isinstance(v, dict):
            print(k, json.dumps(v, indent=1))


if __name__ == "__main__":
    main()
