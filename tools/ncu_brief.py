"""Headline metrics and stall reasons (per issued instruction) of the kernel in an ncu report.
usage: python tools/ncu_brief.py <report.ncu-rep>"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u, v = r[0], r[1], r[-1]
    d = dict(zip(h, v))
    un = dict(zip(h, u))
    print(d.get("Kernel Name"))
    for k in KEYS:
        if k in d:
            print(f"  {k} = {d[k]} {un.get(k, '')}")
    st = {k.split("stalled_")[1].split("_per_issue")[0]: float(x) for k, x in d.items()
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    print("  stalls per issue:", {k: round(x, 2) for k, x in sorted(st.items(), key=lambda kv: -kv[1]) if x > 0.01},
          "total", round(sum(st.values()), 2))


if __name__ == "__main__":
    main(sys.argv[1])
