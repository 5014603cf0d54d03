"""Warp-stall samples and executed instructions aggregated per CUDA source line from an
ncu capture (needs -lineinfo + --import-source).  usage: stall_lines.py <rep> [kernel-regex] [top]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                              text=True, stderr=subprocess.DEVNULL)
fname, rows = None, []
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            rows.append((int(r[4] or 0), int(r[7] or 0), f"{fname}:{r[0]}", r[1].strip()[:90]))
        except ValueError:
            pass
tot = sum(x[0] for x in rows) or 1
toti = sum(x[1] for x in rows) or 1
for smp, ex, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * smp / tot:5.1f}% stall  {100 * ex / toti:5.1f}% inst  {loc:22s} {src}")
