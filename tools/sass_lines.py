"""Per-SASS-instruction executed warp-instructions per warp-decision from an ncu capture
(source page), with the kernel-relative address: the input for range accounting.
usage: python tools/sass_lines.py <report.ncu-rep> <decisions in the captured launch> [> out.txt]"""
import csv
import io
import subprocess
import sys

rep, dec = sys.argv[1], float(sys.argv[2])
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                              text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
iA, iS, iE = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
iT = hdr.index("Thread Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
base = None
wr = dec / 32
for r in data:
    if not r[iS].strip():
        continue
    a = int(r[iA], 16)
    base = a if base is None else base
    e, t, w = int(r[iE] or 0), int(r[iT] or 0), int(r[iW] or 0)
    print(f"{a - base:06x} {e / wr:8.3f} {t / max(1, e):5.1f} {w:7d}  {r[iS].strip()}")
