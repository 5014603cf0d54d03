"""Executed-instruction mix of the replay kernel from an ncu capture (source page, SASS):
warp-instructions per warp-recurrence by opcode, lane efficiency and stall share.
usage: python tools/sass_mix.py <report.ncu-rep> <decisions in the captured launch> [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, dec = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                              text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
iA, iE, iT = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed")
iS = hdr.index("Warp Stall Sampling (All Samples)")
op, thr, st = collections.Counter(), collections.Counter(), collections.Counter()
tot = totS = 0
for r in data:
    src = r[iA].strip()
    if not src:
        continue
    e, t, smp = int(r[iE] or 0), int(r[iT] or 0), int(r[iS] or 0)
    parts = src.split()
    o = parts[1] if parts[0].startswith("@") else parts[0]
    o = o.split(".")[0]
    op[o] += e
    thr[o] += t
    st[o] += smp
    tot += e
    totS += smp
wr = dec / 32
print(f"warp-inst per warp-recurrence {tot / wr:.1f}  (per decision {tot / dec:.2f}); "
      f"lane eff {sum(thr.values()) / max(1, tot):.2f}/32")
for o, c in op.most_common(top):
    print(f"{o:10s} {c / wr:8.1f}  thread-eff {thr[o] / max(1, c):5.1f}  stall% {100 * st[o] / max(1, totS):5.1f}")
