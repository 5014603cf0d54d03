"""Top SASS instructions by one stall reason (default stall_short_sb), with the
instruction that produced the awaited register when it is nearby.
usage: sass_stalls.py <rep> [reason] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
reason = sys.argv[2] if len(sys.argv) > 2 else "stall_short_sb"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                              text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = hdr.index(reason)
isrc = hdr.index("Source")
iex = hdr.index("Instructions Executed")
body = [r for r in rows[2:] if len(r) > ix]
tot = sum(int(r[ix] or 0) for r in body) or 1
alls = sum(int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0) for r in body) or 1
print(f"{reason}: {100 * tot / alls:.1f}% of all samples")
order = sorted(range(len(body)), key=lambda i: -int(body[i][ix] or 0))
for i in order[:top]:
    r = body[i]
    ctx = " | ".join(body[j][isrc].strip()[:34] for j in range(max(0, i - 3), i))
    print(f"{100 * int(r[ix] or 0) / tot:5.1f}% {i:5d} {r[isrc].strip()[:48]:48s} <- {ctx}")
