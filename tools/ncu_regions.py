"""Per-region warp-stall samples of the Thompson-phase kernel from an ncu report with
imported source (tools/sessions/session_ncu_src.sh).  usage: python tools/ncu_regions.py <report.ncu-rep>"""
import collections
import csv
import io
import re
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, top=40):
    def I(v):
        try:
            return int(v)
        except ValueError:
            return 0
    cur, hdr = None, None
    agg, sb, wt, lsb = (collections.Counter() for _ in range(4))
    src = {}
    for x in rows(rep):
        if not x:
            continue
        if x[0] == "File Path":
            cur = x[1].split("/")[-1]
            continue
        if x[0] == "Function Name":
            continue
        if x[0] == "Line No":
            hdr = {k: i for i, k in enumerate(x)}
            continue
        if x[0] == "":
            continue
        key = (cur, int(x[0]))
        src[key] = x[1].strip()
        agg[key] += I(x[hdr["# Samples"]])
        sb[key] += I(x[hdr["stall_short_sb"]])
        wt[key] += I(x[hdr["stall_wait"]])
        lsb[key] += I(x[hdr["stall_long_sb"]])
    tot = sum(agg.values()) or 1
    byfile = collections.Counter()
    for k, v in agg.items():
        byfile[k[0]] += v
    print("samples", tot, {k: round(100 * v / tot, 1) for k, v in byfile.most_common()})
    for k, v in agg.most_common(top):
        print(f"{100*v/tot:5.1f}% sb{100*sb[k]/tot:4.1f} w{100*wt[k]/tot:4.1f} L{100*lsb[k]/tot:4.1f} "
              f"{k[0][:12]}:{k[1]} {src.get(k, '')[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
