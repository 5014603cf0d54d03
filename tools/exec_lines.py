"""Executed warp-instructions per warp-decision by CUDA source line, from an ncu capture with
imported source (the companion of ncu_regions.py, which ranks stall samples).
usage: python tools/exec_lines.py <report.ncu-rep> <decisions in the captured launch> [top]"""
import collections
import sys

from ncu_regions import rows


def main(rep, dec, top=40):
    cur, hdr = None, None
    agg, src = collections.Counter(), {}
    for x in rows(rep):
        if not x or x[0] in ("Function Name", ""):
            continue
        if x[0] == "File Path":
            cur = x[1].split("/")[-1]
            continue
        if x[0] == "Line No":
            hdr = {k: i for i, k in enumerate(x)}
            continue
        try:
            e = int(x[hdr["Instructions Executed"]] or 0)
        except (ValueError, KeyError, TypeError):
            continue
        key = (cur, int(x[0]))
        src[key] = x[1].strip()
        agg[key] += e
    wr = dec / 32
    print(f"total {sum(agg.values()) / wr:.1f} warp-instructions per warp-decision")
    for k, v in agg.most_common(top):
        print(f"{v / wr:7.1f}  {k[0][:12]}:{k[1]:<5d} {src.get(k, '')[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 40)
