"""Per-kernel mean launch times from ncu launch lists (gpu__time_duration.sum CSVs).
usage: python tools/launch_table.py <csv...>"""
import collections
import csv
import sys


def table(path):
    agg = collections.OrderedDict()
    hdr = None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        agg.setdefault(d["Kernel Name"].split("(")[0][:48], []).append(float(d["Metric Value"].replace(",", "")))
    return agg


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        for k, x in table(p).items():
            if max(x) > 20e3:
                print(f"  {k:48s} n={len(x)} mean={sum(x) / len(x) / 1e3:9.1f} us")
