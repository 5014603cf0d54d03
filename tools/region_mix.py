"""Stall samples and executed warp-instructions per source region (line ranges of
kernels.cuh / contract.cuh) from an ncu capture.  usage: region_mix.py <rep>"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                              text=True, stderr=subprocess.DEVNULL)
fname, rows = None, []
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            rows.append((fname, int(r[0]), int(r[4] or 0), int(r[7] or 0), r[1].strip()[:70]))
        except ValueError:
            pass
src = open("paper_2208_06102_b200/csrc/kernels.cuh").read().splitlines()


def region(f, ln):
    if f in ("contract.cuh", "certify.cuh"):
        s = open("paper_2208_06102_b200/csrc/" + f).read().splitlines()
        # name the enclosing function
        for i in range(ln - 1, -1, -1):
            t = s[i].strip()
            if t.startswith("__device__") or t.startswith("__global__"):
                return f.split(".")[0] + ":" + t.split("(")[0].split()[-1]
        return f + ":?"
    if f not in ("kernels.cuh", "thompson.cuh"):
        return f
    lines = src if f == "kernels.cuh" else open("paper_2208_06102_b200/csrc/thompson.cuh").read().splitlines()
    for i in range(ln - 1, -1, -1):
        t = lines[i].strip()
        if t.startswith("// ----------------") or t.startswith("__device__") or t.startswith("__global__") \
                or t.startswith("auto ") or "// REGION" in t:
            return f.split(".")[0] + ":" + t[:60]
    return f + ":?"


agg = {}
for f, ln, smp, ex, _ in rows:
    k = region(f, ln)
    a = agg.setdefault(k, [0, 0])
    a[0] += smp
    a[1] += ex
ts = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
for k, (smp, ex) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{100 * ex / ti:5.1f}% inst {100 * smp / ti * ti / ts:5.1f}% stall  {k}")
