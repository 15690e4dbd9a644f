"""Aggregate warp-stall samples of an .ncu-rep by CUDA source line.
usage: ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, agg, src, tot = None, collections.Counter(), {}, 0.0
hdr = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or not r[0].isdigit():
        continue
    try:
        v = float(r[4] or 0)
    except ValueError:
        continue
    key = (fname, int(r[0]))
    agg[key] += v
    src.setdefault(key, r[1])
    tot += v
print(f"total stall samples {tot:.0f}")
for (f, ln), v in agg.most_common(top):
    print(f"{v / tot:6.3f} {f}:{ln:<5d} {src[(f, ln)].strip()[:90]}")
