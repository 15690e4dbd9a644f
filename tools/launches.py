"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0]
    k = k.replace("(anonymous namespace)::", "").replace("clb::", "")
    v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[-48:]:48s} {n:8d} {v:10.1f} {v / n:9.2f} {v / tot:6.3f}")
print(f"{'total':48s} {sum(v[0] for v in agg.values()):8d} {tot:10.1f}")
