"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[start]
# a multi-kernel report repeats the header per kernel: keep the last kernel's rows
blocks, cur = [], []
for r in rows[start + 1:]:
    if r and r[0] == "Address":
        blocks.append(cur)
        cur = []
    elif len(r) == len(hdr):
        cur.append(dict(zip(hdr, r)))
blocks.append(cur)
data = blocks[int(sys.argv[3])] if len(sys.argv) > 3 else max(blocks, key=len)
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(d[key] or 0) for d in data)
byop = collections.Counter()
for d in data:
    op = d["Source"].split()[0] if d["Source"].split() else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    byop[op.split(".")[0]] += float(d[key] or 0)
print("samples", tot)
for op, v in byop.most_common(15):
    print(f"  {op:12s} {v / tot:6.3f}")
top = sorted(data, key=lambda d: -float(d[key] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for d in top:
    print(f"{float(d[key]) / tot:6.3f} {d['Address']:>6s} {d['Source'][:90]}")
