"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel count, total, share."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    n = d["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[:70]
    v = float(d["Metric Value"])
    if d.get("Metric Unit") == "usecond":
        v *= 1e3
    agg.setdefault(n, [0, 0.0])
    agg[n][0] += 1
    agg[n][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':70s} {'n':>4s} {'total ms':>10s} {'ms/launch':>10s} {'share':>6s}")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:70s} {c:4d} {v / 1e6:10.3f} {v / 1e6 / c:10.4f} {100 * v / tot:5.1f}%")
