# Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel.
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hi]
idx = {h: i for i, h in enumerate(hdr)}
agg = collections.OrderedDict()
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[idx["Kernel Name"]].split("(")[0]
    us = float(r[idx["Metric Value"]].replace(",", "")) * scale[r[idx["Metric Unit"]]]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':64s} {'launches':>8s} {'total_us':>12s} {'share':>7s}")
for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name[:64]:64s} {n:8d} {us:12.1f} {us / tot:7.3f}")
