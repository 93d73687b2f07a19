"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr, data = rows[hi], rows[hi + 1:]
ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = {}
for r in data:
    per.setdefault((int(r[ii]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
tot = 0.0
for (i, k), m in sorted(per.items()):
    name = k.split("(")[0].replace("(anonymous namespace)::", "")[-70:]
    t = m.get("gpu__time_duration.sum", 0.0)
    a = agg[name]
    a[0] += 1
    a[1] += t
    a[2] = max(a[2], t)
    tot += t
print(f"launches {len(per)}  total {tot/1e3:.1f} us-units/1e3 (ncu ns)")
print(f"{'count':>6} {'total':>10} {'share':>6} {'max':>9}  kernel")
for n, (c, t, mx) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{c:6d} {t/1e3:10.1f} {100*t/tot:5.1f}% {mx/1e3:9.1f}  {n}")
