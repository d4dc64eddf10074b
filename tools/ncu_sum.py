"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    v = float(r[iv].replace(",", ""))
    ns = v * {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[iu], 1)
    k = r[ik].split("(")[0]
    agg[k][0] += 1
    agg[k][1] += ns
tot = sum(t for _, t in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t / 1e6:9.3f} ms {100 * t / tot:5.1f}%  {c:5d}  {k}")
print(f"{tot / 1e6:9.3f} ms total")
