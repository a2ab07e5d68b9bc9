"""Per-kernel median durations (us) and counts of a TV launch-list CSV
(ncu --metrics gpu__time_duration.sum --csv): python scratch/tv_launches.py CSV."""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
agg = collections.defaultdict(list)
tot = 0.0
for r in rows[1:]:
    if r[im] == "gpu__time_duration.sum":
        t = float(r[iv].replace(",", "")) / 1e3
        agg[r[ik][:90]].append(t)
        tot += t
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{sorted(v)[len(v) // 2]:9.1f} us x{len(v):3d} sum {sum(v) / 1e3:7.2f} ms  {k}")
print(f"total {tot / 1e3:.2f} ms")
