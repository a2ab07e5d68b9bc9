"""profiles/r01_launches_bench_summary.txt from the launch-list CSV of scratch/profile_all.sh."""
import csv, collections, sys
src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches_bench.csv"
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = {}
for r in rows[1:]:
    d.setdefault(r[iid], {"k": r[ik]})[r[im]] = float(r[iv].replace(",", ""))
out, agg = [], collections.defaultdict(list)
for v in d.values():
    t = v["gpu__time_duration.sum"] / 1e3
    b = (v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)) / 1e6
    out.append(f"{t:10.1f} us {b:9.1f} MB  {v['k'][:80]}")
    agg[v["k"][:80]].append(t)
s = ["# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 120",
     "#   python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e   (cold-cache, serialised launches; first 120)",
     "# per-launch: duration, DRAM bytes (read+write), kernel", *out, "", "# median duration per kernel (us), count"]
for k, v in sorted(agg.items(), key=lambda x: -sorted(x[1])[len(x[1]) // 2]):
    s.append(f"{sorted(v)[len(v) // 2]:10.1f} x{len(v):3d}  {k}")
open("profiles/r01_launches_bench_summary.txt", "w").write("\n".join(s) + "\n")
