"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv, sys, re, collections
def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    out = []
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            out.append((r[ki], float(r[vi].replace(",", "")) / 1e3))
    return out
def short(name):
    name = re.sub(r"\(.*", "", name)
    return name[:70]
if __name__ == "__main__":
    rows = load(sys.argv[1])
    for k, us in rows:
        print(f"{us:10.1f} us  {short(k)}")
    agg = collections.defaultdict(float)
    for k, us in rows: agg[short(k)] += us
    tot = sum(agg.values())
    print("---- share")
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"{v:10.1f} us {100*v/tot:5.1f}%  {k}")
