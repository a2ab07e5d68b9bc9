"""Aggregate stall reasons and list the hottest SASS lines of an ncu --page source --csv export."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
for r in data:
    for i in stall_cols:
        try: tot[hdr[i]] += float(r[i])
        except: pass
s = sum(tot.values())
print("stall share:")
for k, v in tot.most_common(10): print(f"  {k:25s} {100*v/s:5.1f}%")
si = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
top = sorted(data, key=lambda r: -float(r[si] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]
print("hottest instructions:")
for r in top:
    print(f"  {r[si]:>6s}  {r[src].strip()[:90]}")
