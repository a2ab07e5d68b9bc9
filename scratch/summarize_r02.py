"""Summarise the round-2 ncu captures (scratch/profile_r02.sh) into profiles/."""
import csv, glob, os, subprocess, collections
O = "gpurun_out"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"]
out = ["# ncu --set full --clock-control none, one launch each, 2048^2 x 1536, 64 slices (B = 32)",
       "# (scratch/profile_r02.sh; cold-cache, serialised: compare shares, not absolute times)"]
for rep in sorted(glob.glob(f"{O}/r02_full_*.ncu-rep")):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader([l for l in txt.splitlines() if l.startswith('"')]))
    if len(rows) < 3:
        continue
    h, units, r = rows[0], rows[1], rows[2]
    d = dict(zip(h, r)); u = dict(zip(h, units))
    out.append(f"== {d['Kernel Name'][:110]}")
    for key in KEYS:
        if key in d:
            out.append(f"   {key:66s} {d[key]:>18s} {u.get(key, '')}")
    st = {a: float(b.replace(",", "")) for a, b in d.items() if a.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not a.endswith("_not_issued") and b.replace(",", "").replace(".", "").isdigit()}
    tot = sum(st.values()) or 1
    out.append("   stall share: " + ", ".join(f"{a[33:]} {100*b/tot:.0f}%" for a, b in
                                             sorted(st.items(), key=lambda x: -x[1])[:6]))
dst = "profiles/r02_ncu_full_summary.txt" if os.path.isdir("profiles") and not os.environ.get("ON_BOX") else \
    f"{O}/r02_ncu_full_summary.txt"
open(dst, "w").write("\n".join(out) + "\n")
print("\n".join(out))
