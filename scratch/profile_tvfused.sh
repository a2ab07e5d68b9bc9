#!/bin/bash
# ncu --set full of the four fused TV x-pass kernels (one launch each, first outer iteration)
O=gpurun_out
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_tv_rowfft" -c 6 -o $O/r02_full_tvrow python scratch/tv_probe.py 1 > $O/tvrow_ncu.log 2>&1
python - <<'PY'
import csv, subprocess
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]
txt = subprocess.run(["ncu", "-i", "gpurun_out/r02_full_tvrow.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader([l for l in txt.splitlines() if l.startswith('"')]))
h, units = rows[0], rows[1]
out = ["# ncu --set full --clock-control none: fused TV x-pass kernels, 2048^2 x 1536, 64 slices (B = 32), first outer iteration"]
for r in rows[2:]:
    d = dict(zip(h, r)); u = dict(zip(h, units))
    out.append(f"== {d['Kernel Name'][:150]}")
    for key in KEYS:
        if key in d:
            out.append(f"   {key:66s} {d[key]:>18s} {u.get(key, '')}")
    st = {a: float(b.replace(",", "")) for a, b in d.items() if a.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not a.endswith("_not_issued") and b.replace(",", "").replace(".", "").isdigit()}
    tot = sum(st.values()) or 1
    out.append("   stall share: " + ", ".join(f"{a[33:]} {100*b/tot:.0f}%" for a, b in sorted(st.items(), key=lambda x: -x[1])[:7]))
open("gpurun_out/r02_ncu_full_summary_tvrow.txt", "w").write("\n".join(out) + "\n")
PY
rm -f $O/r02_full_tvrow.ncu-rep
