"""Summarise the round's ncu captures into profiles/ (run from the repo root)."""
import csv, json, os, subprocess, sys, collections
O = "gpurun_out"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct"]
def unit_scale(name, val, unit):
    v = float(val.replace(",", ""))
    if unit in ("Gbyte",): v *= 1e9
    elif unit in ("Mbyte",): v *= 1e6
    elif unit in ("Kbyte",): v *= 1e3
    elif unit == "msecond": v *= 1e3
    elif unit == "nsecond": v *= 1e-3
    return v  # bytes, or microseconds for durations
out, traffic = [], {}
for k in ["k_spmm", "k_sh_tma", "k_fft1_fwd_pers", "k_fft1_inv_pers", "k_fft2_col_pers", "k_fft2_row_unpack_pers", "k_fft2_row_pack_pers"]:
    rep = f"{O}/full_{k}.ncu-rep"
    if not os.path.exists(rep): continue
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader([l for l in txt.splitlines() if l.startswith('"')]))
    h, units, r = rows[0], rows[1], rows[2]
    d = dict(zip(h, r)); u = dict(zip(h, units))
    out.append(f"== {d['Kernel Name'][:100]}")
    for key in KEYS:
        if key in d: out.append(f"   {key:60s} {d[key]:>16s} {u.get(key, '')}")
    st = {a: float(b.replace(",", "")) for a, b in d.items() if a.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not a.endswith("_not_issued") and b.replace(",", "").replace(".", "").isdigit()}
    tot = sum(st.values()) or 1
    out.append("   stall share: " + ", ".join(f"{a[33:]} {100*b/tot:.0f}%" for a, b in sorted(st.items(), key=lambda x: -x[1])[:6]))
    rd = unit_scale("r", d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
    wr = unit_scale("w", d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
    traffic[k] = int(rd + wr)
print("\n".join(out))
json.dump({"S": traffic.get("k_spmm"), "S_H": traffic.get("k_sh_tma"), "per_kernel": traffic,
           "source": "ncu --set full --clock-control none, one launch each at 2048^2 x 1536, B=32 (scratch/profile_all.sh)"},
          open("profiles/spmm_traffic.json", "w"), indent=1)
