"""Summarise an .ncu-rep (first kernel): key throughput metrics + stall reasons."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    print("kernel:", d.get("Kernel Name", "")[:100])
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
            "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "lts__t_sectors_srcunit_tex_op_read.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
            "launch__occupancy_limit_shared_mem", "launch__grid_size", "sm__cycles_active.avg"]
    for k in keys:
        if k in d:
            print(f"  {k:75s} {d[k]} {units[hdr.index(k)]}")
    st = {h[33:]: float(v.replace(",", "") or 0) for h, v in d.items()
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
    tot = sum(st.values()) or 1
    print("  stalls:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
