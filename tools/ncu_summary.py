"""Summarise one kernel of an ncu --set full report (raw page CSV) for profiles/."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u = rows[0], rows[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__cycles_elapsed.avg.per_second"]
for v in rows[2:]:
    print("kernel:", v[h.index("Kernel Name")])
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"  {k:60s} {v[i]:>22s} {u[i]}")
    rd = float(v[h.index("dram__bytes_read.sum")].replace(",", ""))
    wr = float(v[h.index("dram__bytes_write.sum")].replace(",", ""))
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
    rd *= scale[u[h.index("dram__bytes_read.sum")]]
    wr *= scale[u[h.index("dram__bytes_write.sum")]]
    print(f"  traffic (read+write) bytes per launch: {int(rd + wr)}")
    st = {}
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v[i] not in ("", "0"):
            st[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(v[i].replace(",", ""))
    tot = sum(st.values()) or 1
    print("  warp-state samples:", ", ".join(f"{k} {100*x/tot:.1f}%" for k, x in sorted(st.items(), key=lambda t: -t[1])[:8]))
