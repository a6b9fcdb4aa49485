"""Summarise an ncu --set full report: key counters + warp-stall breakdown.
usage: python scratch/ncu_summarize.py <report.ncu-rep> [label]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
label = sys.argv[2] if len(sys.argv) > 2 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
get = {n: (u[i], v[i]) for i, n in enumerate(h)}
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__inst_executed.sum.per_cycle_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
print(f"# ncu --set full summary: {label}")
for k in keys:
    if k in get:
        print(f"{k:95s} {get[k][1]:>18s} {get[k][0]}")
st = {n[len('smsp__pcsamp_warps_issue_stalled_'):]: float(get[n][1].replace(',', '') or 0)
      for n in h if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")}
tot = sum(st.values()) or 1
print("# warp-state samples (all warps, incl. control warps parked on mbarriers)")
for k, x in sorted(st.items(), key=lambda kv: -kv[1]):
    if x > 0:
        print(f"  {k:28s} {int(x):8d} {100 * x / tot:5.1f}%")
