"""Text summary of one ncu capture (the --page details / --page raw CSVs that
tools/ncu_pair.sh writes): speed-of-light, pipes, scheduler, occupancy and the
warp stall breakdown.  Usage: python tools/ncu_summary.py gpurun_out/ncu_<name> "<title>" > profiles/....txt"""
import csv
import sys

stem, title = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(stem + ".details.csv")))
h = rows[0]
iS, iM, iU, iV = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
print(title)
keep = ("GPU Speed Of Light", "Compute Workload", "Memory Workload", "Scheduler", "Warp State", "Launch Statistics",
        "Occupancy")
for r in rows[1:]:
    if r[iS].startswith(keep):
        print(f"{r[iS][:28]:28s} | {r[iM]:45s} {r[iV]:>14s} {r[iU]}")
raw = list(csv.reader(open(stem + ".raw.csv")))
d = dict(zip(raw[0], raw[2]))
print("\nwarp stall reasons (cycles per issued instruction):")
st = []
for k, v in d.items():
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            st.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
for v, k in sorted(st, reverse=True)[:12]:
    print(f"  {k:28s} {v:6.2f}")
print("\npipes and traffic:")
for k in ("smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "launch__registers_per_thread"):
    if k in d:
        print(f"  {k:60s} {d[k]}")
