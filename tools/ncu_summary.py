"""One block per profiled launch of an ncu report: time, instructions, issue, pipes, DRAM,
occupancy limits and the top stall reasons (warps per issue).  Usage: ncu_summary.py rep"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
M = ["gpu__time_duration.sum", "smsp__inst_executed.sum",
     "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
     "sm__warps_active.avg.per_cycle_active",
     "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
     "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
     "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "dram__bytes_read.sum", "dram__bytes_write.sum",
     "dram__throughput.avg.pct_of_peak_sustained_elapsed",
     "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
     "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
stall = [c for c in h if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
for v in rows[2:]:
    print("==", v[h.index("Kernel Name")][:90])
    for m in M:
        if m in h:
            print(f"   {m:92s} {v[h.index(m)]}")
    st = []
    for c in stall:
        try:
            st.append((float(v[h.index(c)]), c[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
    print("   stalls:", ", ".join(f"{n}={x:.2f}" for x, n in sorted(st, reverse=True)[:7]))
