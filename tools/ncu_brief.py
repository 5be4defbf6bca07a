"""Key counters + top stall reasons of the first kernel in an .ncu-rep (dev aid): python tools/ncu_brief.py X.ncu-rep [per]"""
import csv
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
per = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
for v in rows[2:]:
    d = dict(zip(rows[0], v))
    print(d.get("Kernel Name", "")[:90])
    for k in ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
              "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum"]:
        print(f"  {k} = {d.get(k)}")
    ie = d.get("smsp__inst_executed.sum")
    if ie:
        print(f"  smsp__inst_executed.sum = {ie} ({float(ie) / per:.0f} per unit)")
    st = [(k, float(x)) for k, x in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
          and k.endswith("_per_issue_active.ratio") and x not in ("", "n/a")]
    for k, x in sorted(st, key=lambda z: -z[1])[:8]:
        print(f"  stall {k[34:-23]} {x}")
