"""Per-launch table from an ncu report (dev aid): python tools/ncu_table.py X.ncu-rep"""
import csv
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
     "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__inst_executed_pipe_tensor_op_dmma.sum"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--print-units", "base",
                      "--metrics", ",".join(M)], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
idx = {k: i for i, k in enumerate(h)}
print(f"{'kernel':48s} {'us':>9s} {'rd MB':>9s} {'wr MB':>9s} {'fp64%':>6s} {'grid':>6s} {'mem%':>6s}")
for r in rows[2:]:
    nm = r[idx["Kernel Name"]].replace("rl::(anonymous namespace)::", "").replace("void ", "")[:48]

    def g(k):
        try:
            return float(r[idx[k]].replace(",", ""))
        except (KeyError, ValueError):
            return float("nan")
    print(f"{nm:48s} {g(M[0]) / 1e3:9.1f} {g(M[1]) / 1e6:9.1f} {g(M[2]) / 1e6:9.1f} {g(M[3]):6.1f} "
          f"{g(M[4]):6.0f} {g(M[5]):6.1f}")
