"""Summarise gpurun_out/ncu_*.ncu-rep (tools/ncu_kernels.sh) into profiles/r02_ncu_kernels.json:
per kernel the duration, DRAM bytes, FP64 / DMMA pipe and issue utilisation on the SMs it ran on,
occupancy, registers, local-memory (spill) traffic, shared memory and the top stall reasons."""
import csv
import glob
import json
import os
import subprocess
import sys

KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "dram_throughput_pct_of_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "fp64_pipe_active_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "dmma_pipe_active_pct": ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "registers_per_thread": ("launch__registers_per_thread", 1),
    "grid_size": ("launch__grid_size", 1),
    "block_size": ("launch__block_size", 1),
    "smem_per_block_bytes": ("launch__shared_mem_per_block", 1),
    "local_load_requests": ("l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum", 1),
    "local_store_requests": ("l1tex__t_requests_pipe_lsu_mem_local_op_st.sum", 1),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    "sm_clock_ghz": ("smsp__cycles_elapsed.avg.per_second", 1e-9),
    "warp_instructions": ("smsp__inst_executed.sum", 1),
}
STALL = "smsp__average_warps_issue_stalled_"

out = {"round": 2, "source": "tools/ncu_kernels.sh: ncu --set full --import-source on --clock-control none, one launch "
                              "per kernel on tools/prof_kernels.py workloads (cold-cache, serialised by the profiler)",
       "kernels": {}}
for rep in sorted(glob.glob("gpurun_out/ncu_*.ncu-rep")):
    name = os.path.basename(rep)[4:-8]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        continue
    h, r = rows[0], rows[2]
    val = dict(zip(h, r))

    def num(k):
        try:
            return float(val[k].replace(",", ""))
        except (KeyError, ValueError):
            return None
    e = {"kernel": val.get("Kernel Name", "?")[:160]}
    for k, (metric, sc) in KEYS.items():
        v = num(metric)
        e[k] = None if v is None else round(v * sc, 4)
    stalls = {k[len(STALL):].replace("_per_issue_active.ratio", ""): num(k) for k in h
              if k.startswith(STALL) and k.endswith("_per_issue_active.ratio") and num(k)}
    e["top_stalls_warps_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:5])
    out["kernels"][name] = e
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_ncu_kernels.json", "w"), indent=1)
print(json.dumps({k: (v["duration_us"], v["issue_active_pct"], v["fp64_pipe_active_pct"], v["dmma_pipe_active_pct"])
                  for k, v in out["kernels"].items()}, indent=1))
