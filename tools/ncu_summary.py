"""Summarize an ncu report: key throughput metrics + stall reasons + top SASS opcodes by stall samples."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
kid = sys.argv[2] if len(sys.argv) > 2 else None


def raw():
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[2:]


h, rows = raw()
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for row in rows:
    print("----")
    for k in want:
        if k in h:
            print(f"  {k:70s} {row[h.index(k)]}")
    stalls = [(k, row[i]) for i, k in enumerate(h) if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    stalls = sorted(((float(v or 0), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")) for k, v in stalls), reverse=True)[:8]
    print("  stalls/issue:", ", ".join(f"{k}={v:.2f}" for v, k in stalls))
