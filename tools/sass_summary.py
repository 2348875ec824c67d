"""Summary of an ncu --set full report of one K1 launch: raw-page headline metrics,
per-opcode SASS instruction / shared-wavefront / bank-conflict / stall totals, and
the hottest conflicted shared-memory instructions.
usage: python tools/sass_summary.py REPORT.ncu-rep > profiles/<round>_c2_pass_sass_summary.txt"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                                 text=True).stdout)))
h, units, v = raw[0], raw[1], raw[2]
print(f"# {rep}: raw page")
for w in ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "sm__throughput.avg.pct_of_peak_sustained_elapsed",
          "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
          "l1tex__throughput.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]:
    if w in h:
        i = h.index(w)
        print(f"  {w:70s} {v[i]} {units[i]}")
rows = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                                                   "sass"], capture_output=True, text=True).stdout)))
hh, R = rows[1], rows[2:]
ix = {k: i for i, k in enumerate(hh)}


def f(r, k):
    try:
        return float(r[ix[k]])
    except (KeyError, ValueError, IndexError):
        return 0.0


agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0])
for r in R:
    t = r[1].strip().split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    a = agg[op]
    a[0] += f(r, "Instructions Executed")
    a[1] += f(r, "L1 Wavefronts Shared")
    a[2] += f(r, "L1 Wavefronts Shared Excessive")
    a[3] += f(r, "Warp Stall Sampling (All Samples)")
print("\n# SASS per opcode: instructions, shared wavefronts, bank-conflict excess, stall samples")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][3])[:25]:
    print(f"  {k:28s} instr {a[0]:12.0f}  wavefronts {a[1]:11.0f}  excess {a[2]:11.0f}  stall-samples {a[3]:6.0f}")
print("\n# hottest conflicted shared accesses (SASS index: instruction, executed, wavefronts/instr, excess/instr)")
for i, r in enumerate(R):
    n, e = f(r, "Instructions Executed"), f(r, "L1 Wavefronts Shared Excessive")
    if n > 100000 and e / n > 1.0:
        print(f"  {i:5d} {r[1].strip()[:48]:48s} {n:9.0f} {f(r, 'L1 Wavefronts Shared') / n:5.2f} {e / n:5.2f}")
