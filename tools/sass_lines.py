"""Per-source-line totals of an ncu --set full report (SASS page joined with the
line table of the kernel's cubin): warp-instructions, stall samples, shared
wavefronts.  usage: python tools/sass_lines.py REPORT.ncu-rep OBJ.o KERNEL_SUBSTR [top]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                                                   "sass"], capture_output=True, text=True).stdout)))
hdr = rows[1]
ia, ist, iie, iwf = (hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"),
                     hdr.index("Instructions Executed"), hdr.index("L1 Wavefronts Shared"))
recs = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    try:
        recs.append((int(r[ia], 16), float(r[ist] or 0), float(r[iie] or 0), float(r[iwf] or 0), r[1].strip()))
    except ValueError:
        pass
base = recs[0][0]
# line table: nvdisasm -g -c on the cubin extracted from the object
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", "-fun", "", os.path.join(td, cub)], capture_output=True,
                         text=True).stdout
    if not dis:
        dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(td, cub)], capture_output=True, text=True).stdout
line_of = {}
cur_fn, cur_line, fn_ok = None, None, False
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        fn_ok = kname in m.group(1)
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur_line = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and fn_ok and cur_line:
        line_of[int(m.group(1), 16)] = cur_line
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for a, st, ie, wf, _ in recs:
    key = line_of.get(a - base, ("?", 0))
    agg[key][0] += ie
    agg[key][1] += st
    agg[key][2] += wf
tot_ie = sum(v[0] for v in agg.values())
tot_st = sum(v[1] for v in agg.values())
print(f"total warp-instr {tot_ie:.3e}  stall samples {tot_st:.0f}")
print(f"{'file:line':34s} {'instr%':>7s} {'stall%':>7s} {'smem wf':>10s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0] + ':' + str(k[1]):34s} {100 * v[0] / tot_ie:7.2f} {100 * v[1] / tot_st:7.2f} {v[2]:10.3g}")
