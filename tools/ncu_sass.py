"""Per-opcode instruction / stall-sample summary of an ncu report's SASS page."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
hdr = next(csv.reader([out[1]]))
ops = collections.defaultdict(lambda: [0.0, 0.0])
seq = []
for line in out[2:]:
    r = next(csv.reader([line]))
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    src = d["Source"].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ie = float(d["Instructions Executed"] or 0)
    ss = float(d["Warp Stall Sampling (All Samples)"] or 0)
    ops[op][0] += ie
    ops[op][1] += ss
    seq.append((d["Address"], ie, ss, src))
ti = sum(v[0] for v in ops.values())
ts = sum(v[1] for v in ops.values())
print(f"total warp-instr {ti:.4e}  samples {ts:.0f}")
for op, (ie, ss) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"{op:>10} instr {100*ie/ti:5.1f}%  samples {100*ss/ts:5.1f}%")
if len(sys.argv) > 2:
    print("--- hottest instructions by samples")
    for a, ie, ss, src in sorted(seq, key=lambda s: -s[2])[:int(sys.argv[2])]:
        print(f"{a[-5:]} {ie:10.0f} {100*ss/ts:5.1f}%  {src[:80]}")
