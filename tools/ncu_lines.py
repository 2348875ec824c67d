"""Per-source-line instruction / stall-sample summary of an ncu report
(ncu -i REP --page source --csv --print-source cuda)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows, fname = [], None
lines = out.splitlines()
i = 0
while i < len(lines):
    if lines[i].startswith('"File Name"'):
        fname = lines[i].split(",")[1].strip('"').split("/")[-1]
        hdr = next(csv.reader([lines[i + 1]]))
        j = i + 2
        while j < len(lines) and not lines[j].startswith('"File Name"') and not lines[j].startswith('"Kernel Name"'):
            r = next(csv.reader([lines[j]]))
            if len(r) == len(hdr):
                d = dict(zip(hdr, r))
                try:
                    ie = float(d.get("Instructions Executed", "0") or 0)
                    ss = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
                except ValueError:
                    ie = ss = 0
                if ie or ss:
                    rows.append((fname, int(d["Line No"]), ie, ss, d["Source"].strip()[:70]))
            j += 1
        i = j
    else:
        i += 1
ti = sum(r[2] for r in rows) or 1
ts = sum(r[3] for r in rows) or 1
print(f"total warp-instr {ti:.3e}  stall samples {ts:.0f}")
for r in sorted(rows, key=lambda r: -r[3])[:top]:
    print(f"{r[0]:>22}:{r[1]:<4} instr {100*r[2]/ti:5.1f}%  samples {100*r[3]/ts:5.1f}%  {r[4]}")
