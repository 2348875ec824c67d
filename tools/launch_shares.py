"""Per-kernel share of device time from an ncu --metrics gpu__time_duration.sum launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
t = defaultdict(float)
n = defaultdict(int)
for r in rows[hi + 1:]:
    if len(r) > iv and r[im] == "gpu__time_duration.sum":
        name = r[ik].split("(")[0]
        t[name] += float(r[iv].replace(",", ""))
        n[name] += 1
tot = sum(t.values())
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'share':>7s} {'avg_us':>10s}")
for k in sorted(t, key=lambda k: -t[k]):
    print(f"{k[:60]:60s} {n[k]:8d} {t[k]/1e3:12.1f} {t[k]/tot*100:6.1f}% {t[k]/n[k]/1e3:10.2f}")
