"""Per-gate phase timing of the f16 tensor-core chain from a -DQT_TIMING build
(libqtraj_timing.so): clock64 sums over sampled CTAs, warp 0 and warp 2."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_02396_b200 import qtraj  # noqa: E402

qtraj.LIB_PATH = qtraj.LIB_PATH.replace("libqtraj.so", "libqtraj_timing.so")
import runpy  # noqa: E402

sys.argv = [sys.argv[1]] + sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
buf = (ctypes.c_ulonglong * 16)()
qtraj.lib().qt_timing_read(buf)
n = max(buf[15], 1)
m = max(buf[14], 1)
print(f"CTA passes sampled: {buf[14]}  (cycles per CTA, thread 0)")
for i, nm in enumerate(["prologue (desc, hoff, TMEM)", "tile load (issue + wait)", "gates", "epilogues",
                        "store issue"]):
    print(f"  {nm:30s} {buf[8 + i] / m:8.0f}")
names = ["wait MMA group 0", "readout group 0", "W wait + fence + barrier", "issue + wait MMA group 1",
         "readout group 1", "W(g+2) + fence + barrier"]
print(f"chained gates sampled: {buf[15]}  (cycles per gate, warp 0)")
for i, nm in enumerate(names):
    print(f"  {nm:30s} {buf[i] / n:8.0f}")
