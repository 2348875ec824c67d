"""Phase timing of the persistent v2 K1 (-DQT_V2_TIMING build, libqtraj_v2t.so):
clock64 sums of the warpgroup leaders of CTA 7, per item.
usage: python tools/v2_timing.py SCRIPT [args]   (runs SCRIPT with the timing library)"""
import ctypes
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_02396_b200 import qtraj  # noqa: E402

qtraj.LIB_PATH = qtraj.LIB_PATH.replace("libqtraj.so", "libqtraj_v2t.so")
sys.argv = [sys.argv[1]] + sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
buf = (ctypes.c_ulonglong * 32)()
qtraj.lib().qt_v2_timing_read(buf)
names = ["tile full wait", "gather", "MMA complete wait", "write back",
         "observables epilogue", "stores + end barrier", "next loads", "MMA issue (after W)", "L/X transition",
         "rho epilogue", "final blocksum epilogue"]
names += [""] * 5 + ["CUDA-core gates (device-chosen operators)", "", "before the observables epilogue", "",
                      "item start barrier", "first W copies issued", "W operand wait (issuer)"]
tot = sum(buf[i] for i in range(11)) + buf[16] + buf[18] + buf[20] + buf[21] + buf[22]
items = max(buf[11], 1)
for i, nm in enumerate(names):
    if not nm:
        continue
    print(f"  {nm:50s} {buf[i]:14d} cyc  {100.0 * buf[i] / max(tot, 1):5.1f}%  {buf[i] / items:9.0f} cyc/item")
print(f"  CUDA-core gates {buf[17]}  observable items {buf[19]}")
print(f"  items {buf[11]}  tensor-core gates {buf[12]}  gathers {buf[13]}  rho items {buf[14]}  final items {buf[15]}")
print(f"  per item: {tot / items:.0f} cyc; per gate (MMA + transition phases): "
      f"{(buf[2] + buf[7] + buf[8]) / max(buf[12], 1):.0f} cyc; per rho item {buf[9] / max(buf[14], 1):.0f} cyc; "
      f"per gather {buf[1] / max(buf[13], 1):.0f} cyc")
