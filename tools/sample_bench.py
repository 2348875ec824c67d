"""qt_sample_bitstrings timing at large n (block-sum heap vs per-shot re-summation)."""
import os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_02396_b200 import qtraj
if len(sys.argv) > 1:
    qtraj.LIB_PATH = qtraj.LIB_PATH.replace("libqtraj.so", sys.argv[1])
ctx = qtraj.Context(0)
n = 32
st = torch.empty(1 << n, dtype=torch.complex64, device="cuda")
st.real.normal_(); st.imag.normal_()
for shots in (1, 64, 1024, 8192):
    ctx.sample_bitstrings(st, seed=1, traj=0, shots=shots)
    torch.cuda.synchronize(); t0 = time.time()
    ctx.sample_bitstrings(st, seed=1, traj=0, shots=shots)
    torch.cuda.synchronize()
    print(sys.argv[1:] or ["libqtraj.so"], "n", n, "shots", shots, "ms %.2f" % ((time.time() - t0) * 1e3), flush=True)
