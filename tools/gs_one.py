import os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads
from paper_2111_02396_b200 import qtraj
qtraj.LIB_PATH = qtraj.LIB_PATH.replace("libqtraj.so", sys.argv[1])
n = int(sys.argv[2]); qs = [int(x) for x in sys.argv[3].split(",")]
ctx = qtraj.Context(0)
rng = np.random.default_rng(1)
state = torch.zeros(1 << n, dtype=torch.complex64, device="cuda"); state[0] = 1.0
U = workloads.haar_unitary(rng, 2 ** len(qs))
ms = ctx.apply_gate(state, qs, U, repeats=3)
torch.cuda.synchronize()
print(n, qs, "ms", ms, flush=True)
