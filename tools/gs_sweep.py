import os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads
from paper_2111_02396_b200 import qtraj
lib = sys.argv[1]
qtraj.LIB_PATH = qtraj.LIB_PATH.replace("libqtraj.so", lib)
ctx = qtraj.Context(0)
rng = np.random.default_rng(1)
for n in [int(x) for x in sys.argv[2].split(",")]:
    state = torch.zeros(1 << n, dtype=torch.complex64, device="cuda")
    state[0] = 1.0
    for k in range(1, 7):
        for name, qs in (("low", list(range(k))), ("high", list(range(n - k, n))),
                         ("mixed", sorted(rng.choice(n, k, replace=False).tolist()))):
            U = workloads.haar_unitary(rng, 2 ** k)
            t0 = time.time()
            ms = ctx.apply_gate(state, qs, U, repeats=int(sys.argv[3]) if len(sys.argv) > 3 else 3)
            gbs = 2.0 ** (n + 4) / (ms / 1e3) / 1e9
            print(n, k, name, qs, "ms %.3f" % ms, "GB/s %.0f frac %.3f" % (gbs, gbs / 6536.4), "wall %.2f" % (time.time() - t0), flush=True)
    del state
    torch.cuda.empty_cache()
