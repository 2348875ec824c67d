"""Single fused-gate HBM passes (n, k) for ncu captures."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2111_02396_b200 import qtraj  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--k", type=int, default=4)
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
ctx = qtraj.Context(0)
state = torch.zeros(1 << a.n, dtype=torch.complex64, device="cuda")
state[0] = 1
rng = np.random.default_rng(1)
U = workloads.haar_unitary(rng, 2 ** a.k)
ms = ctx.apply_gate(state, list(range(a.n - a.k, a.n)), U, repeats=a.reps)
print(f"n={a.n} k={a.k} ms={ms:.3f} GB/s={2 ** (a.n + 4) / ms / 1e6:.0f}")
