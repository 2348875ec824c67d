"""One batch of a G-gate single-pass chain (n = 20, random 4-qubit Haar gates on
12 tile qubits, 128 trajectories) for ncu captures of the multi-gate K1 path."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from workloads import Circuit, Gate  # noqa: E402
from paper_2111_02396_b200 import qtraj  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gates", type=int, default=16)
ap.add_argument("--batch", type=int, default=128)
a = ap.parse_args()
rng = np.random.default_rng(5)
c = Circuit(n_qubits=20, moments=[])
prev = None
for g in range(a.gates):
    while True:
        qs = sorted(rng.choice(12, 4, replace=False).tolist())
        if qs != prev:
            break
    prev = qs
    c.moments.append([Gate(tuple(int(q) for q in qs), workloads.haar_unitary(rng, 16))])
ctx = qtraj.Context(0)
plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
state = torch.empty(a.batch << 20, dtype=torch.complex64, device="cuda")
out = ctx.run_trajectories(plan, state, seed=1, traj_count=a.batch, batch=a.batch, shots=1, profile=True)
torch.cuda.synchronize()
print({k: out["stats"][k] for k in ("passes", "fused_gates", "pass_kernel_ms")})
