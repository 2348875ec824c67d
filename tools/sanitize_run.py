"""Small K1 workload for compute-sanitizer (memcheck / racecheck / synccheck): one
noisy 13-qubit circuit, 4 trajectories, through the per-tile tensor-core kernel
(tile 12) and the persistent TMEM kernel (tile 13), plus conventional channels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2111_02396_b200 import qtraj  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 13
tiles = [int(t) for t in sys.argv[2].split(",")] if len(sys.argv) > 2 else [12, 13]
c = workloads.random_circuit(n, depth=5, seed=3, noise="both", p=0.05, t1_ns=500.0, tphi_ns=800.0, readout=True)
ctx = qtraj.Context(0)
for tb in tiles:
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4, tile_bits=tb)
    state = torch.zeros(4 << n, dtype=torch.complex64, device="cuda")
    out = ctx.run_trajectories(plan, state, seed=9, traj_count=4, shots=2, observables=c.observables)
    torch.cuda.synchronize()
    print("tile", tb, "reductions", out["stats"]["reductions"], "ok")
