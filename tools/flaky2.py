import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle, workloads
from paper_2111_02396_b200 import qtraj
ctx = qtraj.Context(0)
for n, T, batch, depth in [(23, 1, 1, 3), (23, 2, 2, 3), (24, 2, 2, 3), (23, 4, 4, 3), (23, 2, 2, 0)]:
    c = workloads.random_circuit(n, depth=depth, seed=31, max_arity=2, noise="depol", p=0.02) if depth else None
    if c is None:
        c = workloads.random_circuit(n, depth=1, seed=31, max_arity=1, noise="none")
    ref = oracle.run_trajectories(c, seed=3, traj_count=T, shots=4, want_states=False)
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
    fails = 0
    worst = np.zeros(T)
    for rep in range(6):
        state = torch.zeros(batch << n, dtype=torch.complex64, device="cuda")
        out = ctx.run_trajectories(plan, state, seed=3, traj_count=T, shots=4, observables=c.observables, batch=batch)
        torch.cuda.synchronize()
        d = np.abs(out["obs"] - ref["obs"]).max(axis=1)
        worst = np.maximum(worst, d)
        fails += int((d > 1e-4).any())
    info = plan.info(3, 0)
    print("n", n, "T", T, "batch", batch, "depth", depth, "fails", fails, "/6 worst per traj", worst, "passes", info["passes"], flush=True)
