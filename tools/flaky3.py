import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle, workloads
from paper_2111_02396_b200 import qtraj
ctx = qtraj.Context(0)
n = 23
c = workloads.random_circuit(n, depth=3, seed=31, max_arity=2, noise="depol", p=0.02)
for T, batch in [(4, 4), (1, 4), (4, 4)]:
    ref = oracle.run_trajectories(c, seed=3, traj_count=T, shots=4, want_states=False)
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
    for rep in range(6):
        state = torch.zeros(batch << n, dtype=torch.complex64, device="cuda")
        out = ctx.run_trajectories(plan, state, seed=3, traj_count=T, shots=4, observables=c.observables, batch=batch)
        torch.cuda.synchronize()
        d = np.abs(out["obs"] - ref["obs"])
        print(os.environ.get("QT_HEAP_MIN_LG"), "T", T, "batch", batch, "rep", rep, "maxdiff per traj", d.max(axis=1), "bad obs t0", np.flatnonzero(d[0] > 1e-5).tolist(), flush=True)
