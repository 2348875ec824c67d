"""Repeat the n = 23 trajectory parity case: obs / state / bits vs the oracle, several runs."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle, workloads
from paper_2111_02396_b200 import qtraj
ctx = qtraj.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 23
c = workloads.random_circuit(n, depth=3, seed=31, max_arity=2, noise="depol", p=0.02)
print("observables", c.observables[:6], len(c.observables), flush=True)
ref = oracle.run_trajectories(c, seed=3, traj_count=2, shots=4, want_states=True)
plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 8):
    state = torch.zeros(2 << n, dtype=torch.complex64, device="cuda")
    out = ctx.run_trajectories(plan, state, seed=3, traj_count=2, shots=4, observables=c.observables)
    torch.cuda.synchronize()
    psi = state.view(2, -1).cpu().numpy().astype(np.complex128)
    psi /= np.linalg.norm(psi, axis=1, keepdims=True)
    rel = np.linalg.norm(psi - ref["states"], axis=1) / np.linalg.norm(ref["states"], axis=1)
    dobs = np.abs(out["obs"] - ref["obs"]).max(axis=1)
    bad = [int(i) for i in np.flatnonzero(np.abs(out["obs"][0] - ref["obs"][0]) > 1e-4)]
    print(rep, "state rel", rel, "obs maxdiff", dobs, "bits eq", bool((out["bits"] == ref["bits"]).all()),
          "kraus eq", bool((out["kraus"] == ref["kraus"]).all()), "bad obs idx t0", bad[:10], flush=True)
