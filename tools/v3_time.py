"""Timing of v3 (tile_bits 11) vs v2 (13) on a 20-qubit depolarizing circuit (no conventional channels)."""
import os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads
from paper_2111_02396_b200 import qtraj
if len(sys.argv) > 1:
    qtraj.LIB_PATH = qtraj.LIB_PATH.replace("libqtraj.so", sys.argv[1])
ctx = qtraj.Context(0)
c = workloads.random_circuit(20, depth=14, seed=9, max_arity=2, noise="depol", p=0.005)
for tb in (11, 13):
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4, tile_bits=tb)
    state = torch.empty(384 << 20, dtype=torch.complex64, device="cuda")
    for _ in range(2):
        out = ctx.run_trajectories(plan, state, seed=5, traj_count=1536, batch=384, shots=1, profile=True)
        torch.cuda.synchronize()
    st = out["stats"]
    print(sys.argv[1:] or ["libqtraj.so"], "tile_bits", tb, "pass_kernel_ms %.1f passes/traj %.2f gates/traj %.2f" % (
        st["pass_kernel_ms"], st["passes"] / 1536, st["fused_gates"] / 1536), flush=True)
    del state
