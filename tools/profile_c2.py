"""Run a small C2 batch for ncu captures (one batch of `--traj` trajectories)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2111_02396_b200 import qtraj  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--traj", type=int, default=128)
ap.add_argument("--batch", type=int, default=128)
ap.add_argument("--fuse", type=int, default=4)
ap.add_argument("--one-gate", action="store_true")
a = ap.parse_args()
c = workloads.sycamore_grid_qcs(config=2)
ctx = qtraj.Context(0)
plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=a.fuse, one_gate_per_pass=a.one_gate)
state = torch.empty(a.batch << 20, dtype=torch.complex64, device="cuda")
out = ctx.run_trajectories(plan, state, seed=workloads.trajectory_seed(2), traj_count=a.traj, batch=a.batch,
                           shots=1, observables=c.observables, profile=True)
torch.cuda.synchronize()
s = out["stats"]
print({k: s[k] for k in ("passes", "fused_gates", "reductions", "launches", "plan_ms", "device_ms", "pass_kernel_ms")})
