for lib in libqtraj.so libqtraj_1rt.so; do
  python -c "
import sys
from paper_2111_02396_b200 import qtraj
qtraj.LIB_PATH = qtraj.LIB_PATH.replace('libqtraj.so', '$lib')
import torch, workloads, bench
c = workloads.sycamore_grid_qcs(config=2)
ctx = qtraj.Context(0)
plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
state = torch.empty(128 << 20, dtype=torch.complex64, device='cuda')
for i in range(2):
    out = ctx.run_trajectories(plan, state, seed=workloads.trajectory_seed(2), traj_count=512, batch=128, shots=1, observables=c.observables, profile=True)
print('$lib', {k: round(out['stats'][k],2) for k in ('pass_kernel_ms','device_ms')})
del state; torch.cuda.empty_cache()
s = bench.gate_pass_sweep(ctx, 30, torch.device('cuda', 0), 6554.9)
print('$lib sweep k<=4 median', s['k4_median_frac'])
"
done
