import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch, workloads, oracle
from paper_2111_02396_b200 import qtraj
c = workloads.random_circuit(14, depth=8, seed=3, noise="both", p=0.02, t1_ns=800.0, tphi_ns=1500.0, readout=True)
plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
ctx = qtraj.Context(0)
T=8
state = torch.zeros(T << 14, dtype=torch.complex64, device='cuda')
out = ctx.run_trajectories(plan, state, seed=5, traj_count=T, shots=1, observables=c.observables)
torch.cuda.synchronize()
ref = oracle.run_trajectories(c, seed=5, traj_count=T, shots=1, want_states=True)
psi = state.view(T,-1).cpu().numpy().astype(np.complex128); psi /= np.linalg.norm(psi,axis=1,keepdims=True)
print("kraus eq", (out['kraus']==ref['kraus']).all(), "bits eq", (out['bits']==ref['bits']).all(), "rel", (np.linalg.norm(psi-ref['states'],axis=1)).max())
