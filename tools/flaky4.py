import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle, workloads
from paper_2111_02396_b200 import qtraj
if len(sys.argv) > 1:
    qtraj.LIB_PATH = qtraj.LIB_PATH.replace("libqtraj.so", sys.argv[1])
ctx = qtraj.Context(0)
n, T = 23, 4
c = workloads.random_circuit(n, depth=3, seed=31, max_arity=2, noise="depol", p=0.02)
nobs = len(c.observables)
plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
print("pass info", plan.info(3, 0))
os.environ["QT_DUMP_PARTIALS"] = "/tmp/partials.bin"
for rep in range(8):
    state = torch.zeros(T << n, dtype=torch.complex64, device="cuda")
    out = ctx.run_trajectories(plan, state, seed=3, traj_count=T, shots=4, observables=c.observables, batch=T)
    torch.cuda.synchronize()
    raw = np.fromfile("/tmp/partials.bin", dtype=np.float64)
    nt = 1 << (n - 13)
    bs = raw[:T * nt].reshape(T, nt)
    op = raw[T * nt:].reshape(T, nt, nobs)
    psi = state.view(T, -1).cpu().numpy()
    p2 = (np.abs(psi.astype(np.complex128)) ** 2).reshape(T, nt, 8192)
    bs_ref = p2.sum(axis=2)
    idx = np.arange(8192)
    bad_bs = [(s, t) for s in range(T) for t in range(nt) if abs(bs[s, t] - bs_ref[s, t]) > 1e-6 * abs(bs_ref[s, t]) + 1e-12]
    zref = np.stack([(p2 * np.where((idx >> q) & 1, -1, 1)).sum(axis=2) for q in range(8)], axis=2)  # Z_0..Z_7
    bad_op = [(s, t) for s in range(T) for t in range(nt) if np.abs(op[s, t, :8] - zref[s, t]).max() > 1e-6 * bs_ref[s, t] + 1e-12]
    print(rep, "bad blocksum tiles", bad_bs[:12], len(bad_bs), "bad obs tiles", bad_op[:12], len(bad_op), flush=True)
    if bad_op:
        s_, t_ = bad_op[0]
        # which tile's data would give these partials?
        cand = [tt for tt in range(nt) if abs(bs_ref[s_, tt] - bs[s_, t_]) < 1e-9 * bs_ref[s_, tt]]
        print("   tile", (s_, t_), "bs got", bs[s_, t_], "ref", bs_ref[s_, t_], "matching tiles by blocksum", cand[:5], flush=True)
