"""Parity of an experiment build (library file name as argv[1]) against the oracle on
tensor-core (f16-run) trajectories: random noisy circuits n = 12, 14, 16 and C2."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import workloads  # noqa: E402
from paper_2111_02396_b200 import qtraj  # noqa: E402

qtraj.LIB_PATH = qtraj.LIB_PATH.replace("libqtraj.so", sys.argv[1])
ctx = qtraj.Context(0)
worst = 0.0
cases = [(workloads.random_circuit(n, depth=8, seed=n, noise="both", p=0.03, t1_ns=600.0, tphi_ns=900.0,
                                   readout=True), 8) for n in (12, 14, 16)]
cases.append((workloads.sycamore_grid_qcs(config=2), 2))
for c, T in cases:
    ref = oracle.run_trajectories(c, seed=5, traj_count=T, shots=2, want_states=True)
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
    st = torch.zeros(T << c.n_qubits, dtype=torch.complex64, device="cuda")
    out = ctx.run_trajectories(plan, st, seed=5, traj_count=T, shots=2, observables=c.observables)
    torch.cuda.synchronize()
    psi = st.view(T, -1).cpu().numpy().astype(np.complex128)
    psi /= np.linalg.norm(psi, axis=1, keepdims=True)
    rel = np.linalg.norm(psi - ref["states"], axis=1) / np.linalg.norm(ref["states"], axis=1)
    ok = (out["kraus"] == ref["kraus"]).all() and (out["bits"] == ref["bits"]).all()
    worst = max(worst, rel.max())
    print(sys.argv[1], "n", c.n_qubits, "records identical" if ok else "RECORDS DIFFER", "max rel-L2 %.2e" % rel.max(),
          "obs err %.1e" % np.abs(out["obs"] - ref["obs"]).max(), flush=True)
print(sys.argv[1], "PASS" if worst < 1e-5 else "FAIL", flush=True)
