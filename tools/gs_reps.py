"""Experiment: several applications of one gate per tile in the streaming kernel
(QT_GS_REPS), i.e. the cost of multi-gate passes in its TMA / 4-warpgroup pipeline.
Parity against the oracle applying the gate reps times, then the n = 30 pass time."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle, workloads
from paper_2111_02396_b200 import qtraj
ctx = qtraj.Context(0)
rng = np.random.default_rng(2)
for reps in (1, 2, 4, 8):
    os.environ["QT_GS_REPS"] = str(reps)
    n, qs = 17, [2, 7, 11, 15]
    U = workloads.haar_unitary(rng, 16)
    psi = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n); psi /= np.linalg.norm(psi)
    ref = psi.copy()
    for _ in range(reps):
        ref = oracle.apply_gate(ref, qs, U)
    d = torch.from_numpy(psi.astype(np.complex64)).cuda()
    ctx.apply_gate(d, qs, U)
    got = d.cpu().numpy().astype(np.complex128)
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    line = [reps, "rel", float(rel)]
    for k, q in ((4, [0, 1, 2, 3]), (4, [26, 27, 28, 29]), (4, [3, 9, 17, 25]), (5, [2, 6, 16, 17, 29]), (6, [24, 25, 26, 27, 28, 29])):
        n = 30
        st = torch.zeros(1 << n, dtype=torch.complex64, device="cuda"); st[0] = 1
        ms = ctx.apply_gate(st, q, workloads.haar_unitary(rng, 2 ** k), repeats=6)
        line += [k, q[0], "ms %.3f frac %.3f" % (ms, 2 ** 34 / (ms / 1e3) / 6536.4e9)]
        del st
    print(*line, flush=True)
