import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle, workloads
from paper_2111_02396_b200 import qtraj
if len(sys.argv) > 1:
    qtraj.LIB_PATH = qtraj.LIB_PATH.replace("libqtraj.so", sys.argv[1])
ctx = qtraj.Context(0)
rng = np.random.default_rng(1)
for n, k, qs in [(14, 4, [0, 1, 2, 3]), (16, 2, [3, 9]), (18, 6, [12, 13, 14, 15, 16, 17]), (16, 5, [0, 5, 9, 12, 15])]:
    U = workloads.haar_unitary(rng, 2 ** k)
    psi = rng.normal(size=2 ** n) + 1j * rng.normal(size=2 ** n)
    psi /= np.linalg.norm(psi)
    ref = oracle.apply_gate(psi.copy(), qs, U)
    d = torch.from_numpy(psi.astype(np.complex64)).cuda()
    ctx.apply_gate(d, qs, U)
    torch.cuda.synchronize()
    got = d.cpu().numpy().astype(np.complex128)
    print(n, k, qs, "rel", np.linalg.norm(got - ref) / np.linalg.norm(ref), flush=True)
