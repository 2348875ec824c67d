"""Streaming single-gate kernel (gate_stream.cu) quick check: oracle parity for k = 1..6
over placements at a few n, then the n = 30 / 32 gate-pass sweep."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import workloads  # noqa: E402
import bench  # noqa: E402
from paper_2111_02396_b200 import qtraj  # noqa: E402

ctx = qtraj.Context(0)
rng = np.random.default_rng(7)
worst = 0.0
for n in (13, 14, 17, 20, 23):
    for k in range(1, 7):
        if n < 7 + max(k, 4):
            continue
        pl = [list(range(k)), list(range(n - k, n)), sorted(rng.choice(n, k, replace=False).tolist()),
              rng.choice(n, k, replace=False).tolist()]
        for qs in pl:
            U = workloads.haar_unitary(rng, 2 ** k)
            psi = (rng.normal(size=2 ** n) + 1j * rng.normal(size=2 ** n))
            psi /= np.linalg.norm(psi)
            ref = oracle.apply_gate(psi.copy(), qs, U)
            d = torch.from_numpy(psi.astype(np.complex64)).cuda()
            ctx.apply_gate(d, qs, U)
            got = d.cpu().numpy().astype(np.complex128)
            rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            worst = max(worst, rel)
            if rel > 1e-5:
                print("FAIL", n, k, qs, rel, flush=True)
    print("n", n, "done, worst rel-L2 so far", worst, flush=True)
for n in ([int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else []):
    s = bench.gate_pass_sweep(ctx, n, torch.device("cuda", 0), 6536.4, reps=10)
    print(n, [(r["k"], r["placement"], round(r["frac"], 3)) for r in s["rows"]], flush=True)
    torch.cuda.empty_cache()
