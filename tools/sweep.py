"""Gate-pass HBM sweep only (bench.py's SURVEY 8(d) C4 (i) rows): python tools/sweep.py [n] [k...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2111_02396_b200 import qtraj  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
ks = [int(x) for x in sys.argv[2:]] or [1, 2, 3, 4, 5, 6]
peak = bench.load_peaks()[0]["hbm_gbs"]
ctx = qtraj.Context(0)
rng = np.random.default_rng(workloads.circuit_seed(4))
state = torch.zeros(1 << n, dtype=torch.complex64, device="cuda:0")
state[0] = 1.0
for k in ks:
    for name, qs in {"low": list(range(k)), "high": list(range(n - k, n)),
                     "mixed": sorted(int(x) for x in rng.choice(n, size=k, replace=False))}.items():
        U = workloads.haar_unitary(rng, 2 ** k)
        ms = ctx.apply_gate(state, qs, U, repeats=11)
        gbs = 2.0 ** (n + 4) / (ms / 1e3) / 1e9
        print(json.dumps({"k": k, "placement": name, "qubits": qs, "ms": round(ms, 4), "gbs": round(gbs, 1),
                          "frac": round(gbs / peak, 4)}), flush=True)
