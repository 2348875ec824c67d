"""A/B timing of library variants (experiment builds) on the C2 pass kernel and the
n = 30 single-gate sweep.  usage: python tools/ab_libs.py libqtraj.so libqtraj_exp1.so ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, torch
sys.path.insert(0, @ROOT@)
from paper_2111_02396_b200 import qtraj
qtraj.LIB_PATH = qtraj.LIB_PATH.replace("libqtraj.so", @LIB@)
import workloads, bench
c = workloads.sycamore_grid_qcs(config=2)
ctx = qtraj.Context(0)
plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
state = torch.empty(128 << 20, dtype=torch.complex64, device="cuda")
for i in range(3 if @C2@ else 0):
    out = ctx.run_trajectories(plan, state, seed=workloads.trajectory_seed(2), traj_count=1024, batch=128, shots=1,
                               observables=c.observables, profile=True)
if @C2@:
    st = out["stats"]
    print(@LIB@, "C2 1024 traj: pass_kernel_ms %.1f device_ms %.1f" % (st["pass_kernel_ms"], st["device_ms"]), flush=True)
del state; torch.cuda.empty_cache()
if @CHAIN@:
    import numpy as np
    from workloads import Circuit, Gate
    rng = np.random.default_rng(5)
    res = {}
    for G in (1, 2, 4, 8, 16, 32):
        c2 = Circuit(n_qubits=20, moments=[])
        prev = None
        for g in range(G):
            while True:
                qs = sorted(rng.choice(12, 4, replace=False).tolist())
                if qs != prev:
                    break
            prev = qs
            c2.moments.append([Gate(tuple(int(q) for q in qs), workloads.haar_unitary(rng, 16))])
        p2 = qtraj.Plan(qtraj.Circuit.from_description(c2), max_fused=4)
        st2 = torch.empty(128 << 20, dtype=torch.complex64, device="cuda")
        for i in range(3):
            o2 = ctx.run_trajectories(p2, st2, seed=1, traj_count=512, batch=128, shots=1, profile=True)
        s2 = o2["stats"]
        res[G] = (round(s2["pass_kernel_ms"] * 128 / s2["passes"], 4), s2["passes"] / 512)  # ms per 128-slot launch, passes/traj
        del st2
    print(@LIB@, "chain ms per 128-slot pass vs gates/pass:", res, flush=True)
if @SWEEP@:
    s = bench.gate_pass_sweep(ctx, 30, torch.device("cuda", 0), 6554.9)
    print(@LIB@, "sweep", {k: v for k, v in s.items() if "frac" in k or k == "gbps"}, flush=True)
    print(@LIB@, "sweep k=5,6", [(r["k"], r["placement"], round(r["frac"], 3)) for r in s["rows"] if r["k"] >= 5],
          flush=True)
'''
sweep = "--sweep" in sys.argv
chain = "--chain" in sys.argv
for lib in [a for a in sys.argv[1:] if not a.startswith("--")]:
    code = CODE.replace("@ROOT@", repr(ROOT)).replace("@LIB@", repr(lib)).replace("@SWEEP@", str(sweep)).replace("@CHAIN@", str(chain)).replace("@C2@", str("--no-c2" not in sys.argv))
    subprocess.run([sys.executable, "-c", code], cwd=ROOT)
