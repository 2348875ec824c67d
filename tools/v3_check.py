"""tile_pass_v3 (tile_bits = 11) parity vs the oracle on a few circuit families, then C2 timing."""
import os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle, workloads
from paper_2111_02396_b200 import qtraj
import test_gpu_parity as tp

ctx = qtraj.Context(0)


def run_v3(c, seed, T, shots=1, tb=11, batch=0):
    ref = oracle.run_trajectories(c, seed=seed, traj_count=T, shots=shots, want_states=True)
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4, tile_bits=tb)
    batch = batch or T
    state = torch.zeros(batch << c.n_qubits, dtype=torch.complex64, device="cuda")
    out = ctx.run_trajectories(plan, state, seed=seed, traj_count=T, shots=shots, batch=batch, observables=c.observables)
    torch.cuda.synchronize()
    return ref, out, state, plan


cases = [
    ("unitary n14", workloads.random_circuit(14, depth=6, seed=3, noise="none"), 4),
    ("depol n16", workloads.random_circuit(16, depth=6, seed=4, noise="depol", p=0.02), 6),
    ("damping n14", workloads.random_circuit(14, depth=6, seed=5, noise="both", p=0.02, t1_ns=800.0, tphi_ns=1500.0,
                                             readout=True), 8),
    ("C2 n20", workloads.sycamore_grid_qcs(config=2), 16),
]
for name, c, T in cases:
    try:
        ref, out, state, plan = run_v3(c, seed=7, T=T, shots=2)
        info = plan.info(7, 0)
        nd = tp.compare(ref, out, state)
        psi = state.view(T, -1).cpu().numpy().astype(np.complex128)
        psi /= np.linalg.norm(psi, axis=1, keepdims=True)
        rel = np.linalg.norm(psi - ref["states"], axis=1) / np.linalg.norm(ref["states"], axis=1)
        print(name, "OK diverged", nd, "max rel", float(rel.max()), "kernel", info["kernel"], "passes", info["passes"], flush=True)
    except AssertionError as e:
        print(name, "FAIL", str(e)[:300], flush=True)
    except Exception as e:
        print(name, "ERROR", type(e).__name__, str(e)[:300], flush=True)
# timing: C2 1024 trajectories, v3 vs v2
c = workloads.sycamore_grid_qcs(config=2)
for tb in (11, 13, 11, 13):
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4, tile_bits=tb)
    state = torch.empty(384 << 20, dtype=torch.complex64, device="cuda")
    for _ in range(2):
        torch.cuda.synchronize(); t0 = time.time()
        out = ctx.run_trajectories(plan, state, seed=workloads.trajectory_seed(2), traj_count=1536, batch=384, shots=1,
                                   observables=c.observables, profile=True)
        torch.cuda.synchronize()
    st = out["stats"]
    print("tile_bits", tb, "1536 traj: wall %.1f ms pass_kernel_ms %.1f device_ms %.1f passes/traj %.2f" % (
        (time.time() - t0) * 1e3, st["pass_kernel_ms"], st["device_ms"], st["passes"] / 1536), flush=True)
    del state
