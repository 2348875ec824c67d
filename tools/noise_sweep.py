"""NEXT-1: runtime per trajectory vs phase-damping strength, delayed inner
products (Alg. 2) vs the conventional algorithm, cf. Fig. perf_noise
("runtime increases linearly with the noise strength"; "order of
magnitude runtime speedup for low noise with 27 qubits").

Workload: Sycamore-style grid circuit (noiseless gates) with phase_damp(gamma)
on every qubit after every moment (workloads.low_noise_grid with depol = 0).
Prints one JSON line per (n, gamma, mode)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2111_02396_b200 import qtraj  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--qubits", type=str, default="20,26")
    ap.add_argument("--gammas", type=str, default="0.0001,0.001,0.01,0.1")
    ap.add_argument("--cycles", type=int, default=20)
    ap.add_argument("--traj", type=int, default=0, help="0 = auto per n")
    a = ap.parse_args()
    ctx = qtraj.Context(0)
    for n in [int(x) for x in a.qubits.split(",")]:
        rows, cols = {20: (4, 5), 27: (3, 9)}.get(n, (2, n // 2))
        for g in [float(x) for x in a.gammas.split(",")]:
            # pure phase damping (depol = 0 drops the depolarizing channels), as in Fig. perf_noise
            c = workloads.low_noise_grid(rows=rows, cols=cols, cycles=a.cycles, config=3, depol=0.0, gamma_pd=g)
            plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
            for mode in (0, 1):
                T = a.traj or (256 if n <= 20 else 16)
                if mode == 1:
                    T = max(4, T // 16)
                batch = min(T, 128 if n <= 20 else 8)
                state = torch.empty(batch << n, dtype=torch.complex64, device="cuda")
                ctx.run_trajectories(plan, state, seed=11, traj_count=batch, batch=batch, shots=1, mode=mode)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                out = ctx.run_trajectories(plan, state, seed=12, traj_count=T, batch=batch, shots=1, mode=mode)
                torch.cuda.synchronize()
                dt = time.perf_counter() - t0
                st = out["stats"]
                print(json.dumps({"n": n, "gamma": g, "mode": ["delayed", "conventional"][mode], "trajectories": T,
                                  "ms_per_traj": 1e3 * dt / T, "passes_per_traj": st["passes"] / T,
                                  "reductions_per_traj": st["reductions"] / T,
                                  "deferral_fraction": st["channels_deferred"] / max(
                                      1, st["channels_deferred"] + st["channels_conventional"])}), flush=True)
                del state
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
