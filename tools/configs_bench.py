"""Measured runs of the SURVEY 8(d) configs other than the bench line (C2):

  C1     GHZ-4 with depolarizing 0.01 after every gate, 1 000 trajectories in one
         batch (launch-latency bound: the whole state is one 128-byte tile).

  C3     26-qubit low-noise grid (2 x 13, 20 cycles, depolarize 1e-3 after every
         gate + phase_damp 1e-4 on every qubit per moment), f = 4, 5, 6: trajectories/s,
         passes and fused gates per trajectory, deferral fraction, reductions.
  C4(ii) one noisy 32-qubit trajectory (4 x 8 grid, 20 cycles, depolarize 1e-3 +
         amplitude_damp 1e-4): seconds per trajectory, passes, algorithmic GB/s.

Device time from CUDA events around qt_run_trajectories (host planning overlaps).
One JSON line per run."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2111_02396_b200 import qtraj  # noqa: E402


def run(ctx, c, cfg, f, traj, batch, seed, peak):
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=f)
    state = torch.empty(batch << c.n_qubits, dtype=torch.complex64, device="cuda")
    kw = dict(seed=seed, shots=1, batch=batch, observables=c.observables[:4])
    ctx.run_trajectories(plan, state, traj_count=min(batch, traj), traj_begin=10**6, **kw)  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = ctx.run_trajectories(plan, state, traj_count=traj, profile=True, **kw)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st = out["stats"]
    ch = st["channels_deferred"] + st["channels_conventional"]
    line = {"config": cfg, "n": c.n_qubits, "f": f, "trajectories": traj, "batch": batch, "ms": ms,
            "traj_per_s": traj / (ms / 1e3), "ms_per_traj": ms / traj,
            "passes_per_traj": st["passes"] / traj, "fused_gates_per_traj": st["fused_gates"] / traj,
            "reductions_per_traj": st["reductions"] / traj,
            "deferral_fraction": st["channels_deferred"] / max(ch, 1),
            "pass_kernel_ms": st["pass_kernel_ms"],
            "pass_alg_gbs": st["alg_bytes"] / (st["pass_kernel_ms"] / 1e3) / 1e9,
            "pass_alg_frac": st["alg_bytes"] / (st["pass_kernel_ms"] / 1e3) / 1e9 / peak}
    print(json.dumps(line), flush=True)
    del state
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c3-traj", type=int, default=1000)
    ap.add_argument("--c4", type=int, default=1)
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6553.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6553.0
    ctx = qtraj.Context(0)
    c1 = workloads.ghz4_depolarized(0.01)
    run(ctx, c1, "C1 GHZ-4 depolarizing 0.01", 4, 1000, 1000, workloads.trajectory_seed(1), peak)
    c3 = workloads.low_noise_grid(config=3)
    for f in (4, 5, 6):
        run(ctx, c3, "C3 26q low-noise grid", f, a.c3_traj, 32, workloads.trajectory_seed(3), peak)
    if a.c4:
        c4 = workloads.low_noise_grid(rows=4, cols=8, cycles=20, config=4, depol=1e-3, gamma_pd=1e-4,
                                      damping="amplitude")
        run(ctx, c4, "C4(ii) 32q one noisy trajectory", 4, 1, 1, workloads.trajectory_seed(4), peak)


if __name__ == "__main__":
    main()
