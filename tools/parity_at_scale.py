"""Oracle parity at the benchmark's scale (VERDICT r1 "Next round" 1(i)/(ii)).

C2 (20 qubits, bench workload): trajectory indices t = 17 + 39 j, j < 256, spread over
[0, 10^4); the GPU runs them in the bench's launch configuration (f = 4, tensor cores,
batch 256) and, for batch invariance, inside the full 10^4-trajectory bench job; the
oracle (mode (i), one trajectory per host core) runs the same indices.
C3 size (26 qubits, low-noise 2 x 13 grid, `--cycles` cycles): 2 trajectories, GPU at
f = 4 and f = 6, oracle in range-parallel mode (ii).

Reports decision mismatches (explained = oracle margin < 1e-4, SURVEY 8(c) "Marginal
decisions"; unexplained = anything else), the relative L2 error of the final states
(max / p99 over non-diverged trajectories) and the largest observable error.
usage: python tools/parity_at_scale.py [--config 2|3] [--count 256] [--out FILE]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import workloads  # noqa: E402
from paper_2111_02396_b200 import qtraj  # noqa: E402

MARGIN = 1e-4


def compare(ref, out, psi_gpu):
    bad_k = np.argwhere(out["kraus"] != ref["kraus"])
    k_expl = [(int(t), int(c)) for t, c in bad_k if ref["kraus_margin"][t, c] < MARGIN]
    k_unexpl = [(int(t), int(c)) for t, c in bad_k if ref["kraus_margin"][t, c] >= MARGIN]
    diverged = sorted(set(int(t) for t, _ in bad_k))
    bad_b = np.argwhere(out["bits"] != ref["bits"])
    b_expl = [(int(t), int(s)) for t, s in bad_b if int(t) not in diverged and ref["sample_margin"][t, s] < MARGIN]
    b_unexpl = [(int(t), int(s)) for t, s in bad_b if int(t) not in diverged and ref["sample_margin"][t, s] >= MARGIN]
    keep = [t for t in range(len(ref["bits"])) if t not in diverged]
    rel = []
    for t in keep:
        p = psi_gpu[t] / np.linalg.norm(psi_gpu[t])
        rel.append(float(np.linalg.norm(p - ref["states"][t]) / np.linalg.norm(ref["states"][t])))
    obs_err = float(np.max(np.abs(out["obs"][keep] - ref["obs"][keep]))) if keep and ref["obs"].shape[1] else 0.0
    return {
        "trajectories": int(len(ref["bits"])),
        "kraus_decisions": int(ref["kraus"].size), "sample_decisions": int(ref["bits"].size * 0 + ref["bits"].size),
        "kraus_mismatch_explained": len(k_expl), "kraus_mismatch_unexplained": len(k_unexpl),
        "sample_mismatch_explained": len(b_expl), "sample_mismatch_unexplained": len(b_unexpl),
        "diverged_trajectories": diverged,
        "rel_l2_max": max(rel) if rel else None, "rel_l2_p99": float(np.percentile(rel, 99)) if rel else None,
        "rel_l2_median": float(np.median(rel)) if rel else None,
        "obs_max_abs_err": obs_err,
        "min_oracle_kraus_margin": float(np.min(ref["kraus_margin"])),
        "min_oracle_sample_margin": float(np.min(ref["sample_margin"])),
    }


def gpu_run(c, seed, begin, stride, count, f, batch, tile_bits=0):
    ctx = qtraj.Context(0)
    plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=f, tile_bits=tile_bits)
    state = torch.zeros(batch << c.n_qubits, dtype=torch.complex64, device="cuda")
    out = ctx.run_trajectories(plan, state, seed=seed, traj_count=count, traj_begin=begin, traj_stride=stride,
                               shots=1, batch=batch, observables=c.observables)
    torch.cuda.synchronize()
    psi = state.view(batch, -1)[:count].cpu().numpy().astype(np.complex128)
    return out, psi


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--count", type=int, default=256)
    ap.add_argument("--cycles", type=int, default=2)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = {"config": a.config, "host_cores": os.cpu_count()}
    if a.config == 2:
        c = workloads.sycamore_grid_qcs(config=2)
        seed = workloads.trajectory_seed(2)
        begin, stride, count = 17, 39, a.count
        t0 = time.time()
        ref = oracle.run_trajectories(c, seed=seed, traj_begin=begin, stride=stride, traj_count=count, shots=1,
                                      want_states=True)
        res["oracle_s"] = time.time() - t0
        assert ref["rc"] == 0
        # per-tile kernel (12-qubit tiles), persistent TMEM kernel (13, the default), the
        # experimental TMA-pipelined kernel (11); the last full run is the default's
        for tile_bits in (12, 11, 13):
            out, psi = gpu_run(c, seed, begin, stride, count, 4, count, tile_bits)
            res[f"gpu_f4_tile{tile_bits}"] = compare(ref, out, psi)
        # batch invariance: the same indices inside the full bench job (batch 384)
        ctx = qtraj.Context(0)
        plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4)
        state = torch.zeros(384 << c.n_qubits, dtype=torch.complex64, device="cuda")
        full = ctx.run_trajectories(plan, state, seed=seed, traj_count=10000, shots=1, batch=384,
                                    observables=c.observables)
        idx = begin + stride * np.arange(count)
        res["bench_job_records_equal"] = bool((full["kraus"][idx] == out["kraus"]).all() and
                                              (full["bits"][idx] == out["bits"]).all())
    else:
        c = workloads.low_noise_grid(rows=2, cols=13, cycles=a.cycles)
        seed = workloads.trajectory_seed(3)
        t0 = time.time()
        ref = oracle.run_trajectories(c, seed=seed, traj_count=2, shots=1, want_states=True, range_parallel=True)
        res["oracle_s"] = time.time() - t0
        res["ops"] = sum(1 for _ in c.ops())
        assert ref["rc"] == 0
        for f in (4, 6):
            out, psi = gpu_run(c, seed, 0, 1, 2, f, 2)
            res[f"gpu_f{f}"] = compare(ref, out, psi)
        out, psi = gpu_run(c, seed, 0, 1, 2, 4, 2, 11)
        res["gpu_f4_tile11"] = compare(ref, out, psi)
    print(json.dumps(res))
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
