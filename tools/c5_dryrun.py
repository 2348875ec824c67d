"""C5 dry run (BASELINE config 5: 36 qubits over 8 x B200, 33 local + 3 global
qubits, 6 x 6 grid, 10 cycles, noiseless and amplitude damping gamma = 1e-3): the
distributed-state engine (paper_2111_02396_b200/distributed.py) runs its real
schedule -- Belady victim choice, local permutations, all-to-all exchanges, flushes
of buffered local operations through the library's fuser -- on a host-only backend
that keeps no state, and the result is priced with measured B200 rates.

Recorded per trajectory: global-qubit swaps, bytes each rank sends, local
permutation passes, flushes and their tile passes (qt_plan_info of every flushed
plan), conventional rho_Q reductions.  Predicted time per trajectory = tile passes x
2^(n_local + 4) B / HBM rate + permutations x 2^(n_local + 4) B / HBM rate +
reductions x 2^(n_local + 3) B / HBM rate + exchanged bytes / NVLink rate (900 GB/s
per direction per GPU, NVSwitch all-to-all); the HBM rate is the C4 gate-pass sweep's
measured fraction of MEASURED_PEAKS.json (assumption stated in the output).
Conventional channels are priced, but their outcomes are taken as the no-jump
branch (the dry backend holds no amplitudes); every deferred pick is the real draw.

usage: python tools/c5_dryrun.py [--gamma 1e-3] [--hbm-frac 0.70] [--out FILE]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import workloads  # noqa: E402
from workloads import Channel, channels  # noqa: E402
from paper_2111_02396_b200 import distributed as D  # noqa: E402
from paper_2111_02396_b200 import qtraj  # noqa: E402


class DryState:
    """Stands in for a rank's 2^n_local amplitudes: shape bookkeeping only."""

    def __init__(self, nl):
        self.nl = nl
        self.is_cuda = False

    def numel(self):
        return 1 << self.nl

    def contiguous(self):
        return self


class DryBackend:
    def __init__(self, max_fused=4):
        self.max_fused = max_fused
        self.passes = 0
        self.flushes = 0
        self.permutes = 0
        self.reductions = 0
        self.plan_gates = 0

    def new_state(self, nl, rank):
        return DryState(nl)

    def apply_ops(self, state, nl, ops):
        c = qtraj.Circuit(nl)
        for i, (pos, M) in enumerate(ops):
            c.add_matrix(i, pos, M)
        info = qtraj.Plan(c, max_fused=max(self.max_fused, max(len(p) for p, _ in ops))).info(0, 0)
        self.passes += info["passes"]
        self.plan_gates += info["fused_gates"]
        self.flushes += 1

    def permute(self, state, perm):
        self.permutes += 1
        return state

    def take_spare(self, like):
        return DryState(like.nl)

    def give_spare(self, t):
        pass

    def reduce_rho(self, state, positions):
        self.reductions += 1
        d = 1 << len(positions)
        rho = np.zeros((d, d), np.complex128)
        rho[0, 0] = 1.0 / 8  # the no-jump branch dominates; the total over ranks is what matters
        return rho

    def expect(self, state, observables):
        return np.zeros(len(observables)), 1.0 / 8

    def sample_local(self, state, n_total, seed, traj, shot_ids):
        return np.zeros(len(shot_ids), np.uint64)


class DryFabric:
    """All 8 ranks in one process, no data: exchanges keep the (dry) slices."""

    def __init__(self, world):
        self.world = world
        self.local_ranks = list(range(world))
        self.exchanges = []

    def exchange_top(self, states, gbits, s, pool=None, on_chunk=None):
        # per exchange: s and the tile passes per rank of the operations deferred into it
        # (applied per received chunk while the other chunks are in flight); priced once per
        # rank on its whole slice, the same bytes as per chunk
        before = pool.passes if pool is not None else 0
        if on_chunk is not None:
            for r, st in states.items():
                on_chunk(r, st)
        deferred = (pool.passes - before) / self.world if pool is not None else 0.0
        self.exchanges.append((s, deferred))
        return dict(states)

    def allreduce(self, per_rank):
        return sum(np.asarray(v) for v in per_rank.values())

    def allgather(self, per_rank):
        return np.array([float(per_rank[r]) for r in range(self.world)])

    def broadcast_u64(self, arr, owner):
        return arr


def c5_circuit(n, cycles, gamma):
    c = workloads.sycamore_grid_qcs(rows=6, cols=6, cycles=cycles, config=5, noise=False)
    if gamma > 0:
        moms = []
        for m in c.moments:
            moms.append(m)
            moms.append([Channel((q,), channels.amplitude_damp(gamma)) for q in range(n)])
        c.moments = moms
    c.observables = []
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gamma", type=float, default=1e-3)
    ap.add_argument("--cycles", type=int, default=10)
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--hbm-frac", type=float, default=0.70, help="gate-pass fraction of the HBM peak (C4 sweep)")
    ap.add_argument("--nvlink-gbs", type=float, default=900.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    n = 36
    g = a.world.bit_length() - 1
    nl = n - g
    peaks = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm = json.load(open(peaks))["hbm_gbs"] if os.path.exists(peaks) else 6554.9
    rate = hbm * a.hbm_frac * 1e9
    out = {"workload": f"C5 36q 6x6 grid, {a.cycles} cycles", "world": a.world, "n_local": nl,
           "hbm_gbs_peak": hbm, "hbm_frac_assumed": a.hbm_frac, "nvlink_gbs_per_direction": a.nvlink_gbs}
    for gamma in sorted({0.0, a.gamma}):
        c = c5_circuit(n, a.cycles, gamma)
        b = DryBackend()
        fab = DryFabric(a.world)
        tr = D.DistributedTrajectory(b, fab, n)
        res = tr.run(c, seed=workloads.trajectory_seed(5), traj=0, shots=1)
        per_rank_bytes = tr.exchanged_bytes / a.world
        state_b = 8.0 * (1 << nl)
        deferred_passes = sum(d for _, d in fab.exchanges)
        t_pass = (b.passes - deferred_passes * a.world) * 2 * state_b / rate
        t_perm = b.permutes / a.world * 2 * state_b / rate
        t_red = b.reductions / a.world * state_b / rate
        t_x = per_rank_bytes / (a.nvlink_gbs * 1e9)
        # exchange phases: 2^s - 1 pairwise rounds; the deferred passes run per received
        # chunk (own chunk during round 1), so a phase takes
        # R max(x / R, p / 2^s) + p / 2^s for transfer time x and deferred pass time p
        t_xphase, t_xphase_serial = 0.0, 0.0
        for sk, dk in fab.exchanges:
            xk = (1 - 2.0 ** -sk) * state_b / (a.nvlink_gbs * 1e9)
            pk = dk * 2 * state_b / rate
            rr = (1 << sk) - 1
            t_xphase += rr * max(xk / rr, pk / (1 << sk)) + pk / (1 << sk)
            t_xphase_serial += xk + pk
        key = "noiseless" if gamma == 0 else f"amplitude_damping_{gamma:g}"
        out[key] = {
            "ops": sum(1 for _ in c.ops()), "swaps": int(res["swaps"]), "bytes_sent_per_rank": per_rank_bytes,
            "local_permutations_per_rank": b.permutes / a.world, "flushes": b.flushes / a.world,
            "tile_passes_per_rank": b.passes / a.world, "fused_gates_per_rank": b.plan_gates / a.world,
            "rho_reductions_per_rank": b.reductions / a.world,
            "deferred_tile_passes_per_rank": deferred_passes,
            "predicted_s": {"tile_passes": t_pass / a.world, "permutations": t_perm, "reductions": t_red,
                            "exchanges": t_x,
                            "exchange_phases_overlapped": t_xphase,
                            "exchange_phases_serial": t_xphase_serial,
                            "total": t_pass / a.world + t_perm + t_red + t_xphase,
                            "total_without_overlap": t_pass / a.world + t_perm + t_red + t_xphase_serial},
        }
    print(json.dumps(out, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
