"""Distributed-state mode benchmark (config 5 shape: grid circuit, 10 cycles,
noiseless or amplitude damping gamma = 1e-3 per qubit per moment).

  torchrun --nproc-per-node N tools/dist_bench.py --n-local 33    # C5: 36 q on 8 GPUs
  python tools/dist_bench.py --emulate 8 --n-local 26             # one GPU, 8 virtual ranks
  python tools/dist_bench.py --emulate 8 --n-local 30 --mirror    # 33 q: C then C^dag -> |0...0>

Prints one JSON line (rank 0): seconds per trajectory, swaps, exchanged bytes."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from workloads import Channel, channels  # noqa: E402
from paper_2111_02396_b200 import distributed as D  # noqa: E402
from paper_2111_02396_b200 import qtraj  # noqa: E402


def c5_circuit(n, cycles, gamma):
    rows = int(np.floor(np.sqrt(n)))
    while n % rows:
        rows -= 1
    c = workloads.sycamore_grid_qcs(rows=rows, cols=n // rows, cycles=cycles, config=5, noise=False)
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
    ap.add_argument("--n-local", type=int, default=26)
    ap.add_argument("--emulate", type=int, default=0, help="virtual ranks in one process (1 GPU)")
    ap.add_argument("--cycles", type=int, default=10)
    ap.add_argument("--gamma", type=float, default=0.0)
    ap.add_argument("--traj", type=int, default=1)
    ap.add_argument("--mirror", action="store_true",
                    help="noiseless C then C^dag: every sample must be 0...0 and every <Z_q> = 1")
    a = ap.parse_args()
    if a.emulate:
        world, rank, local = a.emulate, 0, 0
        fabric = D.EmulatedFabric(world)
    else:
        import torch.distributed as dist
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        world, rank = dist.get_world_size(), dist.get_rank()
        fabric = D.TorchFabric(device=torch.device("cuda", local))
    g = world.bit_length() - 1
    n = a.n_local + g
    ctx = qtraj.Context(local)
    backend = D.GpuBackend(ctx, torch.device("cuda", local))
    c = c5_circuit(n, a.cycles, 0.0 if a.mirror else a.gamma)
    if a.mirror:
        inv = [[workloads.Gate(op.qubits, np.conj(np.asarray(op.matrix)).T) for op in m] for m in reversed(c.moments)]
        c.moments = c.moments + inv
        c.observables = ["I" * q + "Z" + "I" * (n - q - 1) for q in (0, n // 2, n - 1)]
    shots = 16 if a.mirror else 1
    mirror_ok = True
    times, swaps, xbytes = [], [], []
    for t in range(a.traj + 1):  # trajectory 0 = warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tr = D.DistributedTrajectory(backend, fabric, n)
        out = tr.run(c, seed=workloads.trajectory_seed(5), traj=t, shots=shots, observables=c.observables)
        torch.cuda.synchronize()
        if a.mirror:
            mirror_ok &= bool(np.all(out["bits"] == 0)) and bool(np.allclose(out["obs"], 1.0, atol=1e-4))
        if t:
            times.append(time.perf_counter() - t0)
            swaps.append(out["swaps"])
            xbytes.append(tr.exchanged_bytes)
        del tr
    if rank == 0:
        print(json.dumps({"mode": "emulated" if a.emulate else "nccl", "world": world, "n": n, "n_local": a.n_local,
                          "cycles": a.cycles, "gamma": a.gamma, "ops": sum(1 for _ in c.ops()),
                          "s_per_traj": float(np.mean(times)), "swaps_per_traj": float(np.mean(swaps)),
                          "exchanged_GB_per_rank": float(np.mean(xbytes)) / 1e9 / max(1, len(fabric.local_ranks)),
                          **({"mirror_all_zero_and_Z_1": mirror_ok} if a.mirror else {})}),
              flush=True)


if __name__ == "__main__":
    main()
